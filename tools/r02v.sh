# 1 GPU: decode-GEMM DRAM traffic (ncu) for the bench roofline; attention planner variants at small b
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02v
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_bf16 --csv --log-file gpurun_out/r02v/gemm_traffic.csv python tools/gemm_traffic.py > gpurun_out/r02v/gemm_traffic.log 2>&1
python tools/gemm_traffic.py --summarise gpurun_out/r02v/gemm_traffic.csv --out gpurun_out/r02v/ncu_gemm_traffic.json | head -60
for v in "8 296" "4 296" "2 296" "4 592"; do set -- $v
SGS_ATTN_MINPG=$1 SGS_ATTN_SLOTS=$2 timeout 600 python tools/tb_sweep.py --ctx 2048 8192 --b 1 4 16 64 --decode-iters 8 --out gpurun_out/r02v/tb_minpg$1_slots$2.json > gpurun_out/r02v/tb_minpg$1_slots$2.log 2>&1
echo "minpg=$1 slots=$2"; grep '"b"' gpurun_out/r02v/tb_minpg$1_slots$2.log | cut -c1-120
done
