# 1 GPU: decode-attention planner variants at small b (SGS_ATTN_MINPG / SGS_ATTN_SLOTS), T(b) at ctx 2048 / 8192
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02aa
for v in "8 296" "4 296" "4 592" "2 592"; do set -- $v
SGS_ATTN_MINPG=$1 SGS_ATTN_SLOTS=$2 timeout 600 python tools/tb_sweep.py --ctx 2048 8192 --b 1 4 16 --decode-iters 8 --out gpurun_out/r02aa/tb_minpg$1_slots$2.json > gpurun_out/r02aa/tb_minpg$1_slots$2.log 2>&1
echo "minpg=$1 slots=$2"; grep '"b"' gpurun_out/r02aa/tb_minpg$1_slots$2.log | cut -c1-100
done
timeout 900 python tools/stream_handoff.py --config c2_7b --out gpurun_out/r02aa/stream_handoff_c2.json > gpurun_out/r02aa/stream_handoff_c2.log 2>&1; tail -5 gpurun_out/r02aa/stream_handoff_c2.log | cut -c1-600
