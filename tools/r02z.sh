# 1 GPU: final checks of the round -- pytest -m gpu, smoke, bench, ncu decode-GEMM traffic
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02z
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02z/pytest_gpu.log 2>&1; tail -5 gpurun_out/r02z/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02z/smoke.log 2>&1; tail -2 gpurun_out/r02z/smoke.log
timeout 1500 python bench.py > gpurun_out/r02z/bench.json 2> gpurun_out/r02z/bench.err; tail -c 1500 gpurun_out/r02z/bench.json
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_bf16 --csv --log-file gpurun_out/r02z/gemm_traffic.csv python tools/gemm_traffic.py > gpurun_out/r02z/gemm_traffic.log 2>&1
python tools/gemm_traffic.py --summarise gpurun_out/r02z/gemm_traffic.csv --out gpurun_out/r02z/ncu_gemm_traffic.json | head -40
