set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02m
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "prefill" > gpurun_out/r02m/pytest_prefill.log 2>&1; tail -15 gpurun_out/r02m/pytest_prefill.log
for L in 512 1024 2048; do timeout 120 python tools/prefill_bench.py 32 $L; SGS_PREFILL_LEGACY=1 timeout 120 python tools/prefill_bench.py 32 $L; done 2>&1 | tee gpurun_out/r02m/prefill_bench.log
timeout 900 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider -k "chained or c2_scale or 7b_shape or layer_local or tiny" > gpurun_out/r02m/pytest_engine.log 2>&1; tail -3 gpurun_out/r02m/pytest_engine.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_prefill_tc -s 3 -c 1 -o gpurun_out/r02m/prefill_tc python tools/prefill_bench.py 32 512 > gpurun_out/r02m/ncu.log 2>&1; echo ncu_rc=$?
ncu -i gpurun_out/r02m/prefill_tc.ncu-rep --page details --csv > gpurun_out/r02m/prefill_tc.details.csv 2>/dev/null
