# 2 GPUs: multi-GPU tests (weight sync, TP instances) on the default (tiled) weight layout
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02rr
timeout 1500 python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider > gpurun_out/r02rr/pytest_multi.log 2>&1; grep -E "PASS|FAIL|ERROR|passed|failed" gpurun_out/r02rr/pytest_multi.log | tail -12
