set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02p
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider -k "tensor_parallel and tiny" > gpurun_out/r02p/pytest_tp_tiny.log 2>&1; grep -E "^E|Error|passed|failed" gpurun_out/r02p/pytest_tp_tiny.log | head -30
