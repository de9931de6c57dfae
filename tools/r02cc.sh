# 4 GPUs: NEXT-2 at TP = 4 -- the 7B TP=4 instance against the oracle, and its T(b) (peer-memory exchange vs NCCL)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02cc
timeout 900 python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider -k "tensor_parallel and 4" > gpurun_out/r02cc/pytest_tp4.log 2>&1; grep -E "PASS|FAIL|ERROR|passed|failed|Error" gpurun_out/r02cc/pytest_tp4.log | tail -8
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 tools/tp_experiment.py --mode sweep --b 1 4 16 64 256 --out gpurun_out/r02cc/tp4_sweep.json > gpurun_out/r02cc/tp4_sweep.log 2>&1
grep '"b"' gpurun_out/r02cc/tp4_sweep.log | cut -c1-200
