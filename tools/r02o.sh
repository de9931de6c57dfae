# 2 GPUs: multi-GPU tests incl. the TP = 2 instance vs the oracle, TP T(b) sweep
set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02o
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_kernels.py -q -p no:cacheprovider -k "prefill or 7b_width or chained or prefix" > gpurun_out/r02o/pytest_1gpu.log 2>&1; tail -3 gpurun_out/r02o/pytest_1gpu.log
for L in 512 2048; do timeout 120 python tools/prefill_bench.py 32 $L; done
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/r02o/pytest_multi.log 2>&1; tail -15 gpurun_out/r02o/pytest_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tools/tp_experiment.py --mode sweep --ctx 2048 --out gpurun_out/r02o/tp_sweep_ctx2048.json > gpurun_out/r02o/tp_sweep.log 2>&1; grep '"b"' gpurun_out/r02o/tp_sweep.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 tools/tp_experiment.py --mode sweep --ctx 8192 --b 1 4 16 32 64 --out gpurun_out/r02o/tp_sweep_ctx8192.json > gpurun_out/r02o/tp_sweep8k.log 2>&1; grep '"b"' gpurun_out/r02o/tp_sweep8k.log
