set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02t
export SGS_DEBUG_SIGNALS=1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider -k "tensor_parallel" > gpurun_out/r02t/pytest_tp.log 2>&1; echo rc=$?
tail -30 gpurun_out/r02t/pytest_tp.log | cut -c1-400
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 tools/tp_experiment.py --mode sweep --b 1 4 16 64 256 --out gpurun_out/r02t/tp_sweep.json > gpurun_out/r02t/tp_sweep.log 2>&1
grep '"b"' gpurun_out/r02t/tp_sweep.log | cut -c1-200
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 tools/timeline.py --tp 2 --b 1 16 64 256 --out gpurun_out/r02t/timeline_tp2.json > gpurun_out/r02t/timeline_tp2.log 2>&1
tail -5 gpurun_out/r02t/timeline_tp2.log | cut -c1-300
