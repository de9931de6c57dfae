set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02q
export SGS_TEST_STACK_DUMP_S=150
for ar in nccl p2p; do
timeout 280 python -m pytest tests/test_gpu_multi.py -x -q -s -p no:cacheprovider -k "tensor_parallel and tiny and $ar" > gpurun_out/r02q/tp_tiny_$ar.log 2>&1; echo rc=$?
tail -c 3000 gpurun_out/r02q/tp_tiny_$ar.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 tools/tp_experiment.py --mode sweep --b 1 4 16 64 256 --out gpurun_out/r02q/tp_sweep.json > gpurun_out/r02q/tp_sweep.log 2>&1
tail -12 gpurun_out/r02q/tp_sweep.log | cut -c1-300
