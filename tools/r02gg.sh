# 4 GPUs: the driver's scaling command at N = 2 and 4 (bench.py under torchrun) on the current tree
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02gg
for n in 4 2; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --steps 1 --warmup 3 > gpurun_out/r02gg/bench_n$n.json 2> gpurun_out/r02gg/bench_n$n.err; grep "\[bench" gpurun_out/r02gg/bench_n$n.err; tail -c 300 gpurun_out/r02gg/bench_n$n.json
done
