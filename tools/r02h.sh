# 4 GPUs: config 4 (32B, 8 instances) as two waves of 4 (round-robin and Alg. 2 dispatch),
# the 65.5 GB broadcast at 4 GPUs, trace parity of wave 0, and the NEXT-2 tail experiment
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02h
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 tools/tp_experiment.py --mode tail --out gpurun_out/r02h/tp_tail.json > gpurun_out/r02h/tp_tail.log 2>&1
grep -E "A_tp2|B_dp4" gpurun_out/r02h/tp_tail.log | cut -c1-300
for off in 0 4; do
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$off tools/dp_experiment.py --config c4_32b --instances 8 --instance-offset $off --policies round_robin,skew --bcast-reps $([ $off = 0 ] && echo 3 || echo 0) $([ $off = 0 ] && echo "--dump-trace gpurun_out/r02h/traces") --out gpurun_out/r02h/c4_wave$off.json > gpurun_out/r02h/c4_wave$off.log 2>&1
tail -4 gpurun_out/r02h/c4_wave$off.log | cut -c1-400
done
SGS_TRACE_DIR=gpurun_out/r02h/traces timeout 900 python -m pytest tests/test_dp_traces.py -q -p no:cacheprovider > gpurun_out/r02h/pytest_traces.log 2>&1; tail -3 gpurun_out/r02h/pytest_traces.log
rm -rf gpurun_out/r02h/traces
