# 2 GPUs: multi-GPU pytest (NCCL weight sync), config 3 at N = 2 per dispatch policy, traces vs oracle
set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02e
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/r02e/pytest_multi.log 2>&1; tail -3 gpurun_out/r02e/pytest_multi.log
PROF=${PROF14:-}
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/dp_experiment.py --config c3_14b_2 --policies skew,skew_max,random,round_robin --warmup 0 --bcast-reps 3 --dump-trace gpurun_out/r02e/traces $PROF --out gpurun_out/r02e/c3_n2_oracle_hints.json > gpurun_out/r02e/c3_n2.log 2>&1
tail -6 gpurun_out/r02e/c3_n2.log | cut -c1-400
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/dp_experiment.py --config c3_14b_2 --policies skew,random --hint-noise 0.6 --bcast-reps 0 $PROF --out gpurun_out/r02e/c3_n2_noisy_hints.json > gpurun_out/r02e/c3_n2_noisy.log 2>&1
tail -3 gpurun_out/r02e/c3_n2_noisy.log | cut -c1-400
SGS_TRACE_DIR=gpurun_out/r02e/traces timeout 900 python -m pytest tests/test_dp_traces.py -q -p no:cacheprovider > gpurun_out/r02e/pytest_traces.log 2>&1; tail -3 gpurun_out/r02e/pytest_traces.log
rm -rf gpurun_out/r02e/traces
