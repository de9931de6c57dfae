# 4 GPUs: config 3 at N = 4 per dispatch policy + config 4 (32B) wave 0 of 8 instances + broadcast at 4
set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02g
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 tools/dp_experiment.py --config c3_14b_4 --policies skew,skew_max,random,round_robin --bcast-reps 3 --dump-trace gpurun_out/r02g/traces --out gpurun_out/r02g/c3_n4_oracle_hints.json > gpurun_out/r02g/c3_n4.log 2>&1
tail -5 gpurun_out/r02g/c3_n4.log | cut -c1-300
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 tools/dp_experiment.py --config c3_14b_4 --policies skew,random --hint-noise 0.6 --bcast-reps 0 --out gpurun_out/r02g/c3_n4_noisy_hints.json > gpurun_out/r02g/c3_n4_noisy.log 2>&1
tail -2 gpurun_out/r02g/c3_n4_noisy.log | cut -c1-300
SGS_TRACE_DIR=gpurun_out/r02g/traces timeout 900 python -m pytest tests/test_dp_traces.py -q -p no:cacheprovider > gpurun_out/r02g/pytest_traces.log 2>&1; tail -3 gpurun_out/r02g/pytest_traces.log
rm -rf gpurun_out/r02g/traces
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tools/elastic_experiment.py --steps 6 --out gpurun_out/r02g/elastic_7b.json > gpurun_out/r02g/elastic.log 2>&1
grep step gpurun_out/r02g/elastic.log | cut -c1-300
