set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02n
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/r02n/pytest_gpu.log 2>&1; tail -22 gpurun_out/r02n/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02n/smoke.log 2>&1; tail -1 gpurun_out/r02n/smoke.log
timeout 1200 python bench.py --steps 1 --warmup 1 > gpurun_out/r02n/bench.json 2> gpurun_out/r02n/bench.err; tail -c 2500 gpurun_out/r02n/bench.json
for ps in "" "--prefix-sharing"; do timeout 900 python bench.py --steps 1 --warmup 1 --group-size 8 $ps --no-cpu-baseline --no-timeline > gpurun_out/r02n/bench_grpo8$ps.json 2> gpurun_out/r02n/bench_grpo8$ps.err; head -c 600 gpurun_out/r02n/bench_grpo8$ps.json; echo; done
