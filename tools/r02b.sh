set -x
free -g | head -2; nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -q -m gpu --durations=20 -p no:cacheprovider > gpurun_out/r02b_pytest.log 2>&1
tail -40 gpurun_out/r02b_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; tail -2 gpurun_out/r02b_smoke.log
timeout 900 python bench.py --steps 1 --warmup 1 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; tail -c 3000 gpurun_out/r02b_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_ncu_maxout256.csv python bench.py --steps 1 --warmup 0 --max-out 256 --no-cpu-baseline --no-kernel-timing > gpurun_out/r02b_ncu.log 2>&1
echo ncu_rc=$?
python tools/ncu_shares.py gpurun_out/r02b_ncu_maxout256.csv --what "c2 --max-out 256, whole run" | head -30
