# 1 GPU: final checks -- pytest -m gpu, smoke, T(b) at ctx 2048, the default bench command
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02mm
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02mm/pytest_gpu.log 2>&1; tail -3 gpurun_out/r02mm/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02mm/smoke.log 2>&1; tail -1 gpurun_out/r02mm/smoke.log
timeout 600 python tools/tb_sweep.py --ctx 2048 --b 1 16 64 256 --decode-iters 8 --out gpurun_out/r02mm/tb_ctx2048.json > gpurun_out/r02mm/tb.log 2>&1; grep '"b"' gpurun_out/r02mm/tb.log | cut -c1-100
timeout 1200 python bench.py > gpurun_out/r02mm/bench.json 2> gpurun_out/r02mm/bench.err; grep "\[bench" gpurun_out/r02mm/bench.err; tail -c 200 gpurun_out/r02mm/bench.json
