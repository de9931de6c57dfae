set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02l
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "attention" > gpurun_out/r02l/pytest_attn.log 2>&1; tail -3 gpurun_out/r02l/pytest_attn.log
timeout 600 python tools/attn_sweep.py --b 4 8 16 32 64 128 256 --ctx 1024 8192 32768 --out gpurun_out/r02l/attn.json > gpurun_out/r02l/attn.log 2>&1; tail -1 gpurun_out/r02l/attn.log
timeout 600 python tools/tb_sweep.py --ctx 2048 8192 --b 1 16 32 64 256 --out gpurun_out/r02l/tb.json > gpurun_out/r02l/tb.log 2>&1; grep '"b"' gpurun_out/r02l/tb.log
timeout 900 python bench.py --steps 1 --warmup 1 > gpurun_out/r02l/bench.json 2> gpurun_out/r02l/bench.err; head -c 400 gpurun_out/r02l/bench.json
