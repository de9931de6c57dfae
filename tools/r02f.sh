set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02f
timeout 900 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider -k "tiny or deterministic or weights or 7b_width or c2_scale" > gpurun_out/r02f/pytest_engine.log 2>&1; tail -3 gpurun_out/r02f/pytest_engine.log
timeout 600 python tools/timeline.py --b 1 16 64 128 256 --ctx 2048 --out gpurun_out/r02f/timeline_7b_ctx2048.json > gpurun_out/r02f/timeline.log 2>&1; tail -6 gpurun_out/r02f/timeline.log
for cfg in "296 8" "592 8" "1184 8" "2368 8" "1184 4"; do set -- $cfg
SGS_ATTN_SLOTS=$1 SGS_ATTN_MINPG=$2 timeout 300 python tools/attn_sweep.py --b 8 16 32 64 128 256 --ctx 1024 8192 32768 --out gpurun_out/r02f/attn_s$1_m$2.json > gpurun_out/r02f/attn_s$1_m$2.log 2>&1
tail -1 gpurun_out/r02f/attn_s$1_m$2.log
done
