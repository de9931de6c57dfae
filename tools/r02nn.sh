# 1 GPU: where the tiled-layout stall under CUPTI comes from -- decode-only timeline, then the bench batch without kernel timing
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02nn
SGS_WEIGHT_LAYOUT=tiles timeout 400 python tools/timeline.py --b 1 16 64 256 --ctx 2048 --out gpurun_out/r02nn/timeline_tiles.json > gpurun_out/r02nn/timeline_tiles.log 2>&1; echo rc=$?; grep '"b"' gpurun_out/r02nn/timeline_tiles.log | cut -c1-120
SGS_WEIGHT_LAYOUT=tiles SGS_BENCH_STACK_DUMP_S=200 timeout 500 python bench.py --timeline --steps 1 --warmup 1 --no-cpu-baseline --no-kernel-timing > gpurun_out/r02nn/bench_tl_tiles_nokt.json 2> gpurun_out/r02nn/bench_tl_tiles_nokt.err; echo rc=$?; grep -v "_warn_once" gpurun_out/r02nn/bench_tl_tiles_nokt.err | tail -8
