set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02oo
SGS_WEIGHT_LAYOUT=tiles SGS_BENCH_STACK_DUMP_S=200 timeout 500 python bench.py --timeline --steps 1 --warmup 1 --no-cpu-baseline --no-kernel-timing > gpurun_out/r02oo/bench_tl_tiles_nokt.json 2> gpurun_out/r02oo/bench_tl_tiles_nokt.err; echo rc=$?; grep -v "_warn_once" gpurun_out/r02oo/bench_tl_tiles_nokt.err | tail -8
