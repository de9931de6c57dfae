# 1 GPU: the default bench command; then a diagnostic --timeline run (stack dump if the profiler batch stalls)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02ee
timeout 1200 python bench.py > gpurun_out/r02ee/bench.json 2> gpurun_out/r02ee/bench.err; grep "\[bench" gpurun_out/r02ee/bench.err; tail -c 300 gpurun_out/r02ee/bench.json
SGS_BENCH_STACK_DUMP_S=240 timeout 900 python bench.py --timeline --warmup 3 --no-cpu-baseline > gpurun_out/r02ee/bench_tl.json 2> gpurun_out/r02ee/bench_tl.err; grep -v "UserWarning\|_warn_once" gpurun_out/r02ee/bench_tl.err | tail -40
