# 1 GPU: the CUPTI timeline batch with one warm-up batch (as in r02n) on the final tree
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02kk
SGS_BENCH_STACK_DUMP_S=240 timeout 900 python bench.py --timeline --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02kk/bench_tl.json 2> gpurun_out/r02kk/bench_tl.err; grep -v "UserWarning\|_warn_once" gpurun_out/r02kk/bench_tl.err | tail -20; tail -c 300 gpurun_out/r02kk/bench_tl.json
