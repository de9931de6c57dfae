# 1 GPU: the CUPTI timeline batch with row-major GEMM weights (A/B against the tiled-layout stall)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02ll
SGS_WEIGHT_LAYOUT=rows SGS_BENCH_STACK_DUMP_S=240 timeout 600 python bench.py --timeline --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02ll/bench_tl_rows.json 2> gpurun_out/r02ll/bench_tl_rows.err; grep -v "_warn_once" gpurun_out/r02ll/bench_tl_rows.err | tail -12; tail -c 200 gpurun_out/r02ll/bench_tl_rows.json
