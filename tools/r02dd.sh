# 1 GPU: the default bench command (as the driver runs it), then attention-planner variants and the stream hand-off
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02dd
timeout 1500 python bench.py > gpurun_out/r02dd/bench.json 2> gpurun_out/r02dd/bench.err; grep "\[bench" gpurun_out/r02dd/bench.err; tail -c 400 gpurun_out/r02dd/bench.json
bash tools/r02aa.sh
