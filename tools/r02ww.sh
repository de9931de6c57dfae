# 1 GPU: config 5 attention sweep on the final tree (planner default 16 pages per part)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02ww
timeout 2400 python tools/attn_sweep.py --out gpurun_out/r02ww/attn_sweep_c5_final.json > gpurun_out/r02ww/attn_sweep.log 2>&1; tail -3 gpurun_out/r02ww/attn_sweep.log | cut -c1-300
