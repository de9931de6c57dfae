# 1 GPU: decode attention at small b -- isolated timing and one ncu --set full capture (b = 1 / 16, ctx 2048)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02ff
timeout 600 python tools/attn_sweep.py --b 1 4 16 --ctx 2048 8192 --out gpurun_out/r02ff/attn_small_b.json > gpurun_out/r02ff/attn_small_b.log 2>&1; grep -E '"b"' gpurun_out/r02ff/attn_small_b.log | cut -c1-200 | head
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_decode -c 2 -o gpurun_out/r02ff/attn_b1 python tools/attn_sweep.py --ncu --b 1 16 --ctx 2048 > gpurun_out/r02ff/ncu.log 2>&1; tail -3 gpurun_out/r02ff/ncu.log
