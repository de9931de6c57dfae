# 1 GPU: decode-attention planner, fewer / longer parts at small b (min pages per part 16 / 32)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02ii
for v in 8 16 32; do
SGS_ATTN_MINPG=$v timeout 600 python tools/tb_sweep.py --ctx 2048 8192 --b 1 4 16 64 --decode-iters 8 --out gpurun_out/r02ii/tb_minpg$v.json > gpurun_out/r02ii/tb_minpg$v.log 2>&1
echo "minpg=$v"; grep '"b"' gpurun_out/r02ii/tb_minpg$v.log | cut -c1-100
done
