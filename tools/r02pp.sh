# 1 GPU: try to reproduce the tiled-layout CUPTI stall with the decode-only timeline at long contexts
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02pp
for ctx in 8192 4096; do
SGS_WEIGHT_LAYOUT=tiles timeout 300 python -X faulthandler tools/timeline.py --b 2 8 24 --ctx $ctx --iters 32 --out gpurun_out/r02pp/timeline_tiles_ctx$ctx.json > gpurun_out/r02pp/timeline_tiles_ctx$ctx.log 2>&1; echo "ctx=$ctx rc=$?"; grep '"b"' gpurun_out/r02pp/timeline_tiles_ctx$ctx.log | cut -c1-120
done
