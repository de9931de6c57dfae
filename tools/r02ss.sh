# 1 GPU: decode attention with an L2 prefetch of the pages past the smem ring (distance 2 / 4 / 8) vs none
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02ss
for v in base pf2 pf4 pf8; do
lib=paper_2504_15930_b200/libsgs.so; [ $v != base ] && lib=abtest/libsgs_$v.so
SGS_LIB_PATH=$lib timeout 600 python tools/attn_sweep.py --b 16 64 256 1024 --ctx 2048 8192 32768 --out gpurun_out/r02ss/attn_$v.json > gpurun_out/r02ss/attn_$v.log 2>&1
echo "== $v"; grep '"b"' gpurun_out/r02ss/attn_$v.log | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['ctx'], d['b'], round(d['GB/s']), d.get('judged'))
"
SGS_LIB_PATH=$lib timeout 600 python tools/tb_sweep.py --ctx 2048 8192 --b 1 16 64 256 --decode-iters 8 --out gpurun_out/r02ss/tb_$v.json > gpurun_out/r02ss/tb_$v.log 2>&1
grep '"b"' gpurun_out/r02ss/tb_$v.log | cut -c1-80
done
