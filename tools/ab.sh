#!/bin/bash
# A/B decode timing on one box: alternate two in-tree builds of libsgs.so
# (SGS_LIB_PATH) through the same T(b) sweep, 3 rounds, so box-to-box
# variance does not enter the comparison.
A=${A:-abtest/libsgs_A.so}
B=${B:-paper_2504_15930_b200/libsgs.so}
out=${1:-gpurun_out/ab}
shift
args=${@:---ctx 2048 --b 1 16 64 256 --decode-iters 8}
mkdir -p $out
for r in 1 2 3 4; do
  order="A B"; [ $((r % 2)) = 0 ] && order="B A"  # ABBA: cancels thermal / clock drift
  for v in $order; do
    lib=$A; [ $v = B ] && lib=$B
    SGS_LIB_PATH=$lib python tools/tb_sweep.py $args --out $out/${v}$r.json > $out/${v}$r.log 2>&1
  done
done
python - "$out" <<'PY'
import json, sys, glob, collections
out = sys.argv[1]
res = collections.defaultdict(lambda: collections.defaultdict(list))
for f in sorted(glob.glob(out + "/[AB][0-9].json")):
    v = f.split("/")[-1][0]
    for p in json.load(open(f))["points"]:
        res[(p["ctx"], p["b"])][v].append(p["T_us"])
for k, d in sorted(res.items()):
    a, b = sorted(d["A"]), sorted(d["B"])
    ma, mb = a[len(a) // 2], b[len(b) // 2]
    print("ctx %5d b %4d  A %8.0f  B %8.0f  B/A %.3f   (A %s | B %s)" % (k[0], k[1], ma, mb, mb / ma, a, b))
PY
