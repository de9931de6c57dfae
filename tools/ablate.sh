#!/bin/bash
# In-graph cost of each decode kernel class: T(b) with that class skipped
# (SGS_DEBUG_SKIP bit mask, engine.cu decode_body); delta vs mask 0.
out=${1:-gpurun_out/ablate}
mkdir -p $out
for m in 0 1 2 4 8 16 32 64 128 256 1023; do
  SGS_DEBUG_SKIP=$m python tools/tb_sweep.py --ctx 2048 --b 1 16 64 256 --decode-iters 8 --out $out/m$m.json > $out/m$m.log 2>&1
done
