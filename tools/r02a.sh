set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
bash tools/ablate.sh gpurun_out/r02_ablate > gpurun_out/r02_ablate.log 2>&1
for T in 1 16 64 256; do python tools/decode_ops.py $T; done > gpurun_out/r02_decode_ops.txt 2>&1
cat gpurun_out/r02_decode_ops.txt
