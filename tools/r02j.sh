set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02j
timeout 300 python tools/prof_kernels.py > gpurun_out/r02j/plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 2 -c 1 -o gpurun_out/r02j/attn_b256 python tools/prof_kernels.py > gpurun_out/r02j/ncu1.log 2>&1; echo rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 5 -c 1 -o gpurun_out/r02j/attn_b16_ctx8k python tools/prof_kernels.py > gpurun_out/r02j/ncu2.log 2>&1; echo rc=$?
for f in attn_b256 attn_b16_ctx8k; do ncu -i gpurun_out/r02j/$f.ncu-rep --page raw --csv > gpurun_out/r02j/$f.raw.csv 2>/dev/null; ncu -i gpurun_out/r02j/$f.ncu-rep --page details --csv > gpurun_out/r02j/$f.details.csv 2>/dev/null; done
ls -la gpurun_out/r02j
