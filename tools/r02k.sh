set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02k
timeout 600 python tools/tb_sweep.py --ctx 2048 --b 1 16 64 256 --out gpurun_out/r02k/tb_default.json > gpurun_out/r02k/tb_default.log 2>&1; grep '"b"' gpurun_out/r02k/tb_default.log
SGS_FUSED_NORM=1 timeout 600 python tools/tb_sweep.py --ctx 2048 --b 1 16 64 256 --out gpurun_out/r02k/tb_fused.json > gpurun_out/r02k/tb_fused.log 2>&1; grep '"b"' gpurun_out/r02k/tb_fused.log
timeout 300 python tools/gemm_explore.py --T 16 256 --splits 4 8 > gpurun_out/r02k/gemm.log 2>&1; cat gpurun_out/r02k/gemm.log | cut -c1-200
