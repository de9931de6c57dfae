set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02i
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_kernels.py -q -p no:cacheprovider -x > gpurun_out/r02i/pytest.log 2>&1; tail -3 gpurun_out/r02i/pytest.log
for nf in 0 1; do SGS_NO_FUSED_NORM=$nf timeout 600 python tools/timeline.py --b 1 16 64 128 256 --ctx 2048 --out gpurun_out/r02i/timeline_nf$nf.json > gpurun_out/r02i/timeline_nf$nf.log 2>&1; tail -5 gpurun_out/r02i/timeline_nf$nf.log; done
for nf in 0 1; do SGS_NO_FUSED_NORM=$nf timeout 900 python tools/tb_sweep.py --ctx 2048 --b 1 16 64 256 --out gpurun_out/r02i/tb_nf$nf.json > gpurun_out/r02i/tb_nf$nf.log 2>&1; grep '"b"' gpurun_out/r02i/tb_nf$nf.log; done
