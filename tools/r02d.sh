set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02d
timeout 600 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider -k "tiny or deterministic or weights or 7b_width or c2_scale" > gpurun_out/r02d/pytest_engine.log 2>&1; tail -3 gpurun_out/r02d/pytest_engine.log
timeout 600 python tools/timeline.py --b 1 16 64 128 256 --ctx 2048 --out gpurun_out/r02d/timeline_7b_ctx2048.json > gpurun_out/r02d/timeline.log 2>&1; tail -8 gpurun_out/r02d/timeline.log
for cap in 256 128; do SGS_GEMM_BN_CAP=$cap timeout 300 python tools/gemm_explore.py --T 16 64 128 256 > gpurun_out/r02d/gemm_explore_bn$cap.log 2>&1; done
grep -h '"T": 256' gpurun_out/r02d/gemm_explore_bn*.log | head -40
timeout 900 python tools/attn_sweep.py --out gpurun_out/r02d/attn_sweep.json > gpurun_out/r02d/attn_sweep.log 2>&1; tail -2 gpurun_out/r02d/attn_sweep.log
