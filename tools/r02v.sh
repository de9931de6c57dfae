# 1 GPU: tiled vs row-major GEMM weights (TMA microbenchmark, T(b), GPU tests on the tiled layout)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02v
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/r02v/tma_bw tools/tma_bw.cu -lcuda && timeout 300 gpurun_out/r02v/tma_bw tiled > gpurun_out/r02v/tma_bw_tiled.txt 2>&1; grep -E '"box_KB": (16|32), "box_rows": 128' gpurun_out/r02v/tma_bw_tiled.txt | cut -c1-200; rm -f gpurun_out/r02v/tma_bw
for lay in rows tiles; do
SGS_WEIGHT_LAYOUT=$lay timeout 600 python tools/tb_sweep.py --ctx 2048 --b 1 16 64 256 --decode-iters 8 --out gpurun_out/r02v/tb_$lay.json > gpurun_out/r02v/tb_$lay.log 2>&1
echo "layout=$lay"; grep '"b"' gpurun_out/r02v/tb_$lay.log | cut -c1-120
done
SGS_WEIGHT_LAYOUT=tiles timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/r02v/pytest_tiles.log 2>&1; tail -5 gpurun_out/r02v/pytest_tiles.log
