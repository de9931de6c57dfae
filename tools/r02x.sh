mkdir -p gpurun_out/r02x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/r02x/tma_bw tools/tma_bw.cu -lcuda && timeout 300 gpurun_out/r02x/tma_bw tiled > gpurun_out/r02x/tma_bw.txt 2>&1; grep -E "bulk1d|hbm_tiled" gpurun_out/r02x/tma_bw.txt | cut -c1-200; rm -f gpurun_out/r02x/tma_bw
