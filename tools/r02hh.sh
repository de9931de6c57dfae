# 1 GPU: decode GEMMs with one CTA per SM (whole smem ring, several units per CTA) per mode, T(b) at ctx 2048
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02hh
for m in 0 8 2 16 30; do   # bit k = mode k: 1 split-K, 2 accumulate, 3 gate-up SwiGLU, 4 LM head argmax
SGS_GEMM_ONE_CTA=$m timeout 600 python tools/tb_sweep.py --ctx 2048 --b 1 16 64 256 --decode-iters 8 --out gpurun_out/r02hh/tb_onecta$m.json > gpurun_out/r02hh/tb_onecta$m.log 2>&1
echo "one_cta_modes=$m"; grep '"b"' gpurun_out/r02hh/tb_onecta$m.log | cut -c1-100
done
bash tools/r02ff.sh
