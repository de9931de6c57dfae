# 2 GPUs: the bulk (flag) TP exchange -- parity with it forced on, then T(b) with it from 32 rows vs never
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02xx
SGS_TP_BULK_ROWS=1 timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "tensor_parallel and p2p" > gpurun_out/r02xx/pytest_tp_bulk.log 2>&1; tail -3 gpurun_out/r02xx/pytest_tp_bulk.log
for br in 0 32 8; do
SGS_TP_BULK_ROWS=$br timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2960$br tools/tp_experiment.py --mode sweep --ar p2p --b 1 16 32 64 128 256 --out gpurun_out/r02xx/tp2_bulk$br.json > gpurun_out/r02xx/tp2_bulk$br.log 2>&1
echo "bulk_rows=$br"; grep '"b"' gpurun_out/r02xx/tp2_bulk$br.log | cut -c1-100
done
