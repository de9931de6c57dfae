# 4 GPUs: NEXT-2 tail experiment over alpha (TP = 2 pair for the longest alpha%, two DP instances for the rest)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02w
for al in 5 8 12; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2955$al tools/tp_experiment.py --mode tail --alpha-pct $al --phases A_tp2_tail --out gpurun_out/r02w/tp_tail_alpha$al.json > gpurun_out/r02w/tp_tail_alpha$al.log 2>&1
grep -E "A_tp2|B_dp4" gpurun_out/r02w/tp_tail_alpha$al.log | cut -c1-200
done
