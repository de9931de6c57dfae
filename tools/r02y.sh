# 4 GPUs: NEXT-2 tail experiment with the planner's split (sgs_tp_tail_plan) and alpha 12%
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02y
for al in -1 12; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + ${al#-})) tools/tp_experiment.py --mode tail --alpha-pct $al --phases A_tp2_tail --out gpurun_out/r02y/tp_tail_alpha$al.json > gpurun_out/r02y/tp_tail_alpha$al.log 2>&1
grep -E "plan|A_tp2" gpurun_out/r02y/tp_tail_alpha$al.log | cut -c1-300
done
