# 4 GPUs: 7B tail experiment with the planner's kv/pf terms (DP kv fitted over ctx 1K-32K; TP kv = half of it)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02zz
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29598 tools/tp_experiment.py --mode tail --model qwen2.5-7b --alpha-pct -1 --phases A_tp2_tail --dp-prof 2817210,7339081,96,2321760 --tp-prof 2079646,912767,16,6649180 --dp-kv 8418 --tp-kv 4209 --dp-pf 16500000 --tp-pf 8500000 --dp-pool 150000 --tp-pool 300000 --out gpurun_out/r02zz/tp_tail_7b_kvpf.json > gpurun_out/r02zz/tp_tail_7b_kvpf.log 2>&1
grep -E "plan|A_tp2" gpurun_out/r02zz/tp_tail_7b_kvpf.log | cut -c1-500
