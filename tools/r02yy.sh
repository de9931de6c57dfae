# 4 GPUs: 14B tail experiment with the planner pricing context (kv) and prefill (pf) terms, profiles fitted over ctx 1K-8K
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02yy
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29597 tools/tp_experiment.py --mode tail --model qwen2.5-14b --alpha-pct -1 --phases A_tp2_tail --dp-prof 5365806,7572326,64,17339342 --tp-prof 3809976,3196036,16,16707449 --dp-kv 27342 --tp-kv 13723 --dp-pf 31000000 --tp-pf 16000000 --dp-pool 45000 --tp-pool 100000 --out gpurun_out/r02yy/tp_tail_14b_kvpf.json > gpurun_out/r02yy/tp_tail_14b_kvpf.log 2>&1
grep -E "plan|A_tp2" gpurun_out/r02yy/tp_tail_14b_kvpf.log | cut -c1-500
