# 4 GPUs: NEXT-2 on 32B -- TP = 2 T(b) at ctx 2048 / 8192, kv/pf planner, tail experiment vs four DP instances
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02ab
for ctx in 2048 8192; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2962$((ctx / 2048)) tools/tp_experiment.py --mode sweep --model qwen2.5-32b --ar p2p --b 1 4 16 64 128 --ctx $ctx --out gpurun_out/r02ab/tp2_32b_ctx$ctx.json > gpurun_out/r02ab/tp2_32b_ctx$ctx.log 2>&1
grep '"b"' gpurun_out/r02ab/tp2_32b_ctx$ctx.log | cut -c1-100
done
DP=$(python tools/fit_kv_profile.py profiles/r02/tb_sweep_qwen2.5-32b.json --bmax 256)
TP=$(python tools/fit_kv_profile.py gpurun_out/r02ab/tp2_32b_ctx2048.json gpurun_out/r02ab/tp2_32b_ctx8192.json --exchange p2p)
echo "dp $DP"; echo "tp $TP"
DPP=$(echo $DP | python -c "import json,sys; d=json.load(sys.stdin); print(','.join(map(str,d['profile'])), d['kv_ps'])")
TPP=$(echo $TP | python -c "import json,sys; d=json.load(sys.stdin); print(','.join(map(str,d['profile'])), d['kv_ps'])")
set -- $DPP $TPP
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29629 tools/tp_experiment.py --mode tail --model qwen2.5-32b --alpha-pct -1 --dp-prof $1 --dp-kv $2 --tp-prof $3 --tp-kv $4 --dp-pf 75000000 --tp-pf 38000000 --dp-pool 25000 --tp-pool 65000 --out gpurun_out/r02ab/tp_tail_32b_kvpf.json > gpurun_out/r02ab/tp_tail_32b_kvpf.log 2>&1
grep -E "plan|A_tp2|B_dp4" gpurun_out/r02ab/tp_tail_32b_kvpf.log | cut -c1-500
