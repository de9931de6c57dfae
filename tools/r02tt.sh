# 4 GPUs: NEXT-2 on config 3's model (14B): TP = 2 T(b), then the tail experiment with the planner's split vs four DP instances
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02tt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 tools/tp_experiment.py --mode sweep --model qwen2.5-14b --ar p2p --b 1 4 16 64 128 256 --ctx 2048 --out gpurun_out/r02tt/tp2_14b.json > gpurun_out/r02tt/tp2_14b.log 2>&1
grep '"b"' gpurun_out/r02tt/tp2_14b.log | cut -c1-120
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29592 tools/tp_experiment.py --mode tail --model qwen2.5-14b --alpha-pct -1 --dp-profile-file profiles/r02/tb_sweep_qwen2.5-14b.json --tp-profile-file gpurun_out/r02tt/tp2_14b.json --dp-pool 45000 --tp-pool 100000 --out gpurun_out/r02tt/tp_tail_14b.json > gpurun_out/r02tt/tp_tail_14b.log 2>&1
grep -E "plan|A_tp2|B_dp4" gpurun_out/r02tt/tp_tail_14b.log | cut -c1-400
