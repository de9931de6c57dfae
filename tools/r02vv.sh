# 4 GPUs: 14B TP = 2 T(b) at ctx 8192, then phase A with the planner on the TP side's ctx-8192 profile and real pool sizes
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02vv
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29595 tools/tp_experiment.py --mode sweep --model qwen2.5-14b --ar p2p --b 1 4 16 64 128 --ctx 4096 --out gpurun_out/r02vv/tp2_14b_ctx4096.json > gpurun_out/r02vv/tp2_14b_ctx4096.log 2>&1
grep '"b"' gpurun_out/r02vv/tp2_14b_ctx4096.log | cut -c1-120
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29596 tools/tp_experiment.py --mode tail --model qwen2.5-14b --alpha-pct -1 --phases A_tp2_tail --dp-profile-file profiles/r02/tb_sweep_qwen2.5-14b.json --dp-ctx 1024 --tp-profile-file gpurun_out/r02vv/tp2_14b_ctx4096.json --tp-ctx 4096 --dp-pool 45000 --tp-pool 100000 --out gpurun_out/r02vv/tp_tail_14b.json > gpurun_out/r02vv/tp_tail_14b.log 2>&1
grep -E "plan|A_tp2" gpurun_out/r02vv/tp_tail_14b.log | cut -c1-400
