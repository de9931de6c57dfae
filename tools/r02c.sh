set -x
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02c
timeout 900 python tools/attn_sweep.py --out gpurun_out/r02c/attn_sweep.json > gpurun_out/r02c/attn_sweep.log 2>&1
tail -3 gpurun_out/r02c/attn_sweep.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:attn_decode --csv --log-file gpurun_out/r02c/attn_sweep_ncu.csv python tools/attn_sweep.py --ncu --out gpurun_out/r02c/attn_sweep_ncu.json > gpurun_out/r02c/attn_sweep_ncu.log 2>&1
echo ncu_rc=$?
for m in qwen2.5-7b; do timeout 1200 python tools/tb_sweep.py --model $m --ctx 1024 2048 4096 8192 16384 32768 --out gpurun_out/r02c/tb_sweep_$m.json > gpurun_out/r02c/tb_$m.log 2>&1; tail -2 gpurun_out/r02c/tb_$m.log; done
for m in qwen2.5-14b qwen2.5-32b; do timeout 900 python tools/tb_sweep.py --model $m --ctx 1024 2048 4096 8192 --b 1 2 4 8 16 32 64 96 128 160 192 224 256 320 384 512 --out gpurun_out/r02c/tb_sweep_$m.json > gpurun_out/r02c/tb_$m.log 2>&1; tail -2 gpurun_out/r02c/tb_$m.log; done
timeout 600 python -m pytest tests/test_gpu_engine.py -q -k "c2_scale or deterministic" -p no:cacheprovider > gpurun_out/r02c/pytest_c2.log 2>&1; tail -3 gpurun_out/r02c/pytest_c2.log
for w in "20000 b256" "1700000 tail"; do set -- $w
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $1 -c 460 --csv --log-file gpurun_out/r02c/ncu_window_$2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-kernel-timing > gpurun_out/r02c/ncu_window_$2.log 2>&1
echo ncu_$2 rc=$?
python tools/ncu_shares.py gpurun_out/r02c/ncu_window_$2.csv --what "c2 bench, launches $1..+460" --out gpurun_out/r02c/ncu_window_$2.json | head -12
done
