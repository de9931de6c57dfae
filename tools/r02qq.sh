set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02qq
timeout 900 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider -k "tiled_weight_layout" > gpurun_out/r02qq/pytest_tiled.log 2>&1; tail -15 gpurun_out/r02qq/pytest_tiled.log
