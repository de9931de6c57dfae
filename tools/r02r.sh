python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r02r
SGS_DEBUG_SIGNALS=1 timeout 200 python -u tools/tp_debug.py gpurun_out/r02r nccl > gpurun_out/r02r/run.log 2>&1
cat gpurun_out/r02r/run.log | tail -40
for a in $(grep -o "libsgs.so(+0x[0-9a-f]*)" gpurun_out/r02r/run.log | grep -o "0x[0-9a-f]*" | sort -u); do echo "$a $(addr2line -f -C -e paper_2504_15930_b200/libsgs.so $a | tr '\n' ' ')"; done
for f in gpurun_out/r02r/w*.log; do echo "== $f"; tail -5 $f; done
