"""Decode-layer ops of the 7B shape at batch T through the C-ABI op entry points:
average time of 20 back-to-back launches (CUDA events), for the in-graph cost
picture and as an ncu target (each op also runs 3 times first).

    python tools/decode_ops.py [T] [--only name]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_15930_b200 as sgs  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 256
only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
d, nq, nkv, hd, f, page = 3584, 28, 4, 128, 18944, 16
qkvN = (nq + 2 * nkv) * hd
dev = "cuda"
W = {n: torch.empty(N, K, dtype=torch.bfloat16, device=dev).normal_(0, 0.02)
     for n, (N, K) in dict(qkv=(qkvN, d), o=(d, nq * hd), gu=(2 * f, d), down=(d, f)).items()}
x = torch.randn(T, d, device=dev).bfloat16()
h = torch.randn(T, d, device=dev)
qkv = torch.zeros(T, qkvN, device=dev)
ao = torch.randn(T, nq * hd, device=dev).bfloat16()
m = torch.empty(T, f, dtype=torch.bfloat16, device=dev)
nw = torch.ones(d, dtype=torch.bfloat16, device=dev)
bias = torch.zeros(qkvN, dtype=torch.bfloat16, device=dev)
cs = torch.from_numpy(sgs.rope_table(4096, hd, 1e6)).to(dev)
pos = torch.full((T,), 100, dtype=torch.int32, device=dev)
slot = torch.arange(T, dtype=torch.int32, device=dev)
bt = torch.arange(T * 16, dtype=torch.int32, device=dev).view(T, 16)
pool = torch.zeros(T * 16, nkv, 2, page, hd, dtype=torch.bfloat16, device=dev)
q = torch.empty(T, nq, hd, dtype=torch.bfloat16, device=dev)

ops = {
    "rmsnorm": lambda: sgs.op_rmsnorm(h, nw, x, 1e-6),
    "qkv": lambda: sgs.op_gemm(W["qkv"], x, qkv, mode=1, splits=0),
    "rope": lambda: sgs.op_rope_append(qkv, bias, pos, slot, bt, cs, q, pool, nq, nkv, hd),
    "o": lambda: sgs.op_gemm(W["o"], ao, h, mode=1, splits=0),
    "gate_up": lambda: sgs.op_gemm(W["gu"], x, m, mode=3, splits=1),
    "down": lambda: sgs.op_gemm(W["down"], m, h, mode=1, splits=0),
}
for name, fn in ops.items():
    if only and name != only:
        continue
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    # 20 launches captured in one CUDA graph (no host launch cost in the timing)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:8s} T={T}: {a.elapsed_time(b) / 20 * 1e3:8.1f} us", flush=True)
