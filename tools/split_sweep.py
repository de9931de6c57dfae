"""Split-K sweep for the decode GEMM shapes (CUDA-graph timing of 20 launches).

    python tools/split_sweep.py [T ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_15930_b200 as sgs  # noqa: E402

Ts = [int(x) for x in sys.argv[1:]] or [64, 128, 256]
shapes = {"qkv": (4608, 3584), "o": (3584, 3584), "down": (3584, 18944), "gate_up": (37888, 3584)}
for T in Ts:
    for name, (N, K) in shapes.items():
        W = torch.empty(N, K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02)
        X = torch.randn(T, K, device="cuda").bfloat16()
        C = torch.zeros(T, N, device="cuda")
        res = []
        for s in (1, 2, 3, 4, 5, 6, 8):
            fn = lambda: sgs.op_gemm(W, X, C, mode=1, splits=s)
            try:
                fn()
            except Exception:
                continue
            torch.cuda.synchronize()
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
            res.append((s, a.elapsed_time(b) / 20 * 1e3))
        print(f"T={T:4d} {name:8s} " + "  ".join(f"s{s}:{us:6.1f}" for s, us in res), flush=True)
