"""Decode GEMM configurations at the 7B shapes, weights streamed from HBM
(8 rotating weight copies > L2), 20 launches per configuration captured in a
CUDA graph (PDL between them): mean us per launch for each split-K factor.

    SGS_GEMM_BN_CAP=128 python tools/gemm_explore.py --T 256
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_15930_b200 as sgs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, nargs="*", default=[256])
ap.add_argument("--splits", type=int, nargs="*", default=[1, 2, 3, 4, 5, 6, 8])
ap.add_argument("--which", nargs="*", default=["qkv", "o", "down", "gate_up"])
a = ap.parse_args()
d, nq, nkv, hd, f = 3584, 28, 4, 128, 18944
shapes = dict(qkv=((nq + 2 * nkv) * hd, d, 1), o=(d, nq * hd, 1), down=(d, f, 1), gate_up=(2 * f, d, 3))
copies = 8
for T in a.T:
    for name in a.which:
        N, K, mode = shapes[name]
        Ws = [torch.empty(N, K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02) for _ in range(copies)]
        X = torch.randn(T, K, device="cuda").bfloat16()
        C = torch.empty(T, N // 2, dtype=torch.bfloat16, device="cuda") if mode == 3 else \
            torch.zeros(T, N, device="cuda")
        for s in (a.splits if mode == 1 else [1]):
            fn = lambda W: sgs.op_gemm(W, X, C, mode=mode, splits=s)
            for W in Ws:
                fn(W)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(24):
                    fn(Ws[i % copies])
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 24 * 1e3
            flops = 2.0 * N * K * T
            print(json.dumps({"op": name, "T": T, "splits": s, "bn_cap": os.environ.get("SGS_GEMM_BN_CAP", "256"),
                              "us": round(us, 2), "TFLOP/s": round(flops / us / 1e6, 1),
                              "weight_GB/s": round(2.0 * N * K / us / 1e3, 1)}), flush=True)
        del Ws
        torch.cuda.empty_cache()
