"""Kernel microbenchmarks (CUDA events, L2-cold by rotating buffers larger than L2).

    python tools/kbench.py attn|gemm|all [--json out.json]
Decode attention: 7B shapes (nq 28, nkv 4, hd 128), b x ctx grid, GB/s of algorithmic bytes.
GEMMs: the 7B projection shapes at decode batch sizes, GB/s of weight bytes and TFLOP/s.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_15930_b200 as sgs  # noqa: E402

PEAK_GBS = 6544.7
ARGS = None


def bench(fn, reps=20, warm=3):
    for _ in range(warm):
        fn(0)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for i, (a, b) in enumerate(evs):
        a.record()
        fn(i + 1)
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return ts[len(ts) // 2]


def attn_grid(out):
    nq, nkv, hd, page = 28, 4, 128, 16
    pool_pages = (8 << 30) // (nkv * 2 * page * hd * 2)  # 8 GiB pool >> L2
    pool = torch.empty(pool_pages, nkv, 2, page, hd, dtype=torch.bfloat16, device="cuda").normal_()
    ws = None
    for b in ARGS.b or (1, 8, 32, 64, 128, 256):
        for ctx in ARGS.ctx or (1024, 2048, 4096, 8192):
            npg = (ctx + page - 1) // page
            if b * npg > pool_pages:
                continue
            # several independent page maps so consecutive reps read disjoint memory
            bts = [torch.randperm(pool_pages, device="cuda")[:b * npg].view(b, npg).int() for _ in range(4)]
            q = torch.randn(b, nq, hd, device="cuda").bfloat16()
            o = torch.empty(b, nq, hd, device="cuda", dtype=torch.bfloat16)
            c = torch.full((b,), ctx, dtype=torch.int32, device="cuda")
            need = sgs.lib().sgs_attn_workspace_bytes(b, nq, nkv, hd, npg)
            ws = torch.empty(need, dtype=torch.uint8, device="cuda")
            ms = bench(lambda i: sgs.op_decode_attention(q, pool, bts[i % 4], c, o, workspace=ws))
            by = b * ctx * nkv * hd * 2 * 2 + b * nq * hd * 4
            r = dict(kernel="decode_attention", b=b, ctx=ctx, us=round(ms * 1e3, 1),
                     GBs=round(by / ms / 1e6, 1), frac=round(by / ms / 1e6 / PEAK_GBS, 3))
            print(json.dumps(r), flush=True)
            out.append(r)


def gemm_grid(out):
    shapes = {"qkv": (4608, 3584), "o": (3584, 3584), "gate_up": (37888, 3584), "down": (3584, 18944),
              "lm_head": (152064, 3584)}
    for name, (N, K) in shapes.items():
        if ARGS.name and name not in ARGS.name:
            continue
        nrot = max(2, int((256 << 20) // (N * K * 2)) + 1)  # rotate weights to defeat L2
        Ws = [torch.empty(N, K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02) for _ in range(nrot)]
        for T in ARGS.T or (1, 16, 64, 128, 256):
            X = torch.randn(T, K, device="cuda").bfloat16()
            C = torch.zeros(T, N, device="cuda")
            # the engine's launch: split-K with fp32 red.add where the tile grid is under one wave
            ms = bench(lambda i: sgs.op_gemm(Ws[i % nrot], X, C, mode=1, splits=0))
            # cuBLAS on the same operands (bf16 out), as the library yardstick
            ms_cb = bench(lambda i: torch.matmul(X, Ws[i % nrot].t()))
            r = dict(kernel="gemm", name=name, N=N, K=K, T=T, us=round(ms * 1e3, 1),
                     GBs=round(N * K * 2 / ms / 1e6, 1), frac_hbm=round(N * K * 2 / ms / 1e6 / PEAK_GBS, 3),
                     TFLOPs=round(2 * N * K * T / ms / 1e9, 1), cublas_us=round(ms_cb * 1e3, 1),
                     cublas_TFLOPs=round(2 * N * K * T / ms_cb / 1e9, 1))
            print(json.dumps(r), flush=True)
            out.append(r)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="?", default="all")
    ap.add_argument("--json")
    ap.add_argument("--b", type=int, nargs="*")
    ap.add_argument("--ctx", type=int, nargs="*")
    ap.add_argument("--T", type=int, nargs="*")
    ap.add_argument("--name", nargs="*")
    a = ap.parse_args()
    ARGS = a
    out = []
    if a.what in ("attn", "all"):
        attn_grid(out)
    if a.what in ("gemm", "all"):
        gemm_grid(out)
    if a.json:
        json.dump(out, open(a.json, "w"), indent=1)
