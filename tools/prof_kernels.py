"""Hot-path kernel launches for `ncu --set full` (each case: 2 warm-up launches + 1 profiled).

Cases (7B shapes): decode attention b=256 ctx=1536 and b=16 ctx=8192; GEMMs as the engine
launches them at decode T=256 (gate_up fused SwiGLU, o / down split-K red.add), at T=16
(qkv split-K), and prefill T=8192 (gate_up fused SwiGLU).

    python tools/prof_kernels.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_15930_b200 as sgs  # noqa: E402


def gemm_case(N, K, T, mode):
    W = torch.empty(N, K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02)
    X = torch.randn(T, K, device="cuda").bfloat16()
    if mode == 3:
        C = torch.empty(T, N // 2, dtype=torch.bfloat16, device="cuda")
    else:
        C = torch.zeros(T, N, device="cuda")
    for _ in range(3):
        sgs.op_gemm(W, X, C, mode=mode, splits=0 if mode == 1 else 1)
    torch.cuda.synchronize()


def attn_case(b, ctx):
    nq, nkv, hd, page = 28, 4, 128, 16
    npg = (ctx + page - 1) // page
    pool = torch.empty(b * npg + 64, nkv, 2, page, hd, dtype=torch.bfloat16, device="cuda").normal_()
    bt = torch.randperm(b * npg + 64, device="cuda")[:b * npg].view(b, npg).int()
    q = torch.randn(b, nq, hd, device="cuda").bfloat16()
    o = torch.empty(b, nq, hd, device="cuda", dtype=torch.bfloat16)
    c = torch.full((b,), ctx, dtype=torch.int32, device="cuda")
    for _ in range(3):
        sgs.op_decode_attention(q, pool, bt, c, o)
    torch.cuda.synchronize()


attn_case(256, 1536)
attn_case(16, 8192)
gemm_case(37888, 3584, 256, 3)
gemm_case(3584, 3584, 256, 1)
gemm_case(3584, 18944, 256, 1)
gemm_case(4608, 3584, 16, 1)
gemm_case(37888, 3584, 8192, 3)
