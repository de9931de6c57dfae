"""Run a few hot-path kernel launches (for ncu --set full): GEMM qkv@16, gate_up@256,
lm_head@64, decode attention b=64 ctx=4096 and b=256 ctx=2048.  Each case: 2 warm + 1 profiled."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_15930_b200 as sgs  # noqa: E402

def gemm_case(N, K, T, mode):
    W = torch.empty(N, K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02)
    X = torch.randn(T, K, device="cuda").bfloat16()
    C = torch.zeros(T, N, device="cuda")
    for _ in range(3):
        sgs.op_gemm(W, X, C, mode=mode, splits=0 if mode == 1 else 1)
    torch.cuda.synchronize()

def attn_case(b, ctx):
    nq, nkv, hd, page = 28, 4, 128, 16
    npg = ctx // page
    pool = torch.empty(b * npg + 64, nkv, 2, page, hd, dtype=torch.bfloat16, device="cuda").normal_()
    bt = torch.randperm(b * npg + 64, device="cuda")[:b * npg].view(b, npg).int()
    q = torch.randn(b, nq, hd, device="cuda").bfloat16()
    o = torch.empty(b, nq, hd, device="cuda", dtype=torch.bfloat16)
    c = torch.full((b,), ctx, dtype=torch.int32, device="cuda")
    for _ in range(3):
        sgs.op_decode_attention(q, pool, bt, c, o)
    torch.cuda.synchronize()

gemm_case(4608, 3584, 16, 1)
gemm_case(37888, 3584, 256, 0)
gemm_case(152064, 3584, 64, 0)
attn_case(64, 4096)
attn_case(256, 2048)
