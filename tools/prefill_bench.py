"""Prefill attention throughput: n prompts x L tokens, 7B head shape (28 q / 4 kv heads, hd 128).

    python tools/prefill_bench.py [n] [L]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_15930_b200 as sgs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
L = int(sys.argv[2]) if len(sys.argv) > 2 else 512
nq, nkv, hd = 28, 4, 128
T = n * L
q = torch.randn(T, nq, hd, device="cuda").bfloat16()
k = torch.randn(T, nkv, hd, device="cuda").bfloat16()
v = torch.randn(T, nkv, hd, device="cuda").bfloat16()
offs = torch.arange(0, T + 1, L, dtype=torch.int32, device="cuda")
out = torch.empty_like(q)
for _ in range(10):
    sgs.op_prefill_attention(q, k, v, offs, out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 50
a.record()
for _ in range(reps):
    sgs.op_prefill_attention(q, k, v, offs, out)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
flops = n * nq * (L * (L + 1) / 2) * hd * 4  # causal QK^T + PV
print(f"prefill attention n={n} L={L}: {ms * 1e3:.1f} us  {flops / ms / 1e9:.1f} TFLOP/s (causal flops)")
