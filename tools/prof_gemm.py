"""One GEMM shape, 3 launches (for ncu --set full -c 1 --launch-skip 2).

    python tools/prof_gemm.py N K T [mode] [splits]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_15930_b200 as sgs  # noqa: E402

N, K, T = (int(x) for x in sys.argv[1:4])
mode = int(sys.argv[4]) if len(sys.argv) > 4 else 1
splits = int(sys.argv[5]) if len(sys.argv) > 5 else 0
W = torch.empty(N, K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02)
X = torch.randn(T, K, device="cuda").bfloat16()
C = torch.zeros(T, N, device="cuda")
for _ in range(3):
    sgs.op_gemm(W, X, C, mode=mode, splits=splits)
torch.cuda.synchronize()
print("ok")
