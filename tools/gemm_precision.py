"""Measure the accumulation error of the tcgen05 GEMM vs fp64 and vs cuBLAS (debug aid)."""
import torch, workload
import paper_2504_15930_b200 as sgs
for (N, K, T, mode, splits) in [(4608, 3584, 16, 0, 1), (4608, 3584, 16, 1, 4), (3584, 18944, 16, 0, 1), (512, 128, 16, 0, 1)]:
    W = workload.random_bf16((N, K), 1, 0.02).cuda()
    X = workload.random_bf16((T, K), 2, 1.0).cuda()
    C = torch.zeros(T, N, device="cuda")
    sgs.op_gemm(W, X, C, mode=mode, splits=splits)
    ref = (X.double() @ W.double().T)
    cub = (X @ W.T).float()  # cuBLAS bf16 out
    cub32 = torch.matmul(X.float(), W.float().T)  # fp32 GEMM (tf32 off by default)
    scale = (X.double().abs() @ W.double().abs().T)
    e = (C.double() - ref).abs()
    e32 = (cub32.double() - ref).abs()
    print(N, K, T, mode, splits, "ours: max rel-to-result %.2e  max/|X||W| %.2e | fp32-sgemm: %.2e %.2e" % (
        (e / ref.abs().clamp_min(1e-3)).median().item(), (e / scale).max().item(),
        (e32 / ref.abs().clamp_min(1e-3)).median().item(), (e32 / scale).max().item()))
    # flip rate when rounding to bf16
    fl = (C.to(torch.bfloat16) != ref.float().to(torch.bfloat16)).float().mean().item()
    fl32 = (cub32.to(torch.bfloat16) != ref.float().to(torch.bfloat16)).float().mean().item()
    print("   bf16 flip rate ours %.4f  fp32-sgemm %.4f" % (fl, fl32))
