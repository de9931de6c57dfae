"""Op-level check of the MLP chain (gate/up GEMM -> SiLU*mul -> down GEMM) vs fp64 (debug aid)."""
import numpy as np, torch, oracle, workload
import paper_2504_15930_b200 as sgs
T, d, f = 24, 3584, 512
x = workload.random_bf16((T, d), 5, 1.0)
Wg = torch.from_numpy(oracle.gen_tensor(1, 7, f * d).reshape(f, d)).to(torch.bfloat16)
Wu = torch.from_numpy(oracle.gen_tensor(1, 8, f * d).reshape(f, d)).to(torch.bfloat16)
Wgu = torch.cat([Wg, Wu]).cuda()
for splits in (1, 14):
    gu = torch.zeros(T, 2 * f, device="cuda")
    sgs.op_gemm(Wgu, x.cuda(), gu, mode=1 if splits > 1 else 0, splits=splits)
    torch.cuda.synchronize()
    ref = x.double() @ torch.cat([Wg, Wu]).double().T
    e = (gu.cpu().double() - ref).abs()
    print("splits", splits, "gu max abs err %.3e  max|gu| %.3f  rel-to-|x||w| %.3e" % (
        e.max().item(), ref.abs().max().item(), (e / (x.double().abs() @ Wgu.cpu().double().abs().T)).max().item()))
    g, u = ref[:, :f], ref[:, f:]
    m_ref = (g / (1 + torch.exp(-g)) * u).float().to(torch.bfloat16).double()
    gg, uu = gu.cpu().double()[:, :f], gu.cpu().double()[:, f:]
    m_gpu = (gg / (1 + torch.exp(-gg)) * uu).float().to(torch.bfloat16).double()
    print("   m flips %.4f" % (m_ref != m_gpu).double().mean().item())
# GPU SiLU*mul kernel vs fp64 on the same gu
gu = torch.zeros(T, 2 * f, device="cuda")
sgs.op_gemm(Wgu, x.cuda(), gu, mode=1, splits=14)
m = torch.empty(T, f, dtype=torch.bfloat16, device="cuda")
sgs.op_silu_mul(gu, m)
torch.cuda.synchronize()
gg, uu = gu.cpu().double()[:, :f], gu.cpu().double()[:, f:]
m_ref = (gg / (1 + torch.exp(-gg)) * uu).float().to(torch.bfloat16)
print("silu kernel flips %.4f  max abs diff %.3e" % ((m.cpu() != m_ref).double().mean().item(),
      (m.cpu().double() - m_ref.double()).abs().max().item()))
# down GEMM accumulate (mode 1 split 2, mode 2)
Wd = torch.from_numpy(oracle.gen_tensor(1, 9, d * f).reshape(d, f)).to(torch.bfloat16).cuda()
for mode, sp in ((1, 2), (2, 1), (0, 1)):
    h0 = torch.randn(T, d, device="cuda")
    h = h0.clone()
    sgs.op_gemm(Wd, m, h, mode=mode, splits=sp)
    torch.cuda.synchronize()
    ref = m.cpu().double() @ Wd.cpu().double().T + (h0.cpu().double() if mode else 0)
    print("down mode", mode, "max abs err %.3e" % (h.cpu().double() - ref).abs().max().item())
