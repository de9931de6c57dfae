"""How much do bf16 materialisation points amplify fp32-vs-fp64 differences?  (design study)
Runs a plain torch forward of the Qwen2.5-7B-shaped decoder twice (fp32 and fp64 arithmetic) with
bf16 rounding at a configurable set of points and reports max |logits_fp32 - logits_fp64|."""
import sys, time
import numpy as np, torch, oracle, workload

dev = "cuda"
shape = workload.MODELS["qwen2.5-7b"]
L = int(sys.argv[1]) if len(sys.argv) > 1 else 28
T = 12
seed = 4321
d, hd, nq, nkv, f, V = shape.d_model, shape.head_dim, shape.n_q_heads, shape.n_kv_heads, shape.d_ffn, shape.vocab
g = nq // nkv
toks = torch.from_numpy(np.random.default_rng(1).integers(0, V, size=T))

def W(tid, shp, norm=False):
    return torch.from_numpy(oracle.gen_tensor(seed, tid, int(np.prod(shp)), norm).reshape(shp)).to(dev)

t0 = time.time()
layers = []
for l in range(L):
    b = 16 + 16 * l
    layers.append(dict(wq=W(b, (nq * hd, d)), wk=W(b + 1, (nkv * hd, d)), wv=W(b + 2, (nkv * hd, d)),
                       bq=W(b + 3, (nq * hd,)), bk=W(b + 4, (nkv * hd,)), bv=W(b + 5, (nkv * hd,)),
                       wo=W(b + 6, (d, nq * hd)), wg=W(b + 7, (f, d)), wu=W(b + 8, (f, d)), wd=W(b + 9, (d, f)),
                       n1=W(b + 10, (d,), True), n2=W(b + 11, (d,), True)))
emb, lm, nf = W(0, (V, d)), W(1, (V, d)), W(2, (d,), True)
print("weights", time.time() - t0, file=sys.stderr)
pos = torch.arange(T, device=dev, dtype=torch.float64)
inv = 1e6 ** (-torch.arange(0, hd, 2, device=dev, dtype=torch.float64) / hd)
ang = pos[:, None] * inv[None]
COS, SIN = torch.cos(ang), torch.sin(ang)

def rnd(x, on):
    """on: False (keep), True (bf16), "2" (bf16 hi + bf16 lo, ~16-bit mantissa)."""
    if not on:
        return x
    if on == "h":
        return x.to(torch.float16).to(x.dtype)
    hi = x.to(torch.bfloat16).to(x.dtype)
    if on == "2":
        return hi + (x - hi).to(torch.bfloat16).to(x.dtype)
    return hi

def fwd(dt, pts):
    c = lambda t: t.to(dt)
    h = c(emb[toks.to(dev)])
    cos, sin = c(COS), c(SIN)
    def norm(x, w):
        return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-6) * c(w)
    def rope(x):
        x1, x2 = x[..., :hd // 2], x[..., hd // 2:]
        return torch.cat([x1 * cos[:, None] - x2 * sin[:, None], x2 * cos[:, None] + x1 * sin[:, None]], -1)
    mask = torch.triu(torch.full((T, T), float("-inf"), device=dev, dtype=dt), 1)
    for Ly in layers:
        x = rnd(norm(h, Ly["n1"]), pts.get("x"))
        q = rnd(rope((x @ c(Ly["wq"]).T + c(Ly["bq"])).view(T, nq, hd)), pts.get("q"))
        k = rnd(rope((x @ c(Ly["wk"]).T + c(Ly["bk"])).view(T, nkv, hd)), pts.get("kv"))
        v = rnd((x @ c(Ly["wv"]).T + c(Ly["bv"])).view(T, nkv, hd), pts.get("kv"))
        k, v = k.repeat_interleave(g, 1), v.repeat_interleave(g, 1)
        s = torch.einsum("thd,shd->hts", q, k) / hd ** 0.5 + mask
        o = rnd(torch.einsum("hts,shd->thd", torch.softmax(s, -1), v).reshape(T, nq * hd), pts.get("o"))
        h = h + o @ c(Ly["wo"]).T
        x = rnd(norm(h, Ly["n2"]), pts.get("x"))
        gg, uu = x @ c(Ly["wg"]).T, x @ c(Ly["wu"]).T
        m = rnd(gg * torch.sigmoid(gg) * uu, pts.get("m"))
        h = h + m @ c(Ly["wd"]).T
    x = rnd(norm(h, nf), pts.get("x"))
    return (x @ c(lm).T).double()

torch.backends.cuda.matmul.allow_tf32 = False
B, H, F = True, "2", "h"
for pts in [dict(x=F, q=B, kv=B, o=F, m=F), dict(x=F, q=F, kv=B, o=F, m=F), dict(x=F, q=F, kv=F, o=F, m=F),
            dict(x=H, q=B, kv=B, o=H, m=H)]:
    a, b = fwd(torch.float32, pts), fwd(torch.float64, pts)
    print(L, "layers, bf16 at", pts, "-> max |fp32 - fp64| = %.4f" % (a - b).abs().max().item(), flush=True)
