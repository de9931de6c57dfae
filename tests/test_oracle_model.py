"""Pins for the oracle's numeric half (C6-C8, K11): library routines, closed
forms, invariants and known-answer vectors.  CPU only."""
import numpy as np
import pytest
import torch

import oracle
import workload


# ----------------------------------------------------------------- bf16 + weight generator
def test_bf16_round_matches_torch_rne():
    # IEEE round-to-nearest-even to bf16 == torch's float32 -> bfloat16 cast
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.standard_normal(2000) * 10 ** rng.uniform(-6, 6, 2000),
                         [1.0, 1 + 2 ** -8, 1 + 3 * 2 ** -8, -1 - 2 ** -8, 0.0, -0.0, 65504.0, 3.3895e38]])
    xs = xs.astype(np.float32)
    ref = torch.from_numpy(xs).to(torch.bfloat16).float().numpy()
    got = np.array([oracle.bf16_round(float(x)) for x in xs], np.float32)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def _splitmix(z):
    M = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def test_weight_hash_matches_python_bigint_splitmix():
    # splitmix64 (Steele et al. 2014) written with Python big ints, DESIGN.md §3
    for seed, tid, i in [(0, 0, 0), (1234, 17, 99), (2**63 + 5, 1023, 2**40 + 3)]:
        key = _splitmix(seed ^ ((tid * 0xD1B54A32D192ED03) & ((1 << 64) - 1)))
        assert oracle.weight_hash(seed, tid, i) == _splitmix((key + i) & ((1 << 64) - 1))
    # splitmix64 reference value: first output of the stream seeded with 0
    assert _splitmix(0) == 0xE220A8397B1DCDAF


def test_weight_values_distribution_and_exactness():
    w = oracle.gen_tensor(7, 42, 200_000)
    # bf16 values: low 16 bits zero
    assert (w.view(np.uint32) & 0xFFFF == 0).all()
    assert abs(w.mean()) < 3e-4 and abs(w.std() - 0.02) < 3e-4
    assert np.abs(w).max() <= 0.0347
    # value = bf16(fp32(u) * fp32(0.02*sqrt(3))) with u from the top 24 hash bits
    for i in [0, 1, 12345]:
        h = oracle.weight_hash(7, 42, i)
        u = np.float32(((h >> 40) - (1 << 23)) / 2 ** 23)
        p = np.float32(u * np.float32(0.034641016))
        assert w[i] == torch.tensor([p]).to(torch.bfloat16).float().item()
    nrm = oracle.gen_tensor(7, 43, 10_000, is_norm=True)
    assert nrm.min() >= 0.875 and nrm.max() <= 1.125


def test_checksum_matches_definition():
    w = oracle.gen_tensor(3, 5, 5000)
    bits = (w.view(np.uint32) >> 16).astype(np.uint64)
    ref = int((bits * (2 * np.arange(5000, dtype=np.uint64) + 1)).sum(dtype=np.uint64))
    assert oracle.tensor_checksum(3, 5, 5000) == ref


# ----------------------------------------------------------------- C7 attention
def _bf(shape, seed, scale=1.0):
    return workload.random_bf16(shape, seed, scale).float().numpy()


def test_attention_vs_torch_sdpa_fp64():
    for (nq, nkv, hd, ctx, seed) in [(4, 2, 32, 37, 1), (28, 4, 128, 300, 2), (40, 8, 128, 129, 3)]:
        q, K, V = _bf((nq, hd), seed), _bf((ctx, nkv, hd), seed + 10), _bf((ctx, nkv, hd), seed + 20)
        got = oracle.attention(q, K, V)
        qt = torch.from_numpy(q).double()[None, :, None, :]           # [1, nq, 1, hd]
        Kt = torch.from_numpy(K).double().permute(1, 0, 2)[None]     # [1, nkv, ctx, hd]
        Vt = torch.from_numpy(V).double().permute(1, 0, 2)[None]
        g = nq // nkv
        ref = torch.nn.functional.scaled_dot_product_attention(
            qt, Kt.repeat_interleave(g, 1), Vt.repeat_interleave(g, 1))[0, :, 0, :].numpy()
        assert np.abs(got - ref).max() < 1e-12


def test_attention_special_cases():
    nq, nkv, hd = 8, 2, 64
    q, K, V = _bf((nq, hd), 5), _bf((1, nkv, hd), 6), _bf((1, nkv, hd), 7)
    o = oracle.attention(q, K, V)  # ctx = 1 -> o = v0 exactly
    assert np.array_equal(o, np.repeat(V[0], nq // nkv, axis=0).astype(np.float64))
    ctx = 50
    K = np.repeat(_bf((1, nkv, hd), 8), ctx, axis=0)  # identical keys -> mean of V
    V = _bf((ctx, nkv, hd), 9)
    o = oracle.attention(q, K, V)
    ref = np.repeat(V.astype(np.float64).mean(0), nq // nkv, axis=0)
    assert np.abs(o - ref).max() < 1e-12
    # equal q within a group -> equal outputs; key permutation invariance
    q2 = np.repeat(q[::4], 4, axis=0)
    K = _bf((ctx, nkv, hd), 10)
    o = oracle.attention(q2, K, V)
    assert np.array_equal(o[0], o[3])
    perm = np.random.default_rng(0).permutation(ctx)
    o2 = oracle.attention(q2, K[perm], V[perm])
    assert np.abs(o - o2).max() < 1e-12


# ----------------------------------------------------------------- C6 decoder
def _hf_qwen2(shape, seed):
    from transformers import Qwen2Config, Qwen2ForCausalLM
    c = Qwen2Config(vocab_size=shape.vocab, hidden_size=shape.d_model, intermediate_size=shape.d_ffn,
                    num_hidden_layers=shape.n_layers, num_attention_heads=shape.n_q_heads,
                    num_key_value_heads=shape.n_kv_heads, rms_norm_eps=shape.rms_eps, rope_theta=shape.rope_theta,
                    tie_word_embeddings=False, max_position_embeddings=4096, head_dim=shape.head_dim,
                    attn_implementation="eager")
    m = Qwen2ForCausalLM(c).double().eval()
    d, hd, nq, nkv, f, V = shape.d_model, shape.head_dim, shape.n_q_heads, shape.n_kv_heads, shape.d_ffn, shape.vocab

    def t(tid, shp, norm=False):
        n = int(np.prod(shp))
        return torch.from_numpy(oracle.gen_tensor(seed, tid, n, norm).astype(np.float64).reshape(shp))

    sd = {"model.embed_tokens.weight": t(0, (V, d)), "lm_head.weight": t(1, (V, d)),
          "model.norm.weight": t(2, (d,), True)}
    for l in range(shape.n_layers):
        b = 16 + 16 * l
        p = f"model.layers.{l}."
        sd[p + "self_attn.q_proj.weight"] = t(b + 0, (nq * hd, d))
        sd[p + "self_attn.k_proj.weight"] = t(b + 1, (nkv * hd, d))
        sd[p + "self_attn.v_proj.weight"] = t(b + 2, (nkv * hd, d))
        sd[p + "self_attn.q_proj.bias"] = t(b + 3, (nq * hd,))
        sd[p + "self_attn.k_proj.bias"] = t(b + 4, (nkv * hd,))
        sd[p + "self_attn.v_proj.bias"] = t(b + 5, (nkv * hd,))
        sd[p + "self_attn.o_proj.weight"] = t(b + 6, (d, nq * hd))
        sd[p + "mlp.gate_proj.weight"] = t(b + 7, (f, d))
        sd[p + "mlp.up_proj.weight"] = t(b + 8, (f, d))
        sd[p + "mlp.down_proj.weight"] = t(b + 9, (d, f))
        sd[p + "input_layernorm.weight"] = t(b + 10, (d,), True)
        sd[p + "post_attention_layernorm.weight"] = t(b + 11, (d,), True)
    m.load_state_dict(sd, strict=True)
    return m


def test_decoder_vs_transformers_qwen2_fp64():
    # Library routine: HuggingFace Qwen2ForCausalLM in float64 with the same
    # generated weights.  The oracle rounds to bf16 at the materialisation
    # points (R12), HF does not, so agreement is to bf16 noise; a
    # dropped term, wrong sign/index or transposed operand gives O(1) errors.
    shape = workload.MODELS["tiny"]
    seed = 11
    toks = np.random.default_rng(3).integers(0, shape.vocab, size=40).astype(np.int32)
    got = oracle.decoder_forward(shape, seed, toks, first_row=0)
    m = _hf_qwen2(shape, seed)
    with torch.no_grad():
        ref = m(torch.from_numpy(toks.astype(np.int64))[None]).logits[0].numpy()
    err = np.abs(got - ref).max()
    assert err < 1e-2, err
    assert np.abs(ref).max() > 0.5  # logits are not trivially small
    # and the argmax agrees wherever the top-2 gap is clear
    gap = np.sort(ref, axis=1)[:, -1] - np.sort(ref, axis=1)[:, -2]
    clear = gap > 0.1
    assert (got.argmax(1)[clear] == ref.argmax(1)[clear]).all()


def test_decoder_causality_and_rows():
    shape = workload.MODELS["tiny"]
    toks = np.random.default_rng(4).integers(0, shape.vocab, size=24).astype(np.int32)
    a = oracle.decoder_forward(shape, 5, toks, first_row=0)
    t2 = toks.copy()
    t2[15:] = (t2[15:] + 7) % shape.vocab
    b = oracle.decoder_forward(shape, 5, t2, first_row=0)
    assert np.array_equal(a[:15], b[:15]) and not np.allclose(a[15:], b[15:])
    c = oracle.decoder_forward(shape, 5, toks, first_row=10)
    assert np.array_equal(a[10:], c)


# ----------------------------------------------------------------- C8 sampler
def test_philox_known_answers():
    # Random123 kat_vectors, philox4x32_10
    assert oracle.philox([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert oracle.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert oracle.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_argmax_brute_force_and_ties():
    rng = np.random.default_rng(0)
    for _ in range(50):
        x = rng.integers(-5, 5, size=300).astype(np.float32)
        assert oracle.argmax(x) == int(np.flatnonzero(x == x.max())[0])


def test_top_p_limits():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(512).astype(np.float32) * 3
    # top_p -> 0: argmax
    for s in range(20):
        assert oracle.sample_top_p(x, 1.0, 1e-9, 99, s, 0) == oracle.argmax(x)
    # top_p = 1: full categorical; empirical frequencies follow softmax
    p = np.exp(x - x.max()); p /= p.sum()
    counts = np.zeros(512)
    n = 20000
    for s in range(n):
        counts[oracle.sample_top_p(x, 1.0, 1.0, 7, s, 3)] += 1
    top = np.argsort(-p)[:5]
    assert np.all(np.abs(counts[top] / n - p[top]) < 5 * np.sqrt(p[top] / n) + 1e-3)


def test_rmsnorm_closed_forms():
    d = 64
    w = oracle.gen_tensor(1, 99, d, is_norm=True)
    # constant row c: x / sqrt(c^2 + eps) -> sign(c) * w (up to eps), exactly bf16(w) for eps = 0
    for c in (3.0, -0.25):
        y = oracle.rmsnorm(np.full((1, d), c), w, 0.0)
        assert np.array_equal(y[0], np.sign(c) * w.astype(np.float64))
    # scale invariance and library routine (torch rms_norm in fp64, then bf16)
    x = np.random.default_rng(0).standard_normal((5, d)) * 7
    y1, y2 = oracle.rmsnorm(x, w, 1e-6), oracle.rmsnorm(x * 1000, w, 1e-6 * 1e6)
    assert np.array_equal(y1, y2)
    ref = torch.nn.functional.rms_norm(torch.from_numpy(x), (d,), torch.from_numpy(w).double(), eps=1e-6)
    ref = ref.float().to(torch.bfloat16).double().numpy()
    assert (np.abs(y1 - ref) <= np.abs(ref) * 2 ** -8).all()


def test_rope_invariants():
    hd, theta = 128, 1e6
    rng = np.random.default_rng(2)
    q, k = rng.standard_normal(hd), rng.standard_normal(hd)
    assert np.array_equal(oracle.rope(q, 0, theta), q)            # position 0 = identity
    for p in (1, 37, 9000, 32767):                                 # rotation: norm preserved per pair
        r = oracle.rope(q, p, theta)
        half = hd // 2
        assert np.allclose(r[:half] ** 2 + r[half:] ** 2, q[:half] ** 2 + q[half:] ** 2, rtol=1e-12)
    # relative position: <R_m q, R_n k> depends only on m - n
    dots = [oracle.rope(q, m, theta) @ oracle.rope(k, m - 5, theta) for m in (5, 100, 7777)]
    assert np.allclose(dots, dots[0], rtol=1e-9)
    # first pair rotates by exactly pos radians (inv_freq_0 = 1)
    e = np.zeros(hd); e[0] = 1.0
    r = oracle.rope(e, 3, theta)
    assert abs(r[0] - np.cos(3)) < 1e-15 and abs(r[hd // 2] - np.sin(3)) < 1e-15


def test_decoder_layer_composes_to_forward():
    # regression pin of the layer-local entry point: layer l applied to the
    # stream after layer l-1 reproduces the full forward's dump bit for bit
    shape = workload.MODELS["tiny"]
    toks = np.random.default_rng(5).integers(0, shape.vocab, size=20)
    dump = oracle.decoder_dump(shape, 9, toks)
    for l in range(shape.n_layers):
        assert np.array_equal(oracle.decoder_layer(shape, 9, l, dump[2 * l]), dump[2 * l + 2])
    # and the head on the final stream is the forward's logits
    assert np.array_equal(oracle.decoder_head(shape, 9, dump[-1]),
                          oracle.decoder_forward(shape, 9, toks.astype(np.int32), first_row=0))


def test_top_p_nucleus_golden():
    # tests/golden/top_p_nucleus.json: equal logits make every prefix mass exact,
    # so the ">=" of "smallest prefix with mass >= top_p" (R18), the ascending-id
    # tie order and the renormalisation of u by the nucleus mass are each decided
    # by a hand-derived draw from a Random123 Philox known-answer counter.
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "top_p_nucleus.json")))
    for c in g["cases"]:
        got = oracle.sample_top_p(np.zeros(c["V"], np.float32), 1.0, c["top_p"], c["seed"], c["sample_id"],
                                  c["step"])
        assert got == c["expect"], c["name"]
