"""End-to-end GPU parity: schedules bit-exact and teacher-forced logits within
2e-2 max-abs (north_star) of the oracle decoder, through the C-ABI."""
import numpy as np
import pytest
import torch

import oracle
import workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sgs():
    assert torch.cuda.is_available(), "the -m gpu tests need a B200"
    import paper_2504_15930_b200 as m
    m.lib()
    return m


def _weight_ids(shape):
    ids = [(0, shape.vocab * shape.d_model, 0), (1, shape.vocab * shape.d_model, 0), (2, shape.d_model, 1)]
    d, hd, nq, nkv, f = shape.d_model, shape.head_dim, shape.n_q_heads, shape.n_kv_heads, shape.d_ffn
    sizes = [nq * hd * d, nkv * hd * d, nkv * hd * d, nq * hd, nkv * hd, nkv * hd, d * nq * hd, f * d, f * d, d * f,
             d, d]
    for l in range(shape.n_layers):
        for k, n in enumerate(sizes):
            ids.append((16 + 16 * l + k, n, 1 if k >= 10 else 0))
    return ids


def test_hash_init_bit_identical_to_oracle(sgs):
    shape = workload.MODELS["tiny"]
    inst = sgs.Instance(shape, 16, 512, device=0, n_pages=64, weight_seed=77)
    for tid, n, norm in _weight_ids(shape):
        assert inst.checksum(tid) == oracle.tensor_checksum(77, tid, n, bool(norm)), tid
    inst.load_weights_seed(78)
    assert inst.checksum(17) == oracle.tensor_checksum(78, 17, shape.n_kv_heads * shape.head_dim * shape.d_model)


def _run_collect(inst, tr, batches=None):
    """Run to completion; collect logits rows per (sample id, token index)."""
    rows = {}
    comps = []
    inst.submit_trace(tr)
    while True:
        q, a = inst.pending()
        if q == 0 and a == 0:
            break
        comps += inst.step()
        lg, ids, tk = inst.last_logits()
        for r in range(len(ids)):
            rows[(int(ids[r]), int(tk[r]))] = lg[r].copy()
    return comps, rows


def _check_teacher_forced(shape, seed, tr, comps, rows, sample_ids, tol=2e-2, greedy=True):
    toks = {c["id"]: c["tokens"] for c in comps}
    worst = 0.0
    for sid in sample_ids:
        i = int(np.flatnonzero(tr.ids == sid)[0])
        prompt = tr.tokens[tr.offsets[i]:tr.offsets[i + 1]]
        gen = toks[sid]
        d = len(gen)
        seq = np.concatenate([prompt, gen[:-1]]).astype(np.int32)
        ref = oracle.decoder_forward(shape, seed, seq, first_row=len(prompt) - 1)  # [d, V]
        got = np.stack([rows[(sid, j)] for j in range(d)])
        err = np.abs(got - ref).max()
        worst = max(worst, err)
        assert err <= tol, (sid, err)
        if not greedy:
            continue
        # the emitted token is the argmax of the emitted logits (greedy, lowest index)
        assert np.array_equal(got.argmax(1), gen)
        # and the oracle agrees wherever its top-2 gap is clear of the tolerance
        srt = np.sort(ref, 1)
        clear = (srt[:, -1] - srt[:, -2]) > 2 * tol
        assert np.array_equal(ref.argmax(1)[clear], gen[clear])
    return worst


def test_tiny_config1_end_to_end(sgs):
    c = workload.CONFIGS["c1_tiny"]
    shape = workload.MODELS["tiny"]
    tr = workload.config_trace(c)
    pool = 400
    inst = sgs.Instance(shape, c.max_batch, 16 + 256, device=0, n_pages=pool, weight_seed=1234,
                        flags=sgs.sgs.F_KEEP_LOGITS, max_prefill_tokens=64)
    comps, rows = _run_collect(inst, tr)
    # schedule, block tables and emitted order bit-exact vs the oracle simulator
    o = oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, c.max_batch, c.page_size, pool)
    assert np.array_equal(inst.trace(0), o["iter_blob"])
    assert np.array_equal(inst.trace(1), o["sample_blob"])
    assert [x["id"] for x in comps] == [i for it in o["iters"] for i in it["completed"]]
    # teacher-forced logits for every sample, every position
    worst = _check_teacher_forced(shape, 1234, tr, comps, rows, tr.ids.tolist())
    print("tiny worst max-abs logits error", worst)


def test_graphs_and_concurrent_prefill_match_eager(sgs):
    # equal-length prompts: refill prefill chunks repeat their metadata shape, so
    # their CUDA graphs are captured and replayed, and the prefill stream runs
    # concurrently with the decode graph; the results must equal the eager,
    # sequential program's up to the fp32 summation order of split-K red.add
    # (R21), which a bf16 rounding boundary can amplify to ~1e-3 in
    # a logit: same tokens, logits within 1e-2 (the oracle bound is 2e-2)
    shape = workload.MODELS["tiny"]
    tr = workload.make_trace(40, 16, 24, 1.0, 120, shape.vocab, seed=31)
    runs = []
    for flags in (sgs.sgs.F_KEEP_LOGITS, sgs.sgs.F_KEEP_LOGITS | sgs.sgs.F_NO_GRAPHS):
        inst = sgs.Instance(shape, 6, 200, device=0, n_pages=120, weight_seed=5, flags=flags, max_prefill_tokens=64)
        comps, rows = _run_collect(inst, tr)
        runs.append(({c["id"]: list(c["tokens"]) for c in comps}, rows))
        inst.close()
    same = [i for i in runs[0][0] if runs[0][0][i] == runs[1][0][i]]
    assert len(same) >= 0.95 * len(runs[0][0]), (len(same), len(runs[0][0]))
    for k in runs[0][1]:
        if k[0] in same:
            assert np.abs(runs[0][1][k] - runs[1][1][k]).max() <= 1e-2, k


def test_tiny_ragged_prompts_multi_chunk_prefill(sgs):
    shape = workload.MODELS["tiny"]
    tr = workload.make_trace(24, 40, 20, 1.0, 120, shape.vocab, seed=21, prompt_len_jitter=39)
    inst = sgs.Instance(shape, 6, 200, device=0, n_pages=120, weight_seed=9, flags=sgs.sgs.F_KEEP_LOGITS,
                        max_prefill_tokens=96)
    comps, rows = _run_collect(inst, tr)
    o = oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, 6, 16, 120)
    assert np.array_equal(inst.trace(0), o["iter_blob"])
    _check_teacher_forced(shape, 9, tr, comps, rows, tr.ids.tolist())


def test_tiny_top_p_sampling_end_to_end(sgs):
    """Nucleus sampling inside the engine (sgs_engine_cfg.sampling = 1): the
    logits stay within 2e-2 of the oracle under teacher forcing, and each emitted
    token is the oracle sampler's draw from the engine's own logits row with the
    same Philox counter (sample id, token index) — the draw is compared on the
    same fp32 logits so only the sampler is under test."""
    c = workload.CONFIGS["c1_tiny"]
    shape = workload.MODELS["tiny"]
    tr = workload.config_trace(c)
    seed = 99
    inst = sgs.Instance(shape, c.max_batch, 16 + 256, device=0, n_pages=400, weight_seed=1234,
                        flags=sgs.sgs.F_KEEP_LOGITS, max_prefill_tokens=64, sample_seed=seed,
                        top_p=0.9, temperature=1.0)
    comps, rows = _run_collect(inst, tr)
    _check_teacher_forced(shape, 1234, tr, comps, rows, tr.ids.tolist()[:8], greedy=False)
    toks = {x["id"]: x["tokens"] for x in comps}
    agree = total = greedy_same = 0
    for sid, gen in toks.items():
        for j, t in enumerate(gen):
            lg = rows[(sid, j)]
            agree += oracle.sample_top_p(lg, 1.0, 0.9, seed, sid, j) == int(t)
            greedy_same += int(lg.argmax()) == int(t)
            total += 1
    assert agree >= 0.99 * total, (agree, total)
    assert greedy_same < total  # it really samples
    # same seed: the same draws.  Split-K GEMMs reduce with fp32 atomics, so the
    # logits are reproducible only up to summation order (R21) and a
    # draw that lands within rounding of a nucleus boundary may flip; require
    # almost every sample to repeat exactly.
    inst2 = sgs.Instance(shape, c.max_batch, 16 + 256, device=0, n_pages=400, weight_seed=1234,
                         max_prefill_tokens=64, sample_seed=seed, top_p=0.9, temperature=1.0)
    inst2.submit_trace(tr)
    comps2 = inst2.run()
    again = {x["id"]: list(x["tokens"]) for x in comps2}
    same = sum(again[k] == list(v) for k, v in toks.items())
    assert same >= 0.9 * len(toks), (same, len(toks))


# Teacher-forced logits tolerance for the 28-layer 7B shape (R17):
# any fp32 implementation that materialises bf16 activations differs from the
# fp64 oracle by ~0.12 max-abs at this depth (tools/flip_study.py: torch fp32 vs
# fp64, same rounding points), so 2e-2 is only attainable for shallow models;
# the bound here is 2x that measured floor.  2e-2 holds for the tiny config and
# the 1-layer 7B-width model below.
TOL_7B_28L = 0.25


def test_7b_width_one_layer_within_2e2(sgs):
    import dataclasses
    shape = dataclasses.replace(workload.MODELS["qwen2.5-7b"], n_layers=1)
    tr = workload.make_trace(4, 20, 6, 0.5, 10, shape.vocab, seed=2, prompt_len_jitter=12)
    inst = sgs.Instance(shape, 2, 64, device=0, n_pages=64, weight_seed=4321, flags=sgs.sgs.F_KEEP_LOGITS)
    comps, rows = _run_collect(inst, tr)
    _check_teacher_forced(shape, 4321, tr, comps, rows, tr.ids[:2].tolist(), tol=2e-2)


def test_7b_shape_spot_parity(sgs):
    # full 7B layer shapes (28 layers, d 3584, GQA 28/4, V 152064): a few samples
    # with short prompts, checked position by position against the oracle decoder
    shape = workload.MODELS["qwen2.5-7b"]
    tr = workload.make_trace(6, 20, 6, 0.5, 10, shape.vocab, seed=2, prompt_len_jitter=12)
    inst = sgs.Instance(shape, 4, 64, device=0, n_pages=64, weight_seed=4321, flags=sgs.sgs.F_KEEP_LOGITS)
    comps, rows = _run_collect(inst, tr)
    o = oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, 4, 16, 64)
    assert np.array_equal(inst.trace(0), o["iter_blob"])
    worst = _check_teacher_forced(shape, 4321, tr, comps, rows, tr.ids[:2].tolist(), tol=TOL_7B_28L)
    print("7B worst max-abs logits error", worst)


@pytest.mark.parametrize("model", ["qwen2.5-7b", "qwen2.5-14b", "qwen2.5-32b"])
def test_layer_local_parity_full_shapes(sgs, model):
    # Layer-local parity: the CUDA path's decoder layer l applied to
    # a residual stream supplied by the test equals the oracle's layer l on the
    # same input to within half a bf16 ulp of the largest element (the depth
    # chaos of the end-to-end comparison does not enter); sampled layers of the
    # full 7B/14B/32B shapes, T = 40 positions (spans the 16-token pages and a
    # partial 64-query prefill block).
    shape = workload.MODELS[model]
    inst = sgs.Instance(shape, 4, 128, device=0, n_pages=64, weight_seed=77)
    rng = np.random.default_rng(0)
    T = 40
    for layer in sorted({0, shape.n_layers // 2, shape.n_layers - 1}):
        h_in = (rng.standard_normal((T, shape.d_model)) * (1.0 + layer / 8)).astype(np.float32)
        got = inst.debug_layer(layer, h_in).astype(np.float64)
        ref = oracle.decoder_layer(shape, 77, layer, h_in.astype(np.float64))
        err = np.abs(got - ref).max()
        scale = np.abs(ref).max()
        print(model, "layer", layer, "max err", err, "max |h|", scale)
        assert err <= scale * 2 ** -8, (model, layer, err, scale)
    inst.close()
    del inst
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ boundary: weights through the C-ABI
def _oracle_weights(shape, seed):
    """The canonical weight list (sgs_weight_tensors order) generated by the oracle, as bf16 CPU tensors."""
    import paper_2504_15930_b200 as m
    out = []
    for tid, rows, cols in m.weight_tensors(shape):
        norm = tid == 2 or (tid >= 16 and (tid - 16) % 16 >= 10)
        w = oracle.gen_tensor(seed, tid, rows * cols, norm)
        out.append(torch.from_numpy(w).to(torch.bfloat16).reshape(rows, cols) if cols > 1 else
                   torch.from_numpy(w).to(torch.bfloat16))
    return out


def test_weights_through_abi(sgs):
    # SGS update(weights): the caller's tensors (host or device) are copied
    # into the library's layout; checksums equal the oracle's per tensor, and the
    # generated samples equal those of the same weights hash-initialised on the device
    shape = workload.MODELS["tiny"]
    w = _oracle_weights(shape, 321)
    inst = sgs.Instance(shape, 8, 200, device=0, n_pages=64, weights=w, flags=sgs.sgs.F_DETERMINISTIC)
    for tid, n, norm in _weight_ids(shape):
        assert inst.checksum(tid) == oracle.tensor_checksum(321, tid, n, bool(norm)), tid
    ref = sgs.Instance(shape, 8, 200, device=0, n_pages=64, weight_seed=321, flags=sgs.sgs.F_DETERMINISTIC)
    tr = workload.make_trace(12, 16, 10, 1.0, 40, shape.vocab, seed=8)
    inst.submit_trace(tr)
    ref.submit_trace(tr)
    a = {c["id"]: list(c["tokens"]) for c in inst.run()}
    b = {c["id"]: list(c["tokens"]) for c in ref.run()}
    assert a == b
    # the root's new weights from device memory (world size 1: the copy alone), version + 1
    w2 = [t.cuda() for t in _oracle_weights(shape, 322)]
    inst.update_weights(0, weights=w2)
    assert inst.weight_version() == 1
    for tid, n, norm in _weight_ids(shape):
        assert inst.checksum(tid) == oracle.tensor_checksum(322, tid, n, bool(norm)), tid
    with pytest.raises(sgs.SgsError) as e:  # wrong tensor count
        inst.update_weights(0, weights=w2[:-1])
    assert e.value.code == -1


def test_async_stage_and_begin_right_after_commit(sgs):
    # stage / begin may follow a commit at once (the side stream waits
    # for the commit's shadow -> active copy); trainer path via sgs_stage_weights
    shape = workload.MODELS["tiny"]
    inst = sgs.Instance(shape, 8, 200, device=0, n_pages=64, weight_seed=1, flags=sgs.sgs.F_SHADOW_WEIGHTS)
    inst.stage_weights_seed(2)
    inst.update_weights_begin(0)
    inst.update_weights_commit()
    inst.stage_weights(_oracle_weights(shape, 3))  # immediately after the commit
    inst.update_weights_begin(0)
    inst.update_weights_commit()
    assert inst.weight_version() == 2
    for tid, n, norm in _weight_ids(shape):
        assert inst.checksum(tid) == oracle.tensor_checksum(3, tid, n, bool(norm)), tid


def test_gqa_group_above_8_unsupported_at_init(sgs):
    import dataclasses
    shape = dataclasses.replace(workload.MODELS["tiny"], n_q_heads=18, n_kv_heads=2)  # g = 9
    with pytest.raises(sgs.SgsError) as e:
        sgs.Instance(shape, 4, 64, device=0, n_pages=16)
    assert e.value.code == -7


# ------------------------------------------------------------------ production path == test path, bitwise
def test_deterministic_paths_bitwise_equal(sgs):
    # SGS_F_DETERMINISTIC removes split-K (R21), so the pipelined graph
    # path the bench runs, the logits-keeping unpipelined path and the eager
    # sequential path must give bitwise identical tokens, schedules and
    # completion records -- including a completion cap smaller than the
    # completions of one iteration (leftovers served before the next iteration)
    shape = workload.MODELS["tiny"]
    tr = workload.make_trace(48, 16, 20, 1.0, 100, shape.vocab, seed=41)
    D = sgs.sgs.F_DETERMINISTIC
    runs = {}
    for name, flags, cap in (("pipelined", 0, 2), ("keep", sgs.sgs.F_KEEP_LOGITS, None),
                             ("eager", sgs.sgs.F_KEEP_LOGITS | sgs.sgs.F_NO_GRAPHS, None)):
        inst = sgs.Instance(shape, 6, 200, device=0, n_pages=120, weight_seed=5, flags=flags | D,
                            max_prefill_tokens=64)
        inst.submit_trace(tr)
        comps = []
        while True:
            q, a = inst.pending()
            c = inst.step(cap)
            comps += c
            if not c and q == 0 and a == 0:
                break
        runs[name] = (inst.trace(0), inst.trace(1),
                      [(c["id"], c["admit_iter"], c["finish_iter"], c["slot"], tuple(c["tokens"])) for c in comps])
        inst.close()
    o = oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, 6, 16, 120)
    for name, (t0, t1, recs) in runs.items():
        assert np.array_equal(t0, o["iter_blob"]), name
        assert np.array_equal(t1, o["sample_blob"]), name
        assert recs == runs["keep"][2], name


@pytest.mark.parametrize("model", ["tiny", "qwen2.5-7b"])
def test_tiled_weight_layout_bitwise_equal(sgs, model, monkeypatch):
    # SGS_WEIGHT_LAYOUT=tiles changes only where the GEMM weights
    # live and how TMA fetches them, not the arithmetic: with split-K off
    # (SGS_F_DETERMINISTIC) the kept logits, tokens and schedules equal the
    # row-major run bit for bit; the weight checksums (canonical order) agree
    shape = workload.MODELS[model]
    n, P, med, cap = (24, 16, 12, 40) if model == "tiny" else (4, 24, 6, 8)
    tr = workload.make_trace(n, P, med, 1.0, cap, shape.vocab, seed=43)
    runs = {}
    for lay in ("rows", "tiles"):
        monkeypatch.setenv("SGS_WEIGHT_LAYOUT", lay)
        inst = sgs.Instance(shape, 4, P + cap + 8, device=0, n_pages=64, weight_seed=17,
                            flags=sgs.sgs.F_KEEP_LOGITS | sgs.sgs.F_DETERMINISTIC)
        sums = [inst.checksum(t) for t in (1, 16, 17, 22, 23, 24, 25)]
        inst.submit_trace(tr)
        rows, comps = [], []
        while True:
            q, a = inst.pending()
            if q == 0 and a == 0:
                break
            comps += inst.step()
            lg, ids, tk = inst.last_logits()
            rows.append(lg.copy())
        runs[lay] = (sums, inst.trace(0), sorted((c["id"], tuple(c["tokens"])) for c in comps), rows)
        inst.close()
    (s0, t0, c0, r0), (s1, t1, c1, r1) = runs["rows"], runs["tiles"]
    assert s0 == s1
    assert np.array_equal(t0, t1) and c0 == c1
    assert len(r0) == len(r1) and all(np.array_equal(a, b) for a, b in zip(r0, r1))


# ------------------------------------------------------------------ chained layer-local parity, every layer
@pytest.mark.parametrize("model", ["qwen2.5-7b", "qwen2.5-14b", "qwen2.5-32b"])
def test_chained_layer_parity_every_layer(sgs, model):
    # the oracle's stream after layer l-1 is fed to the CUDA
    # path's layer l for EVERY layer of the 7B/14B/32B shapes; each layer must
    # agree within half a bf16 ulp of the largest element (the depth chaos of an
    # end-to-end comparison does not enter), and the CUDA final norm + LM head
    # on the oracle's final stream within 2e-2 (north_star).  T = 17 positions
    # span a page boundary; the input is the oracle's embedding of real tokens.
    shape = workload.MODELS[model]
    seed = 77
    inst = sgs.Instance(shape, 4, 64, device=0, n_pages=32, weight_seed=seed)
    toks = workload.make_trace(1, 17, 1, 0.0, 1, shape.vocab, seed=5).tokens
    import dataclasses
    h = oracle.decoder_dump(dataclasses.replace(shape, n_layers=0), seed, toks)[0]  # the embedding rows
    worst = 0.0
    for layer in range(shape.n_layers):
        ref = oracle.decoder_layer(shape, seed, layer, h)
        got = inst.debug_layer(layer, h.astype(np.float32)).astype(np.float64)
        err, scale = np.abs(got - ref).max(), np.abs(ref).max()
        worst = max(worst, err / scale)
        assert err <= scale * 2 ** -8, (model, layer, err, scale)
        h = ref
    lg = inst.debug_head(h.astype(np.float32))
    ref = oracle.decoder_head(shape, seed, h)
    head_err = np.abs(lg - ref).max()
    print(model, "worst layer err / max|h|", worst, "head max-abs", head_err)
    assert head_err <= 2e-2, head_err
    inst.close()
    del inst
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ the benchmarked configuration
def test_c2_scale_pipelined_engine(sgs):
    # config-2 scale on the production path -- 7B shape, 256
    # prompts x 512 tokens, B = 256, default flags (CUDA graphs, 16K-token
    # prefill chunks, split-K, host/device pipelining; no KEEP_LOGITS).  The
    # schedule trace is bit-exact against the oracle simulator.  The same batch
    # with SGS_F_KEEP_LOGITS (the same kernels, graphs and concurrent prefill;
    # only the host pipelining is off -- pipelining is bitwise neutral, see
    # test_deterministic_paths_bitwise_equal) exposes the logits: a probe sample
    # (8-token prompt, 24 forced tokens) generated inside the 256-row graphs is
    # teacher-forced through the oracle decoder within the 28-layer tolerance
    # (R17), and the two runs' tokens agree up to split-K summation order (R21).
    shape = workload.MODELS["qwen2.5-7b"]
    seed = 4321
    tr = workload.make_trace(256, 512, 24, 1.0, 64, shape.vocab, seed=12)
    probe = tr.subset([0])
    probe = workload.Trace(probe.ids, np.array([8]), np.array([24]), np.array([64]), probe.tokens[:8],
                           np.array([0, 8]))
    rest = tr.subset(np.arange(1, 256))
    cat = lambda f: np.concatenate([getattr(probe, f), getattr(rest, f)])
    full = workload.Trace(cat("ids"), cat("prompt_len"), cat("forced_len"), cat("hint"),
                          np.concatenate([probe.tokens, rest.tokens]).astype(np.int32),
                          np.concatenate([[0], np.cumsum(cat("prompt_len"))]))
    pool = 256 * 40
    pid = int(probe.ids[0])
    o = oracle.sched_sim(full.ids, full.prompt_len, full.forced_len, full.hint, 256, 16, pool)
    inst = sgs.Instance(shape, 256, 512 + 64, device=0, n_pages=pool, weight_seed=seed)
    inst.submit_trace(full)
    comps = inst.run()
    assert np.array_equal(inst.trace(0), o["iter_blob"])
    assert np.array_equal(inst.trace(1), o["sample_blob"])
    assert [c["id"] for c in comps] == [i for it in o["iters"] for i in it["completed"]]
    toks_a = {c["id"]: c["tokens"] for c in comps}
    inst.close()
    del inst
    inst = sgs.Instance(shape, 256, 512 + 64, device=0, n_pages=pool, weight_seed=seed, flags=sgs.sgs.F_KEEP_LOGITS)
    rows, gaps, comps = {}, {}, []  # full logits rows for the probe only; top-2 gaps for every position
    inst.submit_trace(full)
    while True:
        q, a = inst.pending()
        if q == 0 and a == 0:
            break
        comps += inst.step()
        lg, ids, tk = inst.last_logits()
        top2 = np.sort(np.partition(lg, -2, axis=1)[:, -2:], axis=1) if len(ids) else np.zeros((0, 2))
        for r in range(len(ids)):
            gaps[(int(ids[r]), int(tk[r]))] = float(top2[r, 1] - top2[r, 0])
            if int(ids[r]) == pid:
                rows[(pid, int(tk[r]))] = lg[r].copy()
    assert np.array_equal(inst.trace(0), o["iter_blob"])
    toks_b = {c["id"]: c["tokens"] for c in comps}
    gen = toks_b[pid]
    assert len(gen) == 24
    got = np.stack([rows[(pid, j)] for j in range(24)])
    assert np.array_equal(got.argmax(1), gen)
    seq = np.concatenate([probe.tokens, gen[:-1]]).astype(np.int32)
    ref = oracle.decoder_forward(shape, seed, seq, first_row=7)
    err = np.abs(got - ref).max()
    print("c2-scale probe: teacher-forced max-abs logits error", err)
    assert err <= TOL_7B_28L, err
    srt = np.sort(ref, 1)
    clear = (srt[:, -1] - srt[:, -2]) > 2 * TOL_7B_28L
    assert np.array_equal(ref.argmax(1)[clear], gen[clear])
    # pipelined (bench) run vs logits run: split-K's fp32 summation order (R21)
    # perturbs the 28-layer logits by up to the R17 floor, so with random
    # weights' near-uniform logits many samples take another token somewhere;
    # wherever they first differ the logits run's top-2 gap must lie within
    # 2x the tolerance (a genuine divergence would show at clear positions)
    for i in toks_a:
        d = np.flatnonzero(toks_a[i] != toks_b[i])
        if len(d):
            assert gaps[(i, int(d[0]))] < 2 * TOL_7B_28L, (i, int(d[0]), gaps[(i, int(d[0]))])
    inst.close()
    del inst
    # with SGS_F_DETERMINISTIC (no split-K) the pipelined run and the logits run
    # of the same 256-row production configuration must agree bit for bit
    runs = []
    for flags in (sgs.sgs.F_DETERMINISTIC, sgs.sgs.F_DETERMINISTIC | sgs.sgs.F_KEEP_LOGITS):
        inst = sgs.Instance(shape, 256, 512 + 64, device=0, n_pages=pool, weight_seed=seed, flags=flags)
        inst.submit_trace(full)
        c = inst.run()
        assert np.array_equal(inst.trace(0), o["iter_blob"])
        runs.append({x["id"]: tuple(x["tokens"]) for x in c})
        inst.close()
        del inst
    assert runs[0] == runs[1]


# ------------------------------------------------------------------ NEXT-3 prefix sharing
@pytest.mark.parametrize("model,G,P", [("tiny", 4, 40), ("tiny", 3, 32), ("qwen2.5-7b", 4, 40)])
def test_prefix_sharing_end_to_end(sgs, model, G, P):
    # P:1005-1007 "prefix sharing to save key-value cache usage" (reading R26):
    # GRPO groups of G samples per prompt; the schedule (with the group page
    # rule) is bit-exact against the oracle, and every member's teacher-forced
    # logits -- the first member's from the prefill, the others' first token from
    # a decode row at position P-1 over the shared pages -- match the oracle
    # decoder on its own prompt + tokens
    shape = workload.MODELS[model]
    n = 24 if model == "tiny" else 8
    tr = workload.make_trace(n, P, 12, 0.8, 40 if model == "tiny" else 12, shape.vocab, seed=G * 100 + P,
                             group_size=G)
    B, pool = (6, 200) if model == "tiny" else (4, 64)
    inst = sgs.Instance(shape, B, P + 64, device=0, n_pages=pool, weight_seed=31,
                        flags=sgs.sgs.F_KEEP_LOGITS | sgs.sgs.F_PREFIX_SHARING)
    comps, rows = _run_collect(inst, tr)
    group = np.arange(n) // G
    o = oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, B, 16, pool, group=group)
    assert np.array_equal(inst.trace(0), o["iter_blob"])
    assert np.array_equal(inst.trace(1), o["sample_blob"])
    check = tr.ids.tolist() if model == "tiny" else tr.ids[:G].tolist()  # 7B: one whole group
    tol = 2e-2 if model == "tiny" else TOL_7B_28L
    worst = _check_teacher_forced(shape, 31, tr, comps, rows, check, tol=tol)
    print(model, "prefix sharing worst teacher-forced max-abs", worst)
    inst.close()
