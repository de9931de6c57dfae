"""CPU parity of the product's host control plane (null-device mode of libsgs)
against the oracle: schedules, block tables, emitted order, dispatch and the
T(b) fit must agree bit for bit (north_star)."""
import numpy as np
import pytest

import oracle
import workload
from paper_2504_15930_b200 import Instance, SgsError, dispatch_plan, fit_profile

PROF = (20000, 500, 128, 2000)


def run_null(tr, B, page, pool, N=1, rank=0, batches=None, shape="qwen2.5-7b", **kw):
    inst = Instance(workload.MODELS[shape], B, 40000, device=None, page_size=page, n_pages=pool,
                    n_instances=N, instance_rank=rank, profile=PROF, **kw)
    comps = []
    if batches is None:
        inst.submit_trace(tr)
        comps = inst.run()
    else:
        # batches: list of (trace, submit_after_iterations)
        it = 0
        pending = list(batches)
        while True:
            while pending and pending[0][1] <= it:
                inst.submit_trace(pending.pop(0)[0])
            q, a = inst.pending()
            if q == 0 and a == 0 and not pending:
                break
            if q == 0 and a == 0:
                inst.submit_trace(pending.pop(0)[0])
                continue
            comps.extend(inst.step())
            it += 1
    return inst, comps


def oracle_trace(tr, B, page, pool, batch=None, arrival=None):
    return oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, B, page, pool, batch=batch,
                            arrival_after=arrival)


def assert_same(inst, o):
    got_it = inst.trace(0)
    got_s = inst.trace(1)
    assert np.array_equal(got_it, o["iter_blob"])
    assert np.array_equal(got_s, o["sample_blob"])


@pytest.mark.parametrize("cfg,pool", [("c1_tiny", 2000), ("c1_tiny", 40), ("c2_7b", 171_000), ("c2_7b", 20_000)])
def test_schedule_bit_exact_config_traces(cfg, pool):
    c = workload.CONFIGS[cfg]
    tr = workload.config_trace(c)
    inst, comps = run_null(tr, c.max_batch, c.page_size, pool)
    o = oracle_trace(tr, c.max_batch, c.page_size, pool)
    assert_same(inst, o)
    # emitted order: by finish iteration, ascending id within an iteration
    order = [x["id"] for x in comps]
    exp = [i for it in o["iters"] for i in it["completed"]]
    assert order == exp
    assert all(len(x["tokens"]) == int(tr.forced_len[x["id"]]) for x in comps)


def test_schedule_noisy_hints_and_ragged_prompts():
    tr = workload.make_trace(200, 40, 60, 1.2, 900, 512, seed=9, hint_noise=0.6, prompt_len_jitter=30)
    inst, _ = run_null(tr, 24, 16, 500)
    assert_same(inst, oracle_trace(tr, 24, 16, 500))


def test_schedule_edge_cases():
    # single sample d=1; B=1; all equal lengths; pool exactly one sample
    for (n, P, d, B, pool) in [(1, 1, 1, 4, 10), (5, 3, 7, 1, 100), (9, 16, 16, 3, 100), (4, 20, 13, 4, 3)]:
        ids = np.arange(n)
        tr = workload.Trace(ids, np.full(n, P), np.full(n, d), np.full(n, d),
                            np.zeros(n * P, np.int32), np.arange(n + 1) * P)
        inst, comps = run_null(tr, B, 16, pool)
        assert_same(inst, oracle_trace(tr, B, 16, pool))
        assert len(comps) == n


def test_schedule_multi_batch_fifo():
    a = workload.make_trace(30, 8, 20, 1.0, 120, 512, seed=3)
    b = workload.make_trace(30, 8, 20, 1.0, 120, 512, seed=4, id_base=1000)
    inst, _ = run_null(None, 8, 16, 300, batches=[(a, 0), (b, 25)])
    ids = np.concatenate([a.ids, b.ids])
    cat = lambda f: np.concatenate([getattr(a, f), getattr(b, f)])
    tr = workload.Trace(ids, cat("prompt_len"), cat("forced_len"), cat("hint"), np.zeros(1, np.int32), None)
    o = oracle_trace(tr, 8, 16, 300, batch=np.array([0] * 30 + [1] * 30), arrival=np.array([0] * 30 + [25] * 30))
    assert_same(inst, o)


def test_capacity_and_validation_errors():
    from paper_2504_15930_b200 import SgsError
    inst = Instance(workload.MODELS["tiny"], 4, 100, device=None, n_pages=5)
    tr = workload.make_trace(3, 8, 10, 0.0, 10, 512, seed=1)
    with pytest.raises(SgsError) as e:  # hint 0
        inst.submit(tr.ids, tr.tokens, tr.offsets, np.zeros(3), tr.forced_len)
    assert e.value.code == -1
    with pytest.raises(SgsError) as e:  # P + d - 1 > max_ctx
        inst.submit(tr.ids, tr.tokens, tr.offsets, tr.hint, np.full(3, 200))
    assert e.value.code == -4
    with pytest.raises(SgsError) as e:  # token out of range
        inst.submit(tr.ids, np.full_like(tr.tokens, 999), tr.offsets, tr.hint, tr.forced_len)
    assert e.value.code == -1
    assert inst.submit_trace(tr) == 3
    with pytest.raises(SgsError):  # duplicate id
        inst.submit_trace(tr)
    assert inst.step() == [] or True
    with pytest.raises(SgsError) as e:  # update while busy
        inst.update_weights(0)
    assert e.value.code == -3
    inst.run()
    assert inst.step() == []  # idle: no iteration counted
    n_it = len(oracle.parse_iter_blob(inst.trace(0)))
    inst.update_weights(0)
    assert inst.weight_version() == 1
    assert len(oracle.parse_iter_blob(inst.trace(0))) == n_it


def test_async_weight_sync_state_machine():
    # NEXT-1: one update in flight; commit only at an RL-batch
    # boundary; samples of the batch in flight keep the old version, the next
    # batch gets the new one (staleness 1)
    inst = Instance(workload.MODELS["tiny"], 4, 100, device=None, n_pages=50)
    with pytest.raises(SgsError) as e:  # nothing in flight
        inst.update_weights_commit()
    assert e.value.code == -3
    tr = workload.make_trace(6, 8, 10, 0.5, 10, 512, seed=3)
    inst.submit_trace(tr)
    inst.step()
    inst.update_weights_begin(0)  # overlaps generation
    with pytest.raises(SgsError) as e:  # a second update
        inst.update_weights_begin(0)
    assert e.value.code == -3
    with pytest.raises(SgsError) as e:  # the synchronous path is blocked meanwhile
        inst.update_weights(0)
    assert e.value.code == -3
    assert inst.update_weights_ready()
    with pytest.raises(SgsError) as e:  # samples in flight
        inst.update_weights_commit()
    assert e.value.code == -3
    done = inst.run()
    assert {c["weight_version"] for c in done} == {0}
    inst.update_weights_commit()
    assert inst.weight_version() == 1
    tr2 = workload.make_trace(3, 8, 5, 0.5, 5, 512, seed=4, id_base=100)
    inst.submit_trace(tr2)
    assert {c["weight_version"] for c in inst.run()} == {1}


def test_dispatch_bit_exact_vs_oracle():
    rng = np.random.default_rng(11)
    for trial in range(300):
        n = int(rng.integers(1, 120))
        N = int(rng.integers(1, 9))
        ids = rng.permutation(5000)[:n].astype(np.uint64)
        hint = rng.integers(1, 20000, size=n)
        P = rng.integers(1, 700, size=n)
        B = int(rng.integers(1, 300))
        pool = int(rng.integers(50, 100000))
        prof = (int(rng.integers(100, 9000)), int(rng.integers(1, 200)) * 1000, int(rng.integers(1, 400)),
                int(rng.integers(200, 900)) * 1000)
        alpha = int(rng.integers(0, 101))
        score = int(rng.integers(0, 2))
        tc = int(rng.integers(0, 2))
        got, nl = dispatch_plan(ids, P, hint, N, B, 16, pool, prof, alpha, score, tc)
        exp = oracle.dispatch(ids.astype(np.int64), P, hint, N, B, 16, pool, prof, alpha, score, tc)
        assert np.array_equal(got, exp["instance"]), trial
        if N > 1:
            assert nl == exp["n_l"]


def test_submit_keeps_dispatched_share():
    tr = workload.config_trace("c3_14b_4", n=256)
    N, pool = 4, 50_000
    exp = oracle.dispatch(tr.ids, tr.prompt_len, tr.hint, N, 256, 16, pool, PROF)["instance"]
    seen = []
    for r in range(N):
        inst, comps = run_null(tr, 256, 16, pool, N=N, rank=r)
        mine = sorted(x["id"] for x in comps)
        assert mine == sorted(tr.ids[exp == r].tolist())
        sub = tr.subset(np.flatnonzero(exp == r))
        assert_same(inst, oracle_trace(sub, 256, 16, pool))
        seen += mine
    assert sorted(seen) == tr.ids.tolist()


def test_fit_matches_oracle():
    rng = np.random.default_rng(5)
    for _ in range(40):
        t0, k0, k1 = rng.uniform(500, 5000), rng.uniform(0.5, 20), rng.uniform(25, 80)
        bs = int(rng.choice([32, 64, 128, 192, 256]))
        b = np.array([1, 2, 4, 8, 16, 32, 64, 96, 128, 160, 192, 224, 256, 320, 384, 512, 768, 1024], float)
        T = np.where(b < bs, t0 + k0 * b, t0 + k0 * bs + k1 * (b - bs)) * (1 + rng.uniform(-0.02, 0.02, b.size))
        g, o = fit_profile(b, T), oracle.tb_fit(b, T)
        assert g["profile"][2] == o["b_star"]
        for k in ("t0", "k0", "k1", "t1"):
            assert abs(g[k] - o[k]) <= 1e-6 * max(1.0, abs(o[k]))
        assert g["profile"] == o["profile"]


def test_product_reservation_golden():
    # the product's scheduler on the hand-derived binding-reservation trace
    # (tests/golden/sched_reservation_binds.json)
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sched_reservation_binds.json")))
    s = np.array(g["samples"])
    n = len(s)
    tr = workload.Trace(s[:, 0], s[:, 1], s[:, 2], s[:, 3], np.zeros(int(s[:, 1].sum()), np.int32),
                        np.concatenate([[0], np.cumsum(s[:, 1])]))
    inst, comps = run_null(tr, g["B"], g["page"], g["pool"], shape="tiny")
    o = oracle_trace(tr, g["B"], g["page"], g["pool"])
    assert_same(inst, o)
    assert o["iters"] == g["iters"] and len(comps) == n


def test_product_dispatch_golden():
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "dispatch_eq2_n4_memcap.json")))
    for mode, key in ((0, "expect_sum"), (1, "expect_max")):
        inst, nl = dispatch_plan(g["ids"], g["prompt_len"], g["hint"], g["N"], g["B"], g["page"], g["pool"],
                                 g["profile"], alpha_pct=g["alpha_pct"], score=mode)
        assert nl == g[key]["n_l"]
        assert inst.tolist() == g[key]["instance"]


def test_host_state_bounded_without_trace_and_id_reuse():
    # ADVICE/VERDICT r01: without SGS_F_TRACE the host state is bounded by the
    # samples in flight (records recycled, queue prefix dropped, live ids only);
    # an id may be submitted again once its sample has completed (R22)
    shape = workload.MODELS["tiny"]
    inst = Instance(shape, 8, 400, device=None, n_pages=400, trace=False)
    peak = (0, 0, 0)
    for k in range(30):
        tr = workload.make_trace(100, 8, 20, 1.0, 120, shape.vocab, seed=k)  # same ids 0..99 every batch
        assert inst.submit_trace(tr) == 100
        with pytest.raises(SgsError) as e:  # ids still queued
            inst.submit_trace(tr)
        assert e.value.code == -1
        comps = inst.run()
        assert sorted(c["id"] for c in comps) == list(range(100))
        st = inst.host_state()
        peak = tuple(max(a, b) for a, b in zip(peak, st))
        assert st[2] == 0
    assert peak[0] <= 200 and peak[1] <= 2 * 1024 + 100, peak
    # with tracing every record is kept (the per-sample trace needs them)
    inst = Instance(shape, 8, 400, device=None, n_pages=400, trace=True)
    for k in range(3):
        inst.submit_trace(workload.make_trace(50, 8, 20, 1.0, 120, shape.vocab, seed=k, id_base=1000 * k))
        inst.run()
    assert inst.host_state()[0] == 150


def test_elastic_plan_matches_oracle():
    # NEXT-4: the product's delta' (Alg. 2 + its own scheduler, timed
    # with the integer T(b) profile) equals the oracle's bit for bit, and the
    # decision flips exactly at delta = delta'
    import json
    import os
    from paper_2504_15930_b200 import elastic_plan
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "elastic_delta_prime.json")))
    for delta, dec in g["decisions"]:
        r = elastic_plan(g["ids"], g["P"], g["hint"], g["N"], g["B"], g["page"], g["pool"], g["profile"], delta)
        assert r["t_gen_ps"] == tuple(g["t_gen_ps"]) and r["scale_out"] == dec
    rng = np.random.default_rng(3)
    for _ in range(60):
        n, N = int(rng.integers(1, 120)), int(rng.integers(1, 6))
        ids, P, hint = rng.permutation(10_000)[:n], rng.integers(1, 600, n), rng.integers(1, 3000, n)
        prof = (int(rng.integers(100, 5000)), int(rng.integers(1, 100)) * 1000, int(rng.integers(2, 300)),
                int(rng.integers(100, 300)) * 1000)
        B, pool = int(rng.integers(1, 64)), int(rng.integers(400, 20_000))
        if ((P + hint - 1 + 15) // 16).max() > pool:
            continue
        o = oracle.elastic_plan(ids, P, hint, N, B, 16, pool, prof, 0)
        r = elastic_plan(ids, P, hint, N, B, 16, pool, prof, o["delta_prime_ps"])
        assert r["t_gen_ps"] == o["t_gen_ps"]
        assert r["delta_prime_ps"] == o["delta_prime_ps"]
        assert r["scale_out"] == (o["delta_prime_ps"] > 0)


def test_set_instances_between_batches():
    shape = workload.MODELS["tiny"]
    tr = workload.make_trace(40, 8, 20, 1.0, 100, shape.vocab, seed=4)
    inst = Instance(shape, 8, 400, device=None, n_pages=400, n_instances=1, instance_rank=0, profile=PROF)
    assert inst.submit_trace(tr) == 40
    with pytest.raises(SgsError) as e:
        inst.set_instances(2, 0)
    assert e.value.code == -3
    inst.run()
    inst.set_instances(2, 1)
    tr2 = workload.make_trace(40, 8, 20, 1.0, 100, shape.vocab, seed=5, id_base=1000)
    exp, _ = dispatch_plan(tr2.ids, tr2.prompt_len, tr2.hint, 2, 8, 16, 400, PROF)
    assert inst.submit_trace(tr2) == int((exp == 1).sum())


@pytest.mark.parametrize("G,P,jitter", [(4, 40, 0), (8, 64, 0), (3, 20, 15), (2, 16, 0)])
def test_prefix_sharing_schedule_matches_oracle(G, P, jitter):
    # NEXT-3 (R26): with SGS_F_PREFIX_SHARING the product's schedule,
    # page lists and page log equal the oracle's with the groups the workload
    # implies (identical prompts of one batch); without the flag, the unshared one
    from paper_2504_15930_b200 import sgs as binding
    shape = workload.MODELS["tiny"]
    tr = workload.make_trace(96, P, 30, 1.0, 200, shape.vocab, seed=G * 7 + P, group_size=G,
                             prompt_len_jitter=jitter)
    group = np.arange(len(tr)) // G
    for B, pool in ((8, 4000), (16, 120)):
        inst = Instance(shape, B, 40000, device=None, n_pages=pool, profile=PROF, flags=binding.F_PREFIX_SHARING)
        inst.submit_trace(tr)
        inst.run()
        o = oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, B, 16, pool, group=group)
        assert_same(inst, o)
        if P >= 32:  # shared pages exist only before the page holding position P-1
            u = oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, B, 16, pool)
            assert sum(len(it["alloc"]) for it in o["iters"]) < sum(len(it["alloc"]) for it in u["iters"])
