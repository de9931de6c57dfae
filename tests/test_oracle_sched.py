"""Pins for the oracle's scheduling half (C2-C5): closed forms, brute force,
hand-derived golden traces and the paper's own worked facts.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import workload

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PROF = (100, 1000, 64, 3000)  # t0=100ns, k0=1ns/sample, b*=64, k1=3ns/sample -> t1 = 100+(1-3)*64 < 0? no:
# t1 = t0 + (k0-k1) b* in ns = 100 - 128 = -28 ns (negative control); see PROF_OK for t1 > 0
PROF_OK = (20000, 500, 128, 2000)  # t1 = 20000 + (0.5-2)*128 = 19808 ns > 0


def T(b, prof=PROF_OK):
    return oracle.T_ps(prof, b)


# ----------------------------------------------------------------- C3 T(b)
def test_T_piecewise_and_continuity():
    # appendix equation P:32-37 evaluated by hand
    t0, k0, bs, k1 = PROF_OK
    assert T(1) == t0 * 1000 + k0 * 1
    assert T(bs - 1) == t0 * 1000 + k0 * (bs - 1)
    # continuity k0 b* + t0 = k1 b* + t1: both branches agree at b*
    assert T(bs) == t0 * 1000 + k0 * bs
    t1_ps = t0 * 1000 + (k0 - k1) * bs
    assert T(bs + 10) == k1 * (bs + 10) + t1_ps
    assert T(500) == k1 * 500 + t1_ps


def test_spec_ptl_worked_example():
    # t0=20, k0=0.05, b*=128, k1=0.4 (ms) -> ptl(1)=20.05, ptl(128)=26.4, ptl(200)=55.2
    prof = (20_000_000, 50_000_000, 128, 400_000_000)  # ns, ps
    assert T(1, prof) == 20_050_000_000
    assert T(128, prof) == 26_400_000_000
    assert T(200, prof) == 55_200_000_000


def test_merge_lemma_positive_t1():
    # T(x+y) < T(x)+T(y) for all x,y>=1 iff t1 > 0; with x,y >= b* the
    # gain is exactly t1 (R11 derivation).
    gain, x, y = oracle.min_merge_gain(PROF_OK, 600)
    t0, k0, bs, k1 = PROF_OK
    t1_ps = t0 * 1000 + (k0 - k1) * bs
    assert gain == t1_ps > 0
    assert x >= bs and y >= bs


def test_merge_lemma_negative_control_spec_profile():
    # S:137-139 profile has t1 = -24.8 ms < 0, so the lemma must FAIL on it
    prof = (20_000_000, 50_000_000, 128, 400_000_000)
    gain, x, y = oracle.min_merge_gain(prof, 512)
    assert gain < 0
    assert gain == -24_800_000_000


def test_merge_lemma_below_bstar_gain_is_t0():
    # x + y < b*: D = t0 exactly
    prof = (20000, 500, 10**6, 2000)
    gain, _, _ = oracle.min_merge_gain(prof, 300)
    assert gain == 20000 * 1000


def test_fit_noiseless_roundtrip():
    # points sampled from a known profile recover it
    t0, k0, k1, bs = 1800.0, 2.5, 9.0, 192
    bs_grid = [1, 2, 4, 8, 16, 32, 64, 96, 128, 160, 192, 224, 256, 320, 384, 512, 768, 1024]
    Tn = [t0 + k0 * b if b < bs else t0 + k0 * bs + k1 * (b - bs) for b in bs_grid]
    f = oracle.tb_fit(bs_grid, Tn)
    assert f["ok"] and f["b_star"] == bs
    assert abs(f["t0"] - t0) < 1e-6 * t0 and abs(f["k0"] - k0) < 1e-6 * k0 and abs(f["k1"] - k1) < 1e-6 * k1
    assert abs(f["t1"] - (t0 + (k0 - k1) * bs)) < 1e-6
    assert f["profile"] == (1800, 2500, 192, 9000)


def test_fit_noisy_k1_within_5pct():
    rng = np.random.default_rng(0)
    t0, k0, k1, bs = 3000.0, 4.0, 14.0, 128
    b = np.array([1, 2, 4, 8, 16, 32, 64, 96, 128, 160, 192, 256, 384, 512, 768, 1024], float)
    Tn = np.where(b < bs, t0 + k0 * b, t0 + k0 * bs + k1 * (b - bs))
    Tn = Tn * (1 + rng.uniform(-0.01, 0.01, size=b.shape))
    f = oracle.tb_fit(b, Tn)
    assert abs(f["k1"] - k1) / k1 < 0.05


def test_fit_rejects_degenerate():
    assert not oracle.tb_fit([4, 4, 4], [1.0, 2.0, 3.0])["ok"]


# ----------------------------------------------------------------- C4
def test_lf_counterexample_spec_and_survey():
    # S:350 and SURVEY §0.5-3: [8,7,6,5,4] on 2 slots, LF 17 iterations vs optimum 15
    r = oracle.brute_force([8, 7, 6, 5, 4], 2, (100, 0, 10**9, 0))  # constant T: time = iterations
    assert r["lf_iters"] == 17 and r["opt_iters_min"] == 15
    assert r["lf_time"] == 17 * 100_000 and r["opt_time"] == 15 * 100_000


def test_graham_tight_case():
    # Graham 1969 LPT tight example: [3,3,2,2,2], m=2 -> 7 vs 6 (ratio 4/3 - 1/(3m))
    r = oracle.brute_force([3, 3, 2, 2, 2], 2, (100, 0, 10**9, 0))
    assert r["lf_iters"] == 7 and r["opt_iters_min"] == 6
    assert r["lf_iters"] / r["opt_iters_min"] == pytest.approx(4 / 3 - 1 / 6)


def test_lpt_bound_random_suite():
    # LPT within 4/3 of optimal; >=1000 cases, bound exercised (>1.05)
    rng = np.random.default_rng(1)
    worst = 1.0
    n = 0
    while n < 1000:
        M = int(rng.integers(2, 8))
        B = int(rng.integers(2, 4))
        d = rng.integers(1, 12, size=M)
        r = oracle.brute_force(d, B, (100, 0, 10**9, 0))
        ratio = r["lf_iters"] / r["opt_iters_min"]
        assert ratio <= 4 / 3 + 1e-12
        worst = max(worst, ratio)
        n += 1
    assert worst > 1.05


def test_lf_time_bound_two_segment_profiles():
    # two-segment T with t1 > 0: LF time within 4/3 of the best admission order
    rng = np.random.default_rng(2)
    for _ in range(300):
        M = int(rng.integers(2, 7))
        B = int(rng.integers(2, 4))
        d = rng.integers(1, 10, size=M)
        bs = int(rng.integers(2, 4))
        prof = (int(rng.integers(100, 1000)), int(rng.integers(1, 50)) * 1000, bs, int(rng.integers(50, 200)) * 1000)
        t1 = prof[0] * 1000 + (prof[1] - prof[3]) * bs
        if t1 <= 0:
            continue
        r = oracle.brute_force(d, B, prof)
        assert r["lf_time"] * 3 <= r["opt_time"] * 4


def test_B1_and_B_ge_M_exact():
    prof = PROF_OK
    d = [5, 3, 9, 1]
    r = oracle.brute_force(d, 1, prof)
    assert r["lf_time"] == r["opt_time"] == sum(d) * T(1)
    r = oracle.brute_force(d, 4, prof)
    # M <= B: every order equal, time = sum_t T(#alive_t)
    alive = [sum(1 for x in d if x > t) for t in range(max(d))]
    assert r["lf_time"] == r["opt_time"] == sum(T(a) for a in alive)


# ----------------------------------------------------------------- C2
def test_sched_hand_trace_golden():
    g = json.load(open(os.path.join(GOLD, "sched_hand_trace.json")))
    s = np.array(g["samples"])
    r = oracle.sched_sim(s[:, 0], s[:, 1], s[:, 2], s[:, 3], g["B"], g["page"], g["pool"])
    assert r["iters"] == g["iters"]
    assert {str(k): v for k, v in r["samples"].items()} == g["per_sample"]


def test_sched_eq2_equals_simulator_equal_lengths():
    # S:157 / S:208 / acceptance 4: Eq. 2 = simulated makespan when all lengths
    # equal L and M is a multiple of BS (here BS = B, memory not binding).
    for (M, B, L) in [(8, 4, 5), (12, 3, 7), (16, 16, 3), (64, 16, 10), (30, 5, 1)]:
        ids = np.arange(M)
        r = oracle.sched_sim(ids, np.full(M, 4), np.full(M, L), np.full(M, L), B, 16, 10**6, profile=PROF_OK)
        assert r["n_iters"] == L * (M // B)
        assert r["time_ps"] == T(B) * L * math.ceil(M / B)


def test_sched_closed_forms_B1_and_M_le_B():
    d = np.array([4, 9, 2, 6])
    ids = np.arange(4)
    r = oracle.sched_sim(ids, np.full(4, 3), d, d, 1, 16, 1000, profile=PROF_OK)
    assert r["time_ps"] == int(d.sum()) * T(1)
    r = oracle.sched_sim(ids, np.full(4, 3), d, d, 8, 16, 1000, profile=PROF_OK)
    alive = [int((d > t).sum()) for t in range(d.max())]
    assert r["time_ps"] == sum(T(a) for a in alive)


def _check_invariants(tr, r, B, page, pool):
    ids = tr.ids
    d = dict(zip(ids.tolist(), tr.forced_len.tolist()))
    P = dict(zip(ids.tolist(), tr.prompt_len.tolist()))
    owned = {}
    active = set()
    produced = {i: 0 for i in d}
    for it in r["iters"]:
        for a in it["admitted"]:
            active.add(a)
        assert it["b"] == len(active) <= B
        for i in active:
            produced[i] += 1
        for p in it["alloc"]:
            assert p not in owned and 0 <= p < pool
            owned[p] = True
        assert sorted(it["completed"]) == it["completed"]
        for c in it["completed"]:
            assert produced[c] == d[c]
            active.discard(c)
        for p in it["freed"]:
            del owned[p]
    assert sum(produced.values()) == sum(d.values())  # conservation
    assert not owned and not active
    for i, rec in r["samples"].items():
        assert len(rec["pages"]) == math.ceil((P[i] + d[i] - 1) / page)
        assert rec["finish"] - rec["admit"] + 1 == d[i]


@pytest.mark.parametrize("cfg", ["c1_tiny", "c2_7b"])
def test_sched_invariants_config_traces(cfg):
    c = workload.CONFIGS[cfg]
    tr = workload.config_trace(c)
    pool = 2000 if cfg == "c1_tiny" else 171_000
    r = oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, c.max_batch, c.page_size, pool)
    _check_invariants(tr, r, c.max_batch, c.page_size, pool)
    # longest-first: admission order is (hint desc, id asc) when memory never binds
    adm = [a for it in r["iters"] for a in it["admitted"]]
    order = sorted(tr.ids.tolist(), key=lambda i: (-int(tr.hint[i]), i))
    assert adm == order


def test_sched_reservation_binds_strict_order():
    # memory-tight pool: the reservation rule (P:975-978 reading R3) limits
    # concurrency; admission stays strictly in LF order (no backfill)
    tr = workload.make_trace(40, 8, 30, 1.0, 200, 64, seed=5)
    pool = 60
    r = oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, 16, 4, pool)
    _check_invariants(tr, r, 16, 4, pool)
    assert max(it["b"] for it in r["iters"]) < 16
    adm = [a for it in r["iters"] for a in it["admitted"]]
    assert adm == sorted(tr.ids.tolist(), key=lambda i: (-int(tr.hint[i]), i))


def test_sched_multi_batch_fifo():
    # two RL batches: batch 2 queued after 5 iterations, admitted only after
    # batch 1's queue is empty, may co-run with batch 1's tail (R5)
    a = workload.make_trace(10, 4, 8, 1.0, 40, 64, seed=3)
    b = workload.make_trace(10, 4, 8, 1.0, 40, 64, seed=4, id_base=100)
    ids = np.concatenate([a.ids, b.ids])
    P = np.concatenate([a.prompt_len, b.prompt_len])
    d = np.concatenate([a.forced_len, b.forced_len])
    h = np.concatenate([a.hint, b.hint])
    batch = np.array([0] * 10 + [1] * 10)
    arr = np.array([0] * 10 + [5] * 10)
    r = oracle.sched_sim(ids, P, d, h, 4, 4, 1000, batch=batch, arrival_after=arr)
    adm = [x for it in r["iters"] for x in it["admitted"]]
    assert adm[:10] == sorted(a.ids.tolist(), key=lambda i: (-int(a.hint[i]), i))
    assert all(r["samples"][int(i)]["admit"] >= 5 for i in b.ids)


# ----------------------------------------------------------------- C5
def _disp(ids, P, hint, N, B=256, page=16, pool=10**6, prof=PROF_OK, **kw):
    return oracle.dispatch(ids, P, hint, N, B, page, pool, prof, **kw)


def test_nearest_rank_spec_examples():
    # [1..100] -> p50=50, p90=90; [5,5,5] -> 5; 64 L + 2 (2L): p90 = L
    assert oracle.nearest_rank(np.arange(1, 101), 50) == 50
    assert oracle.nearest_rank(np.arange(1, 101), 90) == 90
    assert oracle.nearest_rank([5, 5, 5], 90) == 5
    assert oracle.nearest_rank([100] * 64 + [200] * 2, 90) == 100


def test_dispatch_toy_example_closed_form():
    # P:824-829 (Fig. design:scheduling left): DP=2, 64 regular of L + 2 long of 2L.
    # alpha=4% -> floor(0.04*66) = 2 tail samples = exactly the long ones; N_l = 1 forced.
    L = 100
    ids = np.arange(66)
    hint = np.array([2 * L] * 2 + [L] * 64)
    P = np.full(66, 16)
    r = _disp(ids, P, hint, 2, alpha_pct=4)
    assert r["n_tail"] == 2 and r["n_l"] == 1
    assert (r["instance"][:2] == 0).all() and (r["instance"][2:] == 1).all()
    # skew-aware makespan max(2L T(2), L T(64)) < random L (T(33)+T(1)) on the simulator
    prof = (100, 1000, 10**9, 0)  # t0 = 100ns, k0 = 1ns/sample: the SURVEY example
    def makespan(sel):
        sub = ids[sel]
        return oracle.sched_sim(sub, P[sel], hint[sel], hint[sel], 256, 16, 10**6, profile=prof)["time_ps"]
    skew = max(makespan(r["instance"] == 0), makespan(r["instance"] == 1))
    rnd_inst = np.array([0, 1] + [i % 2 for i in range(64)])
    rnd = max(makespan(rnd_inst == 0), makespan(rnd_inst == 1))
    assert skew == max(2 * L * T(2, prof), L * T(64, prof))
    assert rnd == L * (T(33, prof) + T(1, prof))
    assert (rnd, skew) == (23_400_000, 20_400_000)  # 23,400 vs 20,400 (ns)


def test_dispatch_exhaustive_argmin_and_partition():
    rng = np.random.default_rng(7)
    for trial in range(200):
        n = int(rng.integers(1, 80))
        N = int(rng.integers(1, 9))
        ids = rng.permutation(1000)[:n]
        hint = rng.integers(1, 5000, size=n)
        P = rng.integers(1, 600, size=n)
        B = int(rng.integers(1, 300))
        pool = int(rng.integers(50, 5000))
        page = 16
        prof = (int(rng.integers(100, 5000)), int(rng.integers(1, 100)) * 1000, int(rng.integers(1, 300)),
                int(rng.integers(100, 300)) * 1000)
        alpha = int(rng.integers(0, 60))
        mode = int(rng.integers(0, 2))
        r = _disp(ids, P, hint, N, B, page, pool, prof, alpha_pct=alpha, score_max=mode)
        # every sample in exactly one instance in [0, N)
        assert r["instance"].min() >= 0 and r["instance"].max() < N
        # re-enumerate Eq. 2 by hand in Python big ints
        n_tail = alpha * n // 100
        Lr, La = oracle.nearest_rank(hint, 50), oracle.nearest_rank(hint, 90)
        Pbar = -(-int(P.sum()) // n)
        def lat(cnt, L, k):
            if cnt == 0:
                return 0
            M = -(-cnt // k)
            bs = max(1, min(M, B, pool // (-(-(Pbar + L - 1) // page))))
            return oracle.T_ps(prof, bs) * L * (-(-M // bs))
        if N > 1 and 0 < n_tail < n:
            sc = []
            for nl in range(1, N):
                a, b = lat(n_tail, La, nl), lat(n - n_tail, Lr, N - nl)
                sc.append(max(a, b) if mode else a + b)
            assert r["scores"] == sc
            assert r["n_l"] == 1 + int(np.argmin(sc))  # first minimum = smaller N_l
        order = sorted(range(n), key=lambda i: (-int(hint[i]), int(ids[i])))
        nl = r["n_l"]
        for j, i in enumerate(order):
            if nl > 0 and (j < n_tail or nl == N):
                assert r["instance"][i] == j % nl
            else:
                jr = j if nl == 0 else j - n_tail
                assert r["instance"][i] == nl + jr % (N - nl)


def test_dispatch_degenerate():
    ids = np.arange(10)
    hint = np.arange(10, 0, -1)
    P = np.full(10, 8)
    r = _disp(ids, P, hint, 1)
    assert (r["instance"] == 0).all() and r["n_l"] == 0
    r = _disp(ids, P, hint, 4, alpha_pct=5)  # floor(0.5) = 0 -> all regular
    assert r["n_tail"] == 0 and r["n_l"] == 0
    assert sorted(np.bincount(r["instance"]).tolist()) == [2, 2, 3, 3]
    # ceil(0.2*66) = 14 with the ceil flag, floor gives 13
    h66 = np.array([200] * 2 + [100] * 64)
    assert _disp(np.arange(66), np.full(66, 8), h66, 2, tail_ceil=1)["n_tail"] == 14
    assert _disp(np.arange(66), np.full(66, 8), h66, 2)["n_tail"] == 13


# ----------------------------------------------------------------- hand-derived goldens (pins)
def test_sched_reservation_binds_golden():
    # tests/golden/sched_reservation_binds.json: the queue head is blocked by its
    # page reservation ceil((P+d-1)/page) (reading R3) while a later,
    # smaller sample would fit; strict LF order means no backfill.
    # A reservation of ceil((P+d)/page) or a backfilling admission fails this.
    g = json.load(open(os.path.join(GOLD, "sched_reservation_binds.json")))
    s = np.array(g["samples"])
    r = oracle.sched_sim(s[:, 0], s[:, 1], s[:, 2], s[:, 3], g["B"], g["page"], g["pool"])
    assert r["iters"] == g["iters"]
    assert {str(k): v for k, v in r["samples"].items()} == g["per_sample"]


@pytest.mark.parametrize("mode,key", [(0, "expect_sum"), (1, "expect_max")])
def test_dispatch_eq2_argmin_n4_memory_cap_golden(mode, key):
    # tests/golden/dispatch_eq2_n4_memcap.json: N = 4, every N_l's Eq. 2 score
    # computed by hand with the memory-capped BS binding for both groups
    # (P:969-978); argmin and the tie (max mode) resolve to N_l = 2.
    g = json.load(open(os.path.join(GOLD, "dispatch_eq2_n4_memcap.json")))
    r = oracle.dispatch(g["ids"], g["prompt_len"], g["hint"], g["N"], g["B"], g["page"], g["pool"], g["profile"],
                        alpha_pct=g["alpha_pct"], score_max=mode)
    e = g[key]
    assert (r["n_tail"], r["L_alpha"], r["L_r"]) == (8, 1000, 120)
    assert r["scores"] == e["scores"]
    assert r["n_l"] == e["n_l"]
    assert r["instance"].tolist() == e["instance"]


def test_elastic_delta_prime_golden():
    # tests/golden/elastic_delta_prime.json: NEXT-4's delta' for N = 1 -> 2 by hand (reading R25)
    g = json.load(open(os.path.join(GOLD, "elastic_delta_prime.json")))
    for delta, dec in g["decisions"]:
        r = oracle.elastic_plan(g["ids"], g["P"], g["hint"], g["N"], g["B"], g["page"], g["pool"], g["profile"], delta)
        assert r["t_gen_ps"] == tuple(g["t_gen_ps"])
        assert r["delta_prime_ps"] == g["delta_prime_ps"]
        assert r["scale_out"] == dec


def test_elastic_delta_prime_is_simulated_makespan_difference():
    # delta' composes C5 and C2: equals max over instances of sched_sim time on the dispatched subsets
    rng = np.random.default_rng(11)
    for _ in range(30):
        n, N = int(rng.integers(2, 60)), int(rng.integers(1, 5))
        ids, P, hint = np.arange(n), rng.integers(1, 40, n), rng.integers(1, 200, n)
        prof = (int(rng.integers(100, 3000)), int(rng.integers(1, 50)) * 1000, int(rng.integers(2, 64)),
                int(rng.integers(50, 200)) * 1000)
        B, page, pool = int(rng.integers(1, 16)), 16, 100000
        r = oracle.elastic_plan(ids, P, hint, N, B, page, pool, prof, 0)
        for k, NN in enumerate((N, N + 1)):
            inst = oracle.dispatch(ids, P, hint, NN, B, page, pool, prof)["instance"]
            mk = 0
            for i in range(NN):
                sel = inst == i
                if sel.any():
                    mk = max(mk, oracle.sched_sim(ids[sel], P[sel], hint[sel], hint[sel], B, page, pool,
                                                  profile=prof)["time_ps"])
            assert r["t_gen_ps"][k] == mk
        assert r["delta_prime_ps"] == r["t_gen_ps"][0] - r["t_gen_ps"][1]


@pytest.mark.parametrize("name", ["sched_prefix_sharing.json", "sched_prefix_sharing_full_page.json"])
def test_sched_prefix_sharing_golden(name):
    # tests/golden/sched_prefix_sharing*.json: NEXT-3 (reading R26) by hand
    g = json.load(open(os.path.join(GOLD, name)))
    s = np.array(g["samples"])
    r = oracle.sched_sim(s[:, 0], s[:, 1], s[:, 2], s[:, 3], g["B"], g["page"], g["pool"], group=s[:, 4])
    assert r["iters"] == g["iters"]
    assert {str(k): v for k, v in r["samples"].items()} == g["per_sample"]


def test_sched_prefix_sharing_invariants_and_savings():
    # random GRPO-style batches: G samples per prompt; conservation, no page owned twice except
    # the shared full prompt pages (held by every active member of a group), fewer page-iterations
    # than without sharing
    rng = np.random.default_rng(8)
    for trial in range(40):
        n_prompts, G = int(rng.integers(2, 12)), int(rng.integers(1, 6))
        P = np.repeat(rng.integers(1, 70, n_prompts), G)
        n = len(P)
        d = rng.integers(1, 60, n)
        ids = rng.permutation(10_000)[:n]
        group = np.repeat(np.arange(n_prompts), G)
        B, page, pool = int(rng.integers(1, 9)), 16, 400
        r = oracle.sched_sim(ids, P, d, d, B, page, pool, group=group)
        u = oracle.sched_sim(ids, P, d, d, B, page, pool)
        held, alive = {}, set()
        for it in r["iters"]:
            for p in it["alloc"]:
                assert p not in held and 0 <= p < pool
                held[p] = True
            for p in it["freed"]:
                del held[p]
        assert not held
        for i, rec in r["samples"].items():
            k = int(np.flatnonzero(ids == i)[0])
            assert len(rec["pages"]) == -(-(int(P[k]) + int(d[k]) - 1) // page)
            assert rec["finish"] - rec["admit"] + 1 == d[k]
        # pages allocated in total never exceed the unshared run's
        assert sum(len(it["alloc"]) for it in r["iters"]) <= sum(len(it["alloc"]) for it in u["iters"]) + n_prompts
