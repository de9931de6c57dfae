"""NEXT-2 two-dimensional dispatch (R27): the oracle pinned to a
hand-derived golden (tests/golden/tp_tail_plan.json) and to brute force over
every split on small random batches, and the product's sgs_tp_tail_plan equal
to the oracle bit for bit (pure host functions, no GPU)."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tp_tail_plan.json")))


def _plan_oracle(g, policy="round_robin"):
    return oracle.tp_tail_plan(g["ids"], g["P"], g["hint"], g["N"], g["B"], g["page"], g["pool"], g["profile"],
                               g["tp_size"], g["tp_B"], g["tp_pool"], g["tp_profile"], policy=policy)


def test_oracle_tail_plan_golden():
    o = _plan_oracle(GOLD)
    assert o["n_tail"] == GOLD["n_tail"]
    assert (o["t_tp_ps"], o["t_dp_ps"], o["t_all_ps"]) == (GOLD["t_tp_ps"], GOLD["t_dp_ps"], GOLD["t_all_ps"])


def _split_times(ids, P, hint, k, N, B, prof, tp_B, tp_prof, page=16, pool=100000, kv=0, tp_kv=0, pf=0, tp_pf=0):
    """Brute force of one split: the k longest on one TP instance (R25 prediction), the rest round robin;
    each iteration's T(b) plus kv ps per cached context token of the iteration and pf ps per prompt
    token it prefills (every prompt once, R27)."""
    order = sorted(range(len(ids)), key=lambda i: (-hint[i], ids[i]))
    top, rest = order[:k], order[k:]

    def sim(sel, B_, prof_, kv_, pf_):
        if not sel:
            return 0
        r = oracle.sched_sim(np.array([ids[i] for i in sel]), np.array([P[i] for i in sel]),
                             np.array([hint[i] for i in sel]), np.array([hint[i] for i in sel]), B_, page, pool,
                             profile=prof_)
        return int(r["time_ps"]) + kv_ * sum(it["sumctx"] for it in r["iters"]) + pf_ * sum(P[i] for i in sel)
    t_tp = sim(top, tp_B, tp_prof, tp_kv, tp_pf)
    t_dp = max((sim([rest[j] for j in range(s, len(rest), N)], B, prof, kv, pf) for s in range(N)), default=0)
    return t_tp, t_dp


@pytest.mark.parametrize("seed", range(8))
def test_oracle_tail_plan_bisection_against_every_split(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 14))
    ids = list(range(100, 100 + n))
    P = rng.integers(1, 40, n).tolist()
    hint = rng.integers(1, 30, n).tolist()
    prof, tp_prof = (3000, 40000, 8, 90000), (1800, 30000, 8, 60000)
    # the context and prefill terms (R27) on half the cases
    kv, tp_kv, pf, tp_pf = (0, 0, 0, 0) if seed < 4 else (700, 500, 3000, 1600)
    N, B, tp_B = 2, 3, 4
    o = oracle.tp_tail_plan(ids, P, hint, N, B, 16, 100000, prof, 2, tp_B, 100000, tp_prof, kv_ps=kv, tp_kv_ps=tp_kv,
                            pf_ps=pf, tp_pf_ps=tp_pf)
    times = [_split_times(ids, P, hint, k, N, B, prof, tp_B, tp_prof, kv=kv, tp_kv=tp_kv, pf=pf, tp_pf=tp_pf)
             for k in range(n + 1)]
    k = o["n_tail"]
    assert (o["t_tp_ps"], o["t_dp_ps"]) == times[k]
    # the rule: the first k with T_tp >= T_dp (when the two sides are monotone, as here), or k - 1
    first = next(j for j in range(n + 1) if times[j][0] >= times[j][1])
    assert k in (first, first - 1)
    if k == first - 1:
        assert max(times[k]) <= max(times[first])
    else:
        assert first == 0 or max(times[first - 1]) > max(times[first])


def test_product_tail_plan_equals_oracle():
    import paper_2504_15930_b200 as sgs
    g = GOLD
    for pol in ("round_robin", "skew"):
        o = _plan_oracle(g, pol)
        p = sgs.tp_tail_plan(g["ids"], g["P"], g["hint"], g["N"], g["B"], g["page"], g["pool"], g["profile"],
                             g["tp_size"], g["tp_B"], g["tp_pool"], g["tp_profile"], dispatch=pol)
        assert (p["n_tail"], p["t_tp_ps"], p["t_dp_ps"], p["t_all_ps"]) == \
            (o["n_tail"], o["t_tp_ps"], o["t_dp_ps"], o["t_all_ps"])
    rng = np.random.default_rng(7)
    for trial in range(8):
        n = int(rng.integers(1, 300))
        ids = rng.permutation(10 * n)[:n].astype(np.int64)
        P = rng.integers(16, 600, n)
        hint = np.minimum(rng.lognormal(5.5, 1.0, n).astype(np.int64) + 1, 4000)
        prof = (2_870_000, 1_200_000, 64, 20_000_000)
        tp_prof = (2_100_000, 900_000, 64, 14_000_000)
        N = int(rng.integers(1, 4))
        pol = ("round_robin", "skew")[trial % 2]
        kv, tp_kv, pf, tp_pf = (0, 0, 0, 0) if trial < 4 else (8850, 4700, 16_000_000, 8_500_000)
        o = oracle.tp_tail_plan(ids, P, hint, N, 64, 16, 3000, prof, 2, 64, 3000, tp_prof, policy=pol, kv_ps=kv,
                                tp_kv_ps=tp_kv, pf_ps=pf, tp_pf_ps=tp_pf)
        p = sgs.tp_tail_plan(ids, P, hint, N, 64, 16, 3000, prof, 2, 64, 3000, tp_prof, dispatch=pol, kv_ps=kv,
                             tp_kv_ps=tp_kv, pf_ps=pf, tp_pf_ps=tp_pf)
        assert (p["n_tail"], p["t_tp_ps"], p["t_dp_ps"], p["t_all_ps"]) == \
            (o["n_tail"], o["t_tp_ps"], o["t_dp_ps"], o["t_all_ps"]), (trial, pol)
