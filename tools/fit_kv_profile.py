"""Fit T(b, C) = T(b) + kv * C to T(b) sweeps at several contexts (C = the
iteration's cached context tokens = b * ctx in a sweep): kv by least squares
on the context dependence at equal b, then the paper's hinge profile T(b) on
T - kv * C (sgs_fit_profile).  Used for sgs_tp_tail_plan's kv terms (R27).

    python tools/fit_kv_profile.py FILE [--exchange p2p] [--bmax 256]
"""
import argparse
import collections
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def fit(path, exchange=None, bmax=256):
    import paper_2504_15930_b200 as sgs
    pts = [p for p in json.load(open(path))["points"] if (exchange is None or p.get("exchange") == exchange)
           and p["b"] <= bmax]
    T = lambda p: p.get("T_us", p.get("T_us_tp2")) * 1e6  # ps
    by_b = collections.defaultdict(list)
    for p in pts:
        by_b[p["b"]].append((p["b"] * p["ctx"], T(p)))
    # kv: pooled within-b regression of T on C
    num = den = 0.0
    for b, v in by_b.items():
        if len(v) < 2:
            continue
        c = np.array([x[0] for x in v], float)
        t = np.array([x[1] for x in v], float)
        num += float(((c - c.mean()) * (t - t.mean())).sum())
        den += float(((c - c.mean()) ** 2).sum())
    kv = num / den if den > 0 else 0.0
    bs = np.array([p["b"] for p in pts], float)
    t0 = np.array([T(p) - kv * p["b"] * p["ctx"] for p in pts], float) / 1e3  # ns
    prof = sgs.fit_profile(bs, t0)["profile"]
    return tuple(int(x) for x in prof), int(round(kv))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("path", nargs="+")
    ap.add_argument("--exchange", default=None)
    ap.add_argument("--bmax", type=int, default=256)
    a = ap.parse_args()
    import tempfile
    pts = []
    for f in a.path:
        pts += json.load(open(f))["points"]
    tmp = tempfile.NamedTemporaryFile("w", suffix=".json", delete=False)
    json.dump({"points": pts}, tmp)
    tmp.close()
    print(json.dumps(dict(zip(("profile", "kv_ps"), fit(tmp.name, a.exchange, a.bmax)))))
