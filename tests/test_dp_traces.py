"""Schedules of the multi-GPU runs (configs 3 and 4, tools/dp_experiment.py
--dump-trace) against the oracle: for every dumped instance, the oracle's
Alg. 2 dispatch of the full batch selects that instance's samples
and the oracle's scheduler simulation of them must equal the
GPU run's iteration and per-sample traces bit for bit.  Runs when
SGS_TRACE_DIR points at the dumps (the GPU runs that write them); skipped
otherwise."""
import glob
import os

import numpy as np
import pytest

import oracle

DIR = os.environ.get("SGS_TRACE_DIR")
FILES = sorted(glob.glob(os.path.join(DIR, "*.npz"))) if DIR else []


@pytest.mark.skipif(not FILES, reason="no dumped multi-GPU traces (set SGS_TRACE_DIR)")
@pytest.mark.parametrize("path", FILES)
def test_dp_trace_matches_oracle(path):
    z = np.load(path)
    policy = str(z["policy"])
    N, me = int(z["N"]), int(z["instance"])
    ids, P, d, hint = z["ids"], z["P"], z["d"], z["hint"]
    if policy == "skew":
        disp = oracle.dispatch(ids, P, hint, N, int(z["B"]), int(z["page"]), int(z["pool"]), tuple(z["profile"]),
                               alpha_pct=int(z["alpha"]), score_max=int(z["score"]))
        inst = disp["instance"]
    elif policy == "round_robin":
        order = sorted(range(len(ids)), key=lambda i: (-int(hint[i]), int(ids[i])))
        inst = np.zeros(len(ids), np.int64)
        for j, i in enumerate(order):
            inst[i] = j % N
    else:
        pytest.skip("the random policy's permutation has no oracle twin")
    sel = np.flatnonzero(inst == me)
    o = oracle.sched_sim(ids[sel], P[sel], d[sel], hint[sel], int(z["B"]), int(z["page"]), int(z["pool"]))
    assert np.array_equal(z["iter_blob"], o["iter_blob"])
    assert np.array_equal(z["sample_blob"], o["sample_blob"])
