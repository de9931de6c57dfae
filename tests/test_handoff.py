"""Streamed hand-off to a trainer (NEXT-4): the consumer policies
of paper_2504_15930_b200.handoff on hand-derived timelines."""
import numpy as np

from paper_2504_15930_b200 import handoff as H


def test_hand_timeline():
    # completions at 1, 2, 3, 10 (10 tokens each), c = 0.1 per token, S_sat = 20 tokens
    td, tk = np.array([1.0, 2.0, 3.0, 10.0]), np.full(4, 10.0)
    b = H.batched(td, tk, 0.1, 20)
    assert (b["end"], b["trainer_idle"]) == (14.0, 10.0)  # 10 + 40 tokens x 0.1
    m = H.minibatch(td, tk, 0.1, 20, 2)
    assert (m["end"], m["trainer_idle"], m["first_start"]) == (12.0, 8.0, 2.0)  # {1,2} at 2 -> 4; {3,10} at 10 -> 12
    d = H.dynamic(td, tk, 0.1, 20)
    assert (d["end"], d["minibatches"], d["first_start"]) == (12.0, 2, 2.0)


def test_dynamic_absorbs_the_long_tail():
    # a long tail: 8 short samples done by t = 4, one long sample at t = 20.  Four fixed
    # mini-batches put the long sample's slow neighbours behind it; the dynamic consumer
    # trains everything that is done, then only the tail
    td = np.array([0.5, 1, 1.5, 2, 2.5, 3, 3.5, 4, 20.0])
    tk = np.array([10, 10, 10, 10, 10, 10, 10, 10, 200.0])
    c, s_sat = 0.05, 20
    m = H.minibatch(td, tk, c, s_sat, 3)  # {0.5,1,1.5} {2,2.5,3} {3.5,4,20}
    d = H.dynamic(td, tk, c, s_sat)
    b = H.batched(td, tk, c, s_sat)
    assert d["end"] <= m["end"] <= b["end"]
    assert d["end"] == 20.0 + 200 * c  # only the tail sample is left at its completion


def test_every_sample_trained_once():
    rng = np.random.default_rng(3)
    td = np.sort(rng.exponential(5.0, 200))
    tk = rng.integers(100, 4000, 200).astype(float)
    c, s_sat = 1e-3, 20000.0
    d = H.dynamic(td, tk, c, s_sat)
    # the trainer's busy time covers every token once (mini-batches below S_sat cost S_sat)
    assert d["end"] - d["trainer_idle"] >= c * tk.sum() - 1e-9
    assert d["end"] >= td.max() + c * min(s_sat, tk[-1:].sum()) - 1e-9
