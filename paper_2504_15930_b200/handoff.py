"""Streamed hand-off of completions to a trainer (second half):
the paper's dynamic-batch pipelining (§4.1) against its strawman,
mini-batch pipelining, and no overlap.

sgs_step streams every completion out as soon as its sample finishes ("stream
generation ... samples are immediately sent to the training stage as soon as
completed").  These functions are the consumer side: given each
sample's completion time on the generation device and its token count, they
replay a trainer that processes mini-batches one after another, with
T_train(x) = c * max(tokens(x), S_sat) -- a mini-batch below the saturating
size S_sat costs as much as a saturating one ("the training stage can start as
soon as it receives enough samples to saturate the GPUs"; "if too
small, it harms training efficiency").  Pure host logic; the trainer
itself is out of scope, so its cost model is an input.

  batched   train once after the last completion (no overlap)
  minibatch M equal-count mini-batches in completion order, each handed over
            when its last sample completes
  dynamic   whenever the trainer is idle it takes every completed, untrained
            sample -- if they reach S_sat tokens, or generation has ended
            
"""
from __future__ import annotations

import numpy as np


def _train(tokens: float, c: float, s_sat: float) -> float:
    return c * max(tokens, s_sat)


def batched(t_done, tokens, c: float, s_sat: float) -> dict:
    t_gen = float(np.max(t_done))
    end = t_gen + _train(float(np.sum(tokens)), c, s_sat)
    return dict(policy="batched", end=end, minibatches=1, trainer_idle=t_gen, first_start=t_gen)


def minibatch(t_done, tokens, c: float, s_sat: float, M: int) -> dict:
    order = np.argsort(t_done, kind="stable")
    parts = np.array_split(order, M)
    free, idle, first = 0.0, 0.0, None
    for p in parts:
        if len(p) == 0:
            continue
        ready = float(np.max(t_done[p]))
        start = max(free, ready)
        idle += start - free
        first = start if first is None else first
        free = start + _train(float(np.sum(tokens[p])), c, s_sat)
    return dict(policy=f"minibatch{M}", end=free, minibatches=M, trainer_idle=idle, first_start=first)


def dynamic(t_done, tokens, c: float, s_sat: float) -> dict:
    order = np.argsort(t_done, kind="stable")
    td, tk = np.asarray(t_done, float)[order], np.asarray(tokens, float)[order]
    n = len(td)
    cum = np.concatenate([[0.0], np.cumsum(tk)])  # cum[j] = tokens of the first j completions
    i, free, idle, first, nmb = 0, 0.0, 0.0, None, 0
    while i < n:
        j = int(np.searchsorted(td, free, side="right"))  # completions by the time the trainer is free
        if j > i and (cum[j] - cum[i] >= s_sat or j == n):
            start = free
        else:  # wait for S_sat tokens past i, or for the last completion
            k = min(int(np.searchsorted(cum, cum[i] + s_sat, side="left")), n)
            start = max(free, td[max(k, i + 1) - 1])
        j = int(np.searchsorted(td, start, side="right"))  # take everything completed by then
        idle += start - free
        first = start if first is None else first
        free = start + _train(cum[j] - cum[i], c, s_sat)
        i, nmb = j, nmb + 1
    return dict(policy="dynamic", end=float(free), minibatches=nmb, trainer_idle=float(idle),
                first_start=None if first is None else float(first))
