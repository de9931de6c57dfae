"""NEXT-4, streamed hand-off to a trainer (dynamic-batch pipelining)
on a measured generation timeline: one RL batch of a config runs on one B200;
every completion's time is the device time of the iterations up to its
finish_iter (the engine's per-iteration CUDA-event log); the consumer policies
of paper_2504_15930_b200.handoff replay a trainer that takes the streamed
completions -- no overlap, mini-batch pipelining with M fixed mini-batches
(the strawman), and dynamic batching.

Trainer stand-in (out of scope): T_train(x) = c * max(tokens(x),
S_sat), c set so that training the whole batch takes `ratio` x the generation
time, S_sat = the tokens of `sat` average samples.

    python tools/stream_handoff.py --config c2_7b --out gpurun_out/stream_handoff.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2_7b")
    ap.add_argument("--ratios", type=float, nargs="*", default=[0.5, 1.0, 2.0])
    ap.add_argument("--sat", type=int, default=32, help="saturating mini-batch, in average samples")
    ap.add_argument("--M", type=int, nargs="*", default=[4, 8, 16])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import paper_2504_15930_b200 as sgs
    from paper_2504_15930_b200 import handoff as H
    cfg = workload.CONFIGS[a.config]
    shape = workload.MODELS[cfg.model]
    tr = workload.make_trace(cfg.n_prompts, cfg.prompt_len, cfg.median_out, cfg.sigma, cfg.max_out, shape.vocab,
                             seed=cfg.seed)
    inst = sgs.Instance(shape, cfg.max_batch, cfg.prompt_len + cfg.max_out, device=0, weight_seed=11, trace=False)
    inst.submit_trace(tr)
    comps = inst.run()
    log = inst.iter_log()
    cum_s = np.cumsum(log[:, 5]) / 1e6  # device seconds at the end of each iteration
    t_of = {int(t): cum_s[k] for k, t in enumerate(log[:, 0])}
    P = {int(i): int(p) for i, p in zip(tr.ids, tr.prompt_len)}
    td = np.array([t_of[int(c["finish_iter"])] for c in comps])
    tk = np.array([P[c["id"]] + len(c["tokens"]) for c in comps], float)
    t_gen = float(td.max())
    s_sat = a.sat * tk.sum() / len(tk)
    out = {"config": a.config, "samples": len(comps), "t_gen_s": round(t_gen, 3), "tokens": int(tk.sum()),
           "completion_quantiles_s": {q: round(float(np.quantile(td, q / 100)), 2) for q in (10, 50, 90, 99, 100)},
           "S_sat_tokens": round(s_sat), "runs": []}
    for r in a.ratios:
        c = r * t_gen / tk.sum()
        res = [H.batched(td, tk, c, s_sat)] + [H.minibatch(td, tk, c, s_sat, m) for m in a.M] + \
              [H.dynamic(td, tk, c, s_sat)]
        row = {"train_over_gen": r, **{x["policy"]: {k: (round(v, 3) if isinstance(v, float) else v)
                                                     for k, v in x.items() if k != "policy"} for x in res}}
        out["runs"].append(row)
        print(json.dumps(row), flush=True)
    print(json.dumps({k: v for k, v in out.items() if k != "runs"}), flush=True)
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
