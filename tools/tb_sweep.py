"""Config 5: decode-iteration time T(b) over batch x context on one B200, and the
paper's piecewise-linear model fitted to it (appendix; "PTL ... can be
profiled in advance").

For each context length, b prompts of that length are submitted with forced
lengths long enough for a few pure-decode iterations; the engine's per-
iteration device time (CUDA events) of the decode-only iterations is the
measured T(b, ctx).  The fit is done twice: by the product (sgs_fit_profile)
and by the oracle (oracle.tb_fit); both must agree.  The batch-merge lemma
T(x+y) < T(x) + T(y) holds on the fitted model iff t1 > 0.

    python tools/tb_sweep.py [--model qwen2.5-7b] [--ctx 1024 2048 ...] [--out profiles/tb_sweep.json]

Prompts are admitted without their prefill (SGS_F_SKIP_PREFILL): the decode
iterations read stale KV pages, which changes no timing, and the sweep costs
only its decode iterations.  A fit is flagged invalid when it breaks the
model's constraints 0 < k0 < k1, t1 > 0.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--ctx", type=int, nargs="*", default=[1024, 2048, 4096, 8192])
    ap.add_argument("--b", type=int, nargs="*",
                    default=[1, 2, 4, 8, 16, 32, 64, 96, 128, 160, 192, 224, 256, 320, 384, 512, 768, 1024])
    ap.add_argument("--decode-iters", type=int, default=6)
    ap.add_argument("--out", default="gpurun_out/tb_sweep.json")
    ap.add_argument("--prefill", action="store_true",
                    help="compute the prompts' prefill (default: SGS_F_SKIP_PREFILL -- decode timing is unchanged)")
    a = ap.parse_args()
    import torch
    import paper_2504_15930_b200 as sgs
    import oracle
    shape = workload.MODELS[a.model]
    bmax = max(a.b)
    out = {"model": a.model, "points": [], "fits": {}}
    flags = 0 if a.prefill else sgs.sgs.F_SKIP_PREFILL
    for ctx in a.ctx:
        # the largest b of the grid whose KV fits the pool decides max_batch
        probe = sgs.Instance(shape, 16, ctx + a.decode_iters + 2, device=0, max_prefill_tokens=max(16384, ctx),
                             weight_seed=5, trace=False, flags=flags)
        per = (ctx + a.decode_iters + 16) // 16 + 1
        fit_b = [b for b in a.b if b * per <= probe.n_pages * 0.97]
        probe.close()
        del probe
        torch.cuda.empty_cache()
        if not fit_b:
            continue
        inst = sgs.Instance(shape, max(fit_b), ctx + a.decode_iters + 2, device=0,
                            max_prefill_tokens=max(16384, ctx), weight_seed=5, trace=False, flags=flags)
        pool = inst.n_pages
        next_id = 0
        for b in fit_b:
            tr = workload.make_trace(b, ctx, a.decode_iters + 1, 0.0, a.decode_iters + 1, shape.vocab, seed=b,
                                     id_base=next_id)
            next_id += b
            n0 = len(inst.iter_log())
            inst.submit_trace(tr)
            inst.run()
            log = inst.iter_log()[n0:]
            dec = log[(log[:, 3] == 0) & (log[:, 1] == b)]  # decode-only iterations at full batch
            if len(dec) == 0:
                continue
            us = float(np.median(dec[:, 5]))
            out["points"].append({"ctx": ctx, "b": b, "T_us": us, "sumctx": int(np.median(dec[:, 4]))})
            print(json.dumps(out["points"][-1]), flush=True)
        inst.close()
        del inst
        torch.cuda.empty_cache()
        pts = [p for p in out["points"] if p["ctx"] == ctx]
        if len(pts) >= 4:
            bb = np.array([p["b"] for p in pts], float)
            tt = np.array([p["T_us"] * 1000.0 for p in pts], float)  # ns
            mine = sgs.fit_profile(bb, tt)
            ref = oracle.tb_fit(bb, tt)
            gain, x, y = oracle.min_merge_gain(ref["profile"], int(2 * max(bb)))
            out["fits"][str(ctx)] = {
                "valid": bool(ref["ok"] and ref["k0"] > 0 and ref["k1"] > ref["k0"] and ref["t1"] > 0),
                "violations": [n for n, bad in (("k0 <= 0", ref["k0"] <= 0), ("k1 <= k0", ref["k1"] <= ref["k0"]),
                                                ("t1 <= 0", ref["t1"] <= 0)) if bad],
                "product": {k: (float(v) if not isinstance(v, tuple) else list(v)) for k, v in mine.items()},
                "oracle": {k: (float(v) if not isinstance(v, (tuple, bool)) else (list(v) if isinstance(v, tuple)
                           else v)) for k, v in ref.items()},
                "profiles_equal": tuple(mine["profile"]) == tuple(ref["profile"]),
                "t1_ns": ref["t1"], "merge_lemma_holds": gain > 0, "min_merge_gain_ps": int(gain),
                "argmin_xy": [x, y]}
            print(json.dumps({"ctx": ctx, "fit": out["fits"][str(ctx)]}), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
