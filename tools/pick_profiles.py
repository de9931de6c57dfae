"""Dispatch profiles (Eq. 2's PTL(BS)) from the config-5 T(b)
sweeps: per workload config, the valid fit (R24: 0 < k0 < k1, t1 > 0) at the
grid context nearest (in log scale) to the workload's mean context
P + E[d]/2 (reading R23; E[d] of the clamped lognormal by sampling).

    python tools/pick_profiles.py profiles/r02/tb_sweep_qwen2.5-*.json
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload  # noqa: E402


def main():
    fits = {}
    for p in sys.argv[1:]:
        d = json.load(open(p))
        fits[d["model"]] = d["fits"]
    for name, cfg in workload.CONFIGS.items():
        if cfg.model not in fits:
            continue
        d = workload.lognormal_lengths(200_000, cfg.median_out, cfg.sigma, cfg.max_out, seed=1)
        ctx = cfg.prompt_len + float(d.mean()) / 2
        cand = sorted(fits[cfg.model].items(), key=lambda kv: abs(math.log(int(kv[0]) / ctx)))
        for c, f in cand:
            if f["valid"]:
                print(json.dumps({"config": name, "model": cfg.model, "mean_ctx": round(ctx), "fit_ctx": int(c),
                                  "profile": f["oracle"]["profile"], "t1_ns": round(f["t1_ns"])}))
                break


if __name__ == "__main__":
    main()
