"""bench.py — generated tokens/s and RL-batch completion time of the Stream
Generation Service hot path (StreamRL, arXiv 2504.15930) on B200.

One step = one RL batch through every hot-path row: submit +
Alg. 2 dispatch, longest-first continuous batching (prefill + paged decode)
until every sample has streamed out, then the weight sync (NCCL broadcast from
rank 0 = the trainer proxy; a version bump at N = 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2_7b] [--impl reference]
N > 1: torchrun, one rank per GPU; weak scaling (512 prompts per GPU, the
whole N*512-prompt batch is submitted on every rank and Alg. 2 keeps each
rank's share; no data-path collective).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workload  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
# T(b) profiles (t0_ns, k0_ps, b_star, k1_ps) used by Alg. 2's Eq. 2; fitted by tools/tb_sweep.py
# (config 5) on B200 — profiles/r01_tb_sweep_{7b,14b,32b}.json (the ctx=2048 fits).  Only the
# dispatch (N > 1) reads them.
DEFAULT_PROFILES = {
    "qwen2.5-7b": (3491220, 29544576, 128, 38479949),
    "qwen2.5-14b": (5987575, 73237116, 160, 71301394),
    "qwen2.5-32b": (11988370, 88930482, 32, 107212340),
    "tiny": (200, 100, 64, 400),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["_source"] = "measured"
        return d
    d = dict(PEAKS_FALLBACK)
    d["_source"] = "fallback"
    return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ reference arm (the CPU oracle)
def run_reference(args):
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return
    import oracle
    cfg = workload.CONFIGS[args.config]
    shape = workload.MODELS[cfg.model]
    res = cpu_oracle_sample(shape, steps=args.steps, warmup=args.warmup)
    line = {"metric": "generated_tokens_per_s", "value": res["value"], "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config}: {cfg.model}-shaped, {cfg.n_prompts} prompts x {cfg.prompt_len}"},
            "cpu_baseline": {"value": res["value"], "unit": "tokens/s", "cores": res["cores"], "kind": "oracle",
                             "sample": res["sample"]},
            "e2e": {"value": res["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_oracle_sample(shape, steps=1, warmup=0, T=8):
    """Time the oracle decoder (as it stands) on a bounded sample of the workload:
    T positions of one sample through layer subsets of the full model, extrapolated
    to all layers (t_full = t_lmhead + L * (t_1layer - t_lmhead))."""
    import dataclasses
    import oracle
    toks = np.random.default_rng(0).integers(0, shape.vocab, size=T).astype(np.int32)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        oracle.decoder_forward(dataclasses.replace(shape, n_layers=0), 1, toks, T - 1)
        t1 = time.perf_counter()
        oracle.decoder_forward(dataclasses.replace(shape, n_layers=1), 1, toks, T - 1)
        t2 = time.perf_counter()
        if i >= warmup:
            t_lm, t_layer = t1 - t0, (t2 - t1) - (t1 - t0)
            times.append(t_lm + shape.n_layers * max(t_layer, 0.0))
    t_full = statistics.median(times)
    return {"value": T / t_full, "ms_per_step": 1e3 * t_full, "cores": os.cpu_count(),
            "sample": f"{T} teacher-forced positions of one sample; 0- and 1-layer {shape.name} runs timed, "
                      f"extrapolated to {shape.n_layers} layers (fp64, OpenMP, weights regenerated per call)"}


def batch_roofline(rows, shape, bw_gbs, tflops):
    """Roofline time of the executed schedule: every iteration of the
    iteration log priced at max(bytes/HBM, flops/bf16) per GEMM, plus the KV bytes
    of decode attention and the causal flops of prefill attention.  Prefill and
    decode rows of a mixed iteration are separate passes, as executed.  Rows:
    (t, b, admitted, prefill tokens, sum ctx, device us)."""
    L, d, nq, nkv, hd, f, V = (shape.n_layers, shape.d_model, shape.n_q_heads, shape.n_kv_heads, shape.head_dim,
                               shape.d_ffn, shape.vocab)
    BW, F = bw_gbs * 1e9, tflops * 1e12
    gemms = [((nq + 2 * nkv) * hd, d), (d, nq * hd), (2 * f, d), (d, f)]

    def gemm_t(T):
        return L * sum(max(N * K * 2 / BW, 2.0 * N * K * T / F) for N, K in gemms) + \
            max(V * d * 2 / BW, 2.0 * V * d * min(T, 1 << 30) / F)

    kv_bytes_per_token = 2 * nkv * hd * 2 * L
    total = 0.0
    for _t, b, adm, pf, sumctx, _us in rows:
        dec = b - adm
        if pf > 0 and adm > 0:
            lp = pf / adm
            attn = adm * 4.0 * nq * hd * (lp * (lp + 1) / 2) * L
            # prefill GEMMs over the prompt tokens; the LM head only for the last token of each prompt
            total += L * sum(max(N * K * 2 / BW, 2.0 * N * K * pf / F) for N, K in gemms) + attn / F + \
                max(V * d * 2 / BW, 2.0 * V * d * adm / F)
        if dec > 0:
            total += gemm_t(dec) + (sumctx - pf) * kv_bytes_per_token / BW
    return total


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--weight-sync", choices=["sync", "async"], default="sync",
                    help="sync: broadcast at the batch boundary; async: overlapped with generation (staleness 1)")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2_7b")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--prompts-per-gpu", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--max-out", type=int, default=None, help="cap forced lengths (profiling runs only)")
    ap.add_argument("--no-kernel-timing", action="store_true")
    ap.add_argument("--iter-log", default=None, help="write the per-iteration log (t,b,adm,pf_tok,sumctx,us) as .npy")
    ap.add_argument("--dispatch", default="skew", choices=["skew", "random", "round_robin"])
    ap.add_argument("--strong", action="store_true", help="fixed global batch (cfg.n_prompts) instead of per GPU")
    ap.add_argument("--profile", default=None, help="T(b) profile t0_ns,k0_ps,b_star,k1_ps for Alg. 2")
    ap.add_argument("--hint-noise", type=float, default=None, help="ranker noise sigma (None: oracle hints)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_2504_15930_b200 as sgs

    world, rank, local = dist_env()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", local))
        pg = dist
    cfg = workload.CONFIGS[args.config]
    if args.max_out:
        import dataclasses
        cfg = dataclasses.replace(cfg, max_out=args.max_out, median_out=min(cfg.median_out, args.max_out // 4))
    shape = workload.MODELS[cfg.model]
    per_gpu = args.prompts_per_gpu or cfg.n_prompts
    n_total = cfg.n_prompts if args.strong else per_gpu * world
    max_ctx = cfg.prompt_len + cfg.max_out

    prof = tuple(int(x) for x in args.profile.split(",")) if args.profile else DEFAULT_PROFILES.get(cfg.model)
    inst = sgs.Instance(shape, cfg.max_batch, max_ctx, device=local, n_instances=world, instance_rank=rank,
                        weight_seed=cfg.seed,
                        flags=(0 if args.no_kernel_timing else sgs.sgs.F_KERNEL_TIMING) |
                        (sgs.sgs.F_SHADOW_WEIGHTS if args.weight_sync == "async" else 0),
                        dispatch=args.dispatch, profile=prof, sample_seed=cfg.seed)
    peaks0 = load_peaks()
    inst.set_roofline(peaks0["hbm_gbs"], peaks0["bf16_tflops_sustained"])
    if world > 1:
        uid = [sgs.comm_unique_id() if rank == 0 else None]
        pg.broadcast_object_list(uid, src=0)
        inst.comm_init(uid[0], rank, world)

    def make_batch(step):
        # a fresh RL batch per step: same length distribution, new ids and prompts
        return workload.make_trace(n_total, cfg.prompt_len, cfg.median_out, cfg.sigma, cfg.max_out, shape.vocab,
                                   seed=cfg.seed + 1000 * step, id_base=step * 1_000_000, hint_noise=args.hint_noise)

    stream = inst.stream

    def one_step(step):
        tr = make_batch(step)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = inst.kernel_launches()
        io0 = inst.io_bytes()
        t0 = time.perf_counter()
        ev0.record(stream)
        mine = inst.submit_trace(tr)
        if args.weight_sync == "async":
            # fully-async pipelining: the next weights are staged and
            # broadcast on a side stream while this batch generates; committed at the boundary
            if rank == 0:
                inst.stage_weights_seed(cfg.seed + step + 1)
            inst.update_weights_begin(0)
            comps = inst.run()
            inst.update_weights_commit()
        else:
            comps = inst.run()
            # weight sync at the RL-step boundary: rank 0 is the trainer proxy
            if rank == 0:
                inst.load_weights_seed(cfg.seed + step + 1)
            inst.update_weights(0)
        ev1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        io1 = inst.io_bytes()
        gen_tokens = int(sum(len(c["tokens"]) for c in comps))
        assert len(comps) == mine
        prompt_bytes = int(tr.tokens.nbytes)
        return dict(dev_s=ev0.elapsed_time(ev1) / 1e3, wall_s=wall, tokens=gen_tokens, samples=len(comps),
                    launches=inst.kernel_launches() - launches0,
                    h2d=io1[0] - io0[0] + prompt_bytes, d2h=io1[1] - io0[1])

    for w in range(args.warmup):
        one_step(w)
    for cls in range(4):
        inst.kernel_stats(cls, reset=True)
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    results = []
    log0 = len(inst.iter_log())
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            results.append(one_step(args.warmup + k))
    if pg:
        pg.barrier()
    torch.cuda.synchronize()

    dev_s = sum(r["dev_s"] for r in results)
    wall_s = sum(r["wall_s"] for r in results)
    tokens = sum(r["tokens"] for r in results)
    stats = {cls: inst.kernel_stats(cls) for cls in range(4)}
    timed_rows = inst.iter_log()[log0:]
    if args.iter_log and rank == 0:
        np.save(args.iter_log, inst.iter_log())
    if pg:
        t = torch.tensor([dev_s, wall_s, float(tokens)], dtype=torch.float64)
        mx = t.clone()
        pg.all_reduce(mx, op=pg.ReduceOp.MAX)
        sm = t.clone()
        pg.all_reduce(sm, op=pg.ReduceOp.SUM)
        dev_s, wall_s, tokens = float(mx[0]), float(mx[1]), int(sm[2])
    if rank != 0:
        pg.destroy_process_group()
        return
    peaks = load_peaks()
    # whole-step roofline of this rank's executed schedule, vs its measured device time
    t_roof = batch_roofline(timed_rows, shape, peaks["hbm_gbs"], peaks["bf16_tflops_sustained"])
    t_meas = float(sum(r[5] for r in timed_rows)) / 1e6
    batch_roof = {"roofline_s": round(t_roof, 3), "measured_s": round(t_meas, 3),
                  "frac": round(t_roof / t_meas, 4) if t_meas > 0 else None,
                  "definition": "sum over the executed iterations of (per GEMM max(weight bytes/HBM, "
                                "flops/bf16 sustained) + KV bytes/HBM + prefill attention flops/bf16); "
                                "measured = sum of the iterations' device time (this rank)"}
    roof, other = None, None
    if stats[3]["ms"] > 0:
        # per-kernel CUDA events are recorded on a 1-in-32 sample of the timed
        # iterations (events between kernels would defeat the PDL overlap);
        # shares are relative to the device time of those same iterations
        names = {0: "decode_attention (K1+K2, paged split-K)", 1: "tcgen05 GEMMs (QKV/O/gate-up/down/LM head)"}
        dom = max((0, 1), key=lambda c: stats[c]["ms"])
        st = stats[dom]
        # The GEMM class spans both regimes (weight streaming at small b, tensor
        # bound at b ~ 256 and in prefill): each timed launch's roofline time is
        # max(bytes / HBM, flops / sustained bf16); frac = sum(roofline) / sum(measured).
        roof_ms = inst.kernel_roofline_ms(dom)
        frac = roof_ms / st["ms"]
        hbm_share = st["bytes"] / (peaks["hbm_gbs"] * 1e6) / max(roof_ms, 1e-9)
        bound = "hbm" if hbm_share >= 0.5 else "tensor"
        if bound == "hbm":
            achieved, peak, unit = st["bytes"] / (st["ms"] / 1e3) / 1e9, peaks["hbm_gbs"], "GB/s"
        else:
            achieved, peak, unit = st["flops"] / (st["ms"] / 1e3) / 1e12, peaks["bf16_tflops_sustained"], "TFLOP/s"
        roof = {"kernel": names[dom], "bound": bound, "achieved": round(achieved, 1), "peak": peak, "unit": unit,
                "frac": round(frac, 4), "frac_definition": "sum over timed launches of max(bytes/HBM, flops/bf16 "
                "sustained) / measured time", "traffic": None,
                "traffic_source": "per-shape ncu --set full captures in profiles/r01c_ncu_full_summary.csv "
                                  "(one number for the mixed-shape GEMM class would not be per launch): decode "
                                  "GEMMs read their algorithmic bytes within 3% (O-proj split-K +13%); the "
                                  "prefill gate_up at T=8192 reads its weights ~3.4x (1.13 GB vs 0.33 GB) while "
                                  "tensor-bound at 1.43 PF/s", "peak_source": peaks["_source"],
                "launches_sampled": st["launches"], "share_of_step": round(st["ms"] / stats[3]["ms"], 4),
                "timing": "CUDA events on the engine stream, 1 in 32 iterations of the timed region"}
        other = {("decode_attention" if c == 0 else "gemm" if c == 1 else "prefill_attention"):
                 {"ms_sampled": round(stats[c]["ms"], 1), "share": round(stats[c]["ms"] / stats[3]["ms"], 4),
                  "roofline_frac": round(inst.kernel_roofline_ms(c) / max(stats[c]["ms"], 1e-9), 4),
                  "GB/s": round(stats[c]["bytes"] / max(stats[c]["ms"], 1e-9) / 1e6, 1),
                  "TFLOP/s": round(stats[c]["flops"] / max(stats[c]["ms"], 1e-9) / 1e9, 1)} for c in range(3)}
    line = {
        "metric": "generated_tokens_per_s",
        "value": round(tokens / dev_s, 1),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * dev_s / args.steps, 1),
        "rl_batch_completion_s": round(dev_s / args.steps, 3),
        "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg.model}-shaped random-init bf16 decoder, {per_gpu} prompts/GPU "
                               f"x {cfg.prompt_len} tokens, lognormal(median {cfg.median_out}, sigma {cfg.sigma}) "
                               f"forced lengths <= {cfg.max_out}, B={cfg.max_batch}, longest-first, Alg. 2 dispatch",
                   "prompts_total": n_total, "global_batch": n_total, "parallelism": f"dp{world}",
                   "dispatch": args.dispatch, "weight_sync": args.weight_sync,
                   "hints": "oracle (= forced)" if args.hint_noise is None else
                   f"noisy sigma {args.hint_noise}", "profile": list(prof) if prof else None,
                   "l2": "inputs larger than L2 (weights 15 GB, KV pool > 100 GB)"},
        "e2e": {"value": round(tokens / wall_s, 1), "unit": "tokens/s",
                "h2d_bytes_per_step": int(statistics.mean(r["h2d"] for r in results)),
                "d2h_bytes_per_step": int(statistics.mean(r["d2h"] for r in results))},
        "gpu_launches": int(sum(r["launches"] for r in results)),
        "roofline": roof,
        "batch_roofline": batch_roof,
        "kernels": other,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        cb = cpu_oracle_sample(shape)
        line["cpu_baseline"] = {"value": round(cb["value"], 4), "unit": "tokens/s", "cores": cb["cores"],
                                "kind": "oracle", "sample": cb["sample"]}
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
