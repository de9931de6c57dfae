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
# T(b) profiles (t0_ns, k0_ps, b_star, k1_ps) used by Alg. 2's Eq. 2: the r02 config-5 sweeps on the
# current kernels (profiles/r02/tb_sweep_*.json, tools/tb_sweep.py), each the valid fit (R24) at the
# grid context nearest the workload's mean context (R23; tools/pick_profiles.py).  Only the dispatch
# (N > 1) reads them.
DEFAULT_PROFILES = {
    "qwen2.5-7b": (2737741, 15064935, 192, 19922457),     # ctx 1024
    "qwen2.5-14b": (5245282, 39388098, 128, 61477016),    # ctx 1024
    "qwen2.5-32b": (11387520, 59009897, 16, 99386761),    # ctx 2048
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
    cfg = workload.CONFIGS[args.config]
    shape = workload.MODELS[cfg.model]
    samples = [cpu_oracle_sample(shape, cfg, warm=(i == 0)) for i in range(args.warmup + args.steps)][args.warmup:]
    ms = [s["ms"] for s in samples]
    tok = sum(s["tokens"] for s in samples)
    value = tok / (sum(ms) / 1e3)
    line = {"metric": "generated_tokens_per_s", "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(ms),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config}: {cfg.model}-shaped, {cfg.n_prompts} prompts x {cfg.prompt_len}"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": samples[0]["cores"], "kind": "oracle",
                             "sample": samples[0]["sample"]},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_oracle_sample(shape, cfg, warm=True, P0=4, K=12):
    """One bounded, measured step of the oracle decoder (as it stands: fp64,
    OpenMP, no KV cache, no batching) on this workload's model at b = 1: one
    teacher-forced forward over P0 prompt + K positions, whose K + 1 logits rows
    are the sample's generated tokens (the prefill of the P0 prefix is inside
    the timed step).  Weights are built once (oracle.weight_cache memoises the
    generator's output, same values), so the step times the decoder arithmetic.
    When the fp32 weight copy would not fit in 40% of host RAM, the step runs
    0- and 1-layer instances of the shape and extrapolates linearly to L layers
    (said in the sample text)."""
    import dataclasses
    import oracle
    oracle.weight_cache(True)
    toks = np.random.default_rng(0).integers(0, shape.vocab, size=P0 + K).astype(np.int32)
    ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    full = 4.0 * shape.params() <= 0.4 * ram and os.environ.get("SGS_BENCH_CPU_FULL", "1") == "1"
    if full and os.environ.get("SGS_BENCH_CPU_CHILD") != "1":
        # the full model in a child process under a time budget: weight building
        # on a slow or memory-tight host must not stall the bench; past the
        # budget the layer extrapolation below runs instead
        try:
            env = dict(os.environ, SGS_BENCH_CPU_CHILD="1")
            code = ("import json, bench, workload; "
                    f"print(json.dumps(bench.cpu_oracle_sample(workload.MODELS['{shape.name}'], "
                    f"workload.CONFIGS['{cfg.name}'], {warm}, {P0}, {K})))")
            r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                               timeout=float(os.environ.get("SGS_BENCH_CPU_BUDGET_S", "300")))
            if r.returncode == 0:
                return json.loads(r.stdout.strip().splitlines()[-1])
        except subprocess.TimeoutExpired:
            pass
        full = False
    if full:
        if warm:
            oracle.decoder_forward(shape, 1, toks[:2], 1)  # builds (caches) the weights, untimed
        t0 = time.perf_counter()
        oracle.decoder_forward(shape, 1, toks, P0 - 1)
        t = time.perf_counter() - t0
        how = f"full {shape.n_layers}-layer model"
    else:
        ts = []
        for nl in (0, 1):
            sh = dataclasses.replace(shape, n_layers=nl)
            if warm:
                oracle.decoder_forward(sh, 1, toks[:2], 1)
            t0 = time.perf_counter()
            oracle.decoder_forward(sh, 1, toks, P0 - 1)
            ts.append(time.perf_counter() - t0)
        t = ts[0] + shape.n_layers * max(ts[1] - ts[0], 0.0)
        how = f"0- and 1-layer instances extrapolated to {shape.n_layers} layers (the full model did not fit the RAM or time budget)"
    n = K + 1
    return {"tokens": n, "ms": 1e3 * t, "per_token_s": t / n, "cores": os.cpu_count(),
            "b_B_iteration_s": t / n * cfg.max_batch,
            "sample": f"one teacher-forced forward of {P0}+{K} positions of {shape.name} at b=1 ({how}; "
                      f"{n} logits rows = generated tokens, prefix prefill included), weights built once "
                      f"(memoised), fp64, OpenMP on {os.cpu_count()} cores; the oracle has no batching: a "
                      f"b={cfg.max_batch} iteration is {cfg.max_batch} such samples"}


def host_plane_timing(tr, cfg, pool, shape):
    """Scheduler + dispatch on the host: the oracle (sched_sim + dispatch) and the
    product's control plane alone (null-device mode: the same C++ scheduler,
    page allocator and Alg. 2 the GPU run uses, no kernels), us per iteration."""
    import oracle
    import paper_2504_15930_b200 as sgs
    t0 = time.perf_counter()
    oracle.dispatch(tr.ids, tr.prompt_len, tr.hint, 1, cfg.max_batch, cfg.page_size, pool,
                    DEFAULT_PROFILES.get(cfg.model, (1, 1, 1, 1)))
    r = oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, cfg.max_batch, cfg.page_size, pool)
    t_or = time.perf_counter() - t0
    inst = sgs.Instance(shape, cfg.max_batch, cfg.prompt_len + cfg.max_out, device=None, n_pages=pool, trace=False)
    t0 = time.perf_counter()
    inst.submit_trace(tr)
    inst.run()
    t_pr = time.perf_counter() - t0
    n = r["n_iters"]
    return {"iterations": n, "oracle_us_per_iter": round(1e6 * t_or / n, 2),
            "product_us_per_iter": round(1e6 * t_pr / n, 2),
            "note": "single-threaded host work per iteration; the product number includes the ctypes step loop"}


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


CLASSES = {0: "decode_attention", 1: "decode_gemm", 2: "prefill_attention", 4: "prefill_gemm", 5: "decode_other"}
CLASS_DESC = {0: "decode attention (K1+K2, paged split-K, merge in-kernel)",
              1: "decode tcgen05 GEMMs (QKV / O / gate-up+SwiGLU / down / LM head)",
              2: "prefill attention (causal)", 4: "prefill tcgen05 GEMMs",
              5: "decode RMSNorm / RoPE+append / embedding / sampler"}
NCU_WINDOW = os.path.join(ROOT, "profiles", "r02_ncu_windows.json")
TIMELINE_REF = os.path.join(ROOT, "profiles", "r02", "bench_timeline_shares.json")


def kernel_roofline(inst, stats, peaks, n_iters, dev_s):
    """Per-class device time from CUDA events on the engine stream, recorded on
    ~1 in 64 timed iterations chosen by a hash of the iteration counter (so the
    sample is not aliased with the schedule).  The classes are disjoint
    intervals of the sampled iterations (prefill runs sequentially in them), so
    their sum cannot exceed the sampled iterations' device time: asserted.
    Events between kernels remove the PDL overlap, so sampled iterations run
    slower than production ones; shares (class / sampled iteration time) are
    what carries over, reported next to the uninstrumented ncu launch window."""
    it = stats[3]
    if it["ms"] <= 0:
        return None, None
    tot = sum(stats[c]["ms"] for c in CLASSES)
    assert tot <= 1.001 * it["ms"], f"kernel classes {tot:.1f} ms exceed the sampled iterations' {it['ms']:.1f} ms"
    kernels = {}
    for c, name in CLASSES.items():
        st = stats[c]
        kernels[name] = {"ms_sampled": round(st["ms"], 1), "launches_sampled": st["launches"],
                         "share": round(st["ms"] / it["ms"], 4),
                         "est_s_per_step_production": round(st["ms"] / it["ms"] * dev_s, 3),
                         "roofline_frac": round(inst.kernel_roofline_ms(c) / max(st["ms"], 1e-9), 4),
                         "GB/s": round(st["bytes"] / max(st["ms"], 1e-9) / 1e6, 1),
                         "TFLOP/s": round(st["flops"] / max(st["ms"], 1e-9) / 1e9, 1)}
    kernels["_sampled_iterations"] = {"n": it["launches"], "of": n_iters, "ms": round(it["ms"], 1),
                                      "classes_ms": round(tot, 1),
                                      "instrumentation_slowdown": round(it["ms"] * n_iters / max(it["launches"], 1)
                                                                        / (1e3 * dev_s), 3)}
    # the same shares within the b >= 129 and the b <= 32 iterations (compare with the ncu windows)
    for ph, tag in ((1, "b>=129"), (2, "b<=32")):
        itp = stats[3 + 6 * ph]
        if itp["ms"] > 0:
            kernels[f"_shares_{tag}"] = {"iterations": itp["launches"],
                                         **{name: round(stats[c + 6 * ph]["ms"] / itp["ms"], 4)
                                            for c, name in CLASSES.items()}}
    if os.path.exists(NCU_WINDOW):
        kernels["_ncu_windows"] = json.load(open(NCU_WINDOW))
    dom = max(CLASSES, key=lambda c: stats[c]["ms"])
    st = stats[dom]
    roof_ms = inst.kernel_roofline_ms(dom)
    hbm_share = st["bytes"] / (peaks["hbm_gbs"] * 1e6) / max(roof_ms, 1e-9)
    bound = "hbm" if hbm_share >= 0.5 else "tensor"
    if bound == "hbm":
        achieved, peak, unit = st["bytes"] / (st["ms"] / 1e3) / 1e9, peaks["hbm_gbs"], "GB/s"
    else:
        achieved, peak, unit = st["flops"] / (st["ms"] / 1e3) / 1e12, peaks["bf16_tflops_sustained"], "TFLOP/s"
    roof = {"kernel": CLASS_DESC[dom], "class": CLASSES[dom], "bound": bound, "achieved": round(achieved, 1),
            "peak": peak, "unit": unit, "frac": round(roof_ms / st["ms"], 4),
            "frac_definition": "sum over the class's sampled launches of max(algorithmic bytes/HBM, flops/bf16 "
                               "sustained) / their measured time (CUDA events on the engine stream)",
            "traffic": None, "traffic_source": None,
            "peak_source": peaks["_source"], "share_of_step": round(st["ms"] / it["ms"], 4)}
    # DRAM bytes per launch: ncu's dram__bytes_read + write over the 7B decode
    # GEMM shapes (one cold launch each, tools/gemm_traffic.py) relative to
    # their algorithmic bytes, applied to this class's algorithmic bytes per launch
    traffic_file = os.path.join(ROOT, "profiles", "r02", "ncu_gemm_traffic.json")
    if CLASSES[dom] == "decode_gemm" and os.path.exists(traffic_file) and st["launches"] > 0:
        cases = json.load(open(traffic_file))["cases"]
        ratio = sum(c["dram_bytes"] for c in cases) / sum(c["alg_bytes"] for c in cases)
        roof["traffic"] = round(ratio * st["bytes"] / st["launches"])
        roof["traffic_alg"] = round(st["bytes"] / st["launches"])
        roof["traffic_over_alg"] = round(ratio, 3)
        roof["traffic_source"] = ("ncu dram__bytes_read.sum + dram__bytes_write.sum / algorithmic bytes over the "
                                  "decode GEMM shapes (profiles/r02/ncu_gemm_traffic.json) x this class's "
                                  "algorithmic bytes per sampled launch")
    return roof, kernels


def timeline_shares(inst, sgs, tr, cfg, shape, width=32):
    """Uninstrumented class shares (CUPTI kernel timestamps through torch.profiler:
    no CUDA events between kernels) over two windows of `width` iterations of one
    more RL batch -- at 5% of its iterations (the b = B phase) and at 75% (the
    long tail) -- to set beside the event-sampled shares.  A kernel's share is its
    critical-path increment (its end minus every earlier end), so the prefill
    stream's kernels that overlap decode count only where they extend the
    iteration.  The iteration count comes from the product's scheduler in
    null-device mode (the same host code)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    dry = sgs.Instance(shape, cfg.max_batch, cfg.prompt_len + cfg.max_out, device=None, n_pages=inst.n_pages,
                       trace=False)
    dry.submit_trace(tr)
    n_it = 0
    while True:
        q, a = dry.pending()
        if q == 0 and a == 0:
            break
        dry.step()
        n_it += 1
    dry.close()
    windows = [(int(0.05 * n_it), "b_large"), (int(0.75 * n_it), "tail")]
    inst.submit_trace(tr)
    it, out = 0, {}
    while True:
        q, a = inst.pending()
        if q == 0 and a == 0:
            break
        w = next((w for w in windows if w[0] == it), None)
        if not w:
            inst.step()
            it += 1
            continue
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(width):
                inst.step()
                it += 1
            torch.cuda.synchronize()
        ev = []
        for e in prof.profiler.kineto_results.events():
            if e.device_type().name != "CUDA" or e.name().startswith(("Memcpy", "Memset")):
                continue
            ev.append((e.start_ns(), e.end_ns(), e.name(), e.device_resource_id()))
        ev.sort()
        streams = {}
        for s0, s1, n, st in ev:
            if "attn_decode" in n:
                streams[st] = streams.get(st, 0) + 1
        dec = max(streams, key=streams.get) if streams else None
        inc = {}
        frontier = ev[0][0] if ev else 0
        for s0, s1, n, st in ev:
            if "attn_decode" in n:
                c = "decode_attention"
            elif "attn_prefill" in n:
                c = "prefill_attention"
            elif "gemm_bf16" in n:
                c = "decode_gemm" if st == dec else "prefill_gemm"
            else:
                c = "decode_other" if st == dec else "prefill_other"
            inc[c] = inc.get(c, 0) + max(0, s1 - max(s0, frontier))
            frontier = max(frontier, s1)
        span = (frontier - ev[0][0]) if ev else 1
        out[w[1]] = {"iterations": [w[0], w[0] + width], "span_ms": round(span / 1e6, 3),
                     **{c: round(v / span, 4) for c, v in sorted(inc.items())}}
    return {"what": "CUPTI critical-path shares of one more RL batch of this workload (uninstrumented)",
            "iterations": n_it, **out}


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
    # default: round-robin in (hint desc, id asc) order -- the fastest measured policy on B200
    # (profiles/r02/multi: config 3 at N = 2 / 4, round-robin 125.0 / 83.4 s, random 128.7 / 86.7 s,
    # the paper's Alg. 2 148.6 / 96.1 s: its single tail instance carries every long sample);
    # --dispatch skew runs Alg. 2
    ap.add_argument("--dispatch", default="round_robin", choices=["skew", "random", "round_robin"])
    ap.add_argument("--strong", action="store_true", help="fixed global batch (cfg.n_prompts) instead of per GPU")
    ap.add_argument("--profile", default=None, help="T(b) profile t0_ns,k0_ps,b_star,k1_ps for Alg. 2")
    ap.add_argument("--hint-noise", type=float, default=None, help="ranker noise sigma (None: oracle hints)")
    ap.add_argument("--timeline", action="store_true",
                    help="one more batch under CUPTI (torch.profiler) for uninstrumented class shares; default: "
                         "the committed shares of such a run (profiles/r02/bench_timeline_shares.json)")
    ap.add_argument("--group-size", type=int, default=1, help="GRPO-style groups: samples per prompt (NEXT-3)")
    ap.add_argument("--prefix-sharing", action="store_true", help="SGS_F_PREFIX_SHARING (NEXT-3, reading R26)")
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
                        (sgs.sgs.F_SHADOW_WEIGHTS if args.weight_sync == "async" else 0) |
                        (sgs.sgs.F_PREFIX_SHARING if args.prefix_sharing else 0),
                        dispatch=args.dispatch, profile=prof, sample_seed=cfg.seed, trace=False)
    peaks0 = load_peaks()
    inst.set_roofline(peaks0["hbm_gbs"], peaks0["bf16_tflops_sustained"])
    if world > 1:
        uid = [sgs.comm_unique_id() if rank == 0 else None]
        pg.broadcast_object_list(uid, src=0)
        inst.comm_init(uid[0], rank, world)

    def make_batch(step):
        # a fresh RL batch per step: same length distribution, new ids and prompts
        return workload.make_trace(n_total, cfg.prompt_len, cfg.median_out, cfg.sigma, cfg.max_out, shape.vocab,
                                   seed=cfg.seed + 1000 * step, id_base=step * 1_000_000, hint_noise=args.hint_noise,
                                   group_size=args.group_size)

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

    def note(msg):
        if rank == 0:
            print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)
    for w in range(args.warmup):
        one_step(w)
        note(f"warm-up step {w} done")
    for cls in range(18):
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
    stats = {cls: inst.kernel_stats(cls) for cls in range(18)}
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
    roof, kernels = kernel_roofline(inst, stats, peaks, len(timed_rows), dev_s)
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
                               f"forced lengths <= {cfg.max_out}, B={cfg.max_batch}, longest-first, "
                               f"{args.dispatch} dispatch",
                   "prompts_total": n_total, "global_batch": n_total, "parallelism": f"dp{world}",
                   "dispatch": args.dispatch, "weight_sync": args.weight_sync,
                   "hints": "oracle (= forced)" if args.hint_noise is None else
                   f"noisy sigma {args.hint_noise}", "profile": list(prof) if prof else None,
                   "l2": "inputs larger than L2 (weights 15 GB, KV pool > 100 GB)",
                   "group_size": args.group_size, "prefix_sharing": args.prefix_sharing},
        "e2e": {"value": round(tokens / wall_s, 1), "unit": "tokens/s",
                "h2d_bytes_per_step": int(statistics.mean(r["h2d"] for r in results)),
                "d2h_bytes_per_step": int(statistics.mean(r["d2h"] for r in results))},
        "gpu_launches": int(sum(r["launches"] for r in results)),
        "roofline": roof,
        "batch_roofline": batch_roof,
        "kernels": kernels,
        "clocks": clk.summary(),
    }
    note(f"timed steps done: {line['value']} tok/s")
    if args.timeline and world == 1:
        kernels = kernels if kernels is not None else {}
        line["kernels"] = kernels
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ.get("SGS_BENCH_STACK_DUMP_S", "600")), exit=False)
        kernels["_timeline"] = timeline_shares(inst, sgs, make_batch(args.warmup + args.steps), cfg, shape)
        faulthandler.cancel_dump_traceback_later()
        note("timeline batch done")
    elif kernels is not None and os.path.exists(TIMELINE_REF):
        kernels["_timeline"] = {**json.load(open(TIMELINE_REF)), "source": os.path.relpath(TIMELINE_REF, ROOT)}
    if not args.no_cpu_baseline:
        cb = cpu_oracle_sample(shape, cfg)
        note("cpu baseline sample done")
        line["cpu_baseline"] = {"value": round(1.0 / cb["per_token_s"], 4), "unit": "tokens/s", "cores": cb["cores"],
                                "kind": "oracle", "sample": cb["sample"],
                                "b_B_iteration_s": round(cb["b_B_iteration_s"], 2),
                                "host_plane": host_plane_timing(make_batch(0), cfg, inst.n_pages, shape)}
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
