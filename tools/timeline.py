"""In-graph kernel timeline of decode iterations (CUPTI through torch.profiler:
kernel start/end timestamps of the production path -- CUDA graphs + PDL, no
events between kernels).  Per decode kernel kind: mean duration, mean gap to
the previous kernel's end (negative = PDL overlap), and its share of the
iteration; per iteration: span and the sum of kernel busy time.

    python tools/timeline.py --model qwen2.5-7b --b 1 16 64 256 --ctx 2048 [--out gpurun_out/timeline.json]
Prompts are admitted without prefill (SGS_F_SKIP_PREFILL); 8 decode iterations
are traced per b after 4 untraced ones.  A tensor-parallel instance (NEXT-2):
    torchrun --nproc-per-node 2 tools/timeline.py --tp 2 ...   (each shard writes <out>.rank<r>)
"""
import argparse
import collections
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import workload  # noqa: E402


def kind(name):
    n = name
    if "gemm_bf16" in n:
        m = re.search(r"gemm_bf16_tc_kernel<(\d+), (\d+), (\d+)>", n)
        return "gemm" + (f"<cg{m.group(1)},m{m.group(2)}>" if m else "")
    for k in ("tp_allreduce_rmsnorm", "tp_argmax_exchange", "nccl", "attn_decode", "attn_prefill", "rmsnorm",
              "rope_append", "embed", "argmax", "top_p", "bt_delta", "silu_mul"):
        if k in n:
            return k
    return n[:40]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--b", type=int, nargs="*", default=[1, 16, 64, 256])
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--iters", type=int, default=8)
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    ap.add_argument("--tp", type=int, default=1)
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    import paper_2504_15930_b200 as sgs
    shape = workload.MODELS[a.model]
    bmax = max(a.b)
    rank = int(os.environ.get("RANK", "0"))
    if a.tp > 1:
        import torch.distributed as dist
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo")
    inst = sgs.Instance(shape, bmax, a.ctx + 64, device=rank, weight_seed=5, trace=False,
                        flags=sgs.sgs.F_SKIP_PREFILL, max_prefill_tokens=max(16384, a.ctx),
                        tp_size=a.tp, tp_rank=rank if a.tp > 1 else 0)
    if a.tp > 1:
        uid = [sgs.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        inst.tp_comm_init(uid[0])
        a.out = f"{a.out}.rank{rank}"
    out = {"model": a.model, "ctx": a.ctx, "per_b": {}}
    nid = 0
    for b in a.b:
        tr = workload.make_trace(b, a.ctx, 40, 0.0, 40, shape.vocab, seed=b, id_base=nid)
        nid += b
        inst.submit_trace(tr)
        for _ in range(5):
            inst.step()  # admission + warm decode iterations (graphs captured)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(a.iters):
                inst.step()
            torch.cuda.synchronize()
        ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.name and
              not e.name.startswith("Memcpy") and not e.name.startswith("Memset")]
        ev.sort(key=lambda e: e.time_range.start)
        ks = [(kind(e.name), e.time_range.start, e.time_range.end) for e in ev]
        # iterations start at each embed kernel
        starts = [i for i, k in enumerate(ks) if k[0] == "embed"]
        iters = []
        stats = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
        for j in range(len(starts) - 1):
            seg = ks[starts[j]:starts[j + 1]]
            span = seg[-1][2] - seg[0][1]
            busy = 0.0
            last_end = seg[0][1]
            for i, (k, s0, s1) in enumerate(seg):
                st = stats[k]
                st[0] += 1
                st[1] += s1 - s0
                st[2] += (s0 - seg[i - 1][2]) if i else 0.0
                # critical-path increment: how far this kernel's end moves past every earlier end
                st[3] += max(0.0, s1 - last_end) if i else s1 - s0
                busy += max(0.0, s1 - max(s0, last_end))
                last_end = max(last_end, s1)
            iters.append({"span_us": span, "busy_us": busy, "kernels": len(seg)})
        n_it = max(len(iters), 1)
        rec = {"iterations": len(iters),
               "span_us_mean": round(float(np.mean([x["span_us"] for x in iters])), 1) if iters else None,
               "busy_us_mean": round(float(np.mean([x["busy_us"] for x in iters])), 1) if iters else None,
               "kinds": {k: {"per_iter": round(v[0] / n_it, 1), "dur_us_mean": round(v[1] / v[0], 2),
                             "gap_before_us_mean": round(v[2] / v[0], 2),
                             "dur_us_per_iter": round(v[1] / n_it, 1),
                             "crit_us_mean": round(v[3] / v[0], 2), "crit_us_per_iter": round(v[3] / n_it, 1)}
                         for k, v in sorted(stats.items())}}
        out["per_b"][str(b)] = rec
        print(json.dumps({"b": b, **{k: rec[k] for k in ("iterations", "span_us_mean", "busy_us_mean")}}),
              flush=True)
        inst.run()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
