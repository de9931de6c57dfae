"""Configs 3 and 4 on hardware: independent data-parallel generation instances
(one per GPU, torchrun) with the paper's skewness-aware dispatch (Alg. 2,
P:924-984) against random and round-robin dispatch, Eq. 2 score sum vs max,
oracle vs noisy ranker hints (fig:eval:scheduling), plus the
per-RL-step NCCL weight broadcast.

Every rank submits the same full batch and keeps its Alg. 2 share (no
data-path communication).  --instances/--instance-offset let one torchrun of
G GPUs be a wave of a larger job (config 4: 8 instances as two waves of 4 under
gpurun's 4-GPU limit; instances are independent, so the 8-instance makespan is
the max over both waves).  Each policy runs the same batch; per instance:
device time (CUDA events on its stream), generated tokens, iterations.

    torchrun --nproc-per-node 2 tools/dp_experiment.py --config c3_14b_2 --policies skew,skew_max,random,round_robin
    ... --dump-trace gpurun_out/traces   (per-instance schedule traces for tests/test_dp_traces.py)
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import workload  # noqa: E402

PROFILES = {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3_14b_2")
    ap.add_argument("--instances", type=int, default=None, help="total DP instances of the job (default: world)")
    ap.add_argument("--instance-offset", type=int, default=0)
    ap.add_argument("--policies", default="skew,random,round_robin")
    ap.add_argument("--hint-noise", type=float, default=None)
    ap.add_argument("--prompts", type=int, default=None, help="batch size (default: the config's n_prompts)")
    ap.add_argument("--profile", default=None, help="t0_ns,k0_ps,b_star,k1_ps (default: bench.DEFAULT_PROFILES)")
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=0, help="untimed warm-up batches (short) before the policies")
    ap.add_argument("--bcast-reps", type=int, default=3)
    ap.add_argument("--dump-trace", default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    import bench
    import paper_2504_15930_b200 as sgs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", local))
    cfg = workload.CONFIGS[a.config]
    shape = workload.MODELS[cfg.model]
    N = a.instances or world
    me = a.instance_offset + rank
    n = a.prompts or cfg.n_prompts
    seed = cfg.seed if a.seed is None else a.seed
    prof = tuple(int(x) for x in a.profile.split(",")) if a.profile else bench.DEFAULT_PROFILES[cfg.model]
    max_ctx = cfg.prompt_len + cfg.max_out
    tr = workload.make_trace(n, cfg.prompt_len, cfg.median_out, cfg.sigma, cfg.max_out, shape.vocab, seed=seed,
                             hint_noise=a.hint_noise)
    results = []
    insts = {}
    t_init = time.perf_counter()
    for spec in a.policies.split(","):
        policy, score = (spec.split("_max")[0], 1) if spec.endswith("_max") else (spec, 0)
        key = (policy, score)
        # one engine per (policy, score): the dispatch policy is an engine setting
        inst = None
        for k in list(insts):
            insts.pop(k).close()
        torch.cuda.empty_cache()
        inst = sgs.Instance(shape, cfg.max_batch, max_ctx, device=local, n_instances=N, instance_rank=me,
                            weight_seed=cfg.seed, dispatch=policy, score=score, profile=prof, sample_seed=seed,
                            trace=a.dump_trace is not None)
        insts[key] = inst
        if a.warmup:
            w = workload.make_trace(min(n, 64 * N), cfg.prompt_len, 32, 0.5, 64, shape.vocab, seed=seed + 99,
                                    id_base=10_000_000)
            inst.submit_trace(w)
            inst.run()
            inst.trace_clear() if a.dump_trace else None
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record(inst.stream)
        mine = inst.submit_trace(tr)
        comps = inst.run()
        ev1.record(inst.stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        log = inst.iter_log()
        r = {"policy": spec, "instance": me, "samples": mine, "tokens": int(sum(len(c["tokens"]) for c in comps)),
             "dev_s": ev0.elapsed_time(ev1) / 1e3, "wall_s": wall, "iterations": int(len(log)),
             "max_forced": int(max((len(c["tokens"]) for c in comps), default=0)), "n_pages": inst.n_pages}
        if a.dump_trace:
            os.makedirs(a.dump_trace, exist_ok=True)
            np.savez_compressed(os.path.join(a.dump_trace, f"{a.config}_{spec}_N{N}_i{me}.npz"),
                                ids=tr.ids, P=tr.prompt_len, d=tr.forced_len, hint=tr.hint, N=N, instance=me,
                                B=cfg.max_batch, page=cfg.page_size, pool=inst.n_pages, profile=np.array(prof),
                                alpha=20, score=score, policy=policy, iter_blob=inst.trace(0),
                                sample_blob=inst.trace(1))
        gathered = [None] * world
        if world > 1:
            dist.all_gather_object(gathered, r)
        else:
            gathered = [r]
        if rank == 0:
            span = max(x["dev_s"] for x in gathered)
            tok = sum(x["tokens"] for x in gathered)
            line = {"config": a.config, "model": cfg.model, "policy": spec, "instances_total": N,
                    "wave_instances": [x["instance"] for x in gathered], "prompts": n,
                    "hints": "oracle" if a.hint_noise is None else f"noisy sigma {a.hint_noise}",
                    "profile": list(prof), "wave_makespan_s": round(span, 3),
                    "wave_tokens_per_s": round(tok / span, 1), "per_instance": gathered}
            results.append(line)
            print(json.dumps(line), flush=True)
    # weight sync: NCCL broadcast of the whole bf16 weight range from rank 0 (trainer proxy)
    if world > 1 and a.bcast_reps > 0:
        inst = next(iter(insts.values()))
        uid = [sgs.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        inst.comm_init(uid[0], rank, world)
        ptr, nbytes = None, None
        wb = int(sum(r * c for _, r, c in sgs.weight_tensors(shape)) * 2)
        ms = []
        for k in range(a.bcast_reps + 1):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(inst.stream)
            inst.update_weights(0)
            e1.record(inst.stream)
            torch.cuda.synchronize()
            if k:
                ms.append(e0.elapsed_time(e1))
        t = torch.tensor([max(ms)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            line = {"weight_sync": "ncclBroadcast from rank 0", "world": world, "model": cfg.model,
                    "weight_bytes": wb, "ms_max_over_ranks": round(float(t[0]), 2), "reps": a.bcast_reps,
                    "algbw_GBps": round(wb / float(t[0]) / 1e6, 1)}
            results.append(line)
            print(json.dumps(line), flush=True)
    if rank == 0 and a.out:
        json.dump({"results": results, "init_s": round(time.perf_counter() - t_init, 1)}, open(a.out, "w"), indent=1)
    for i in insts.values():
        i.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
