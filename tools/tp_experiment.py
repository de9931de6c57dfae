"""NEXT-2 on hardware: tensor-parallel (TP = 2) generation instances for the
long tail ("tensor parallelism ... to reduce the per-sample
latency"; dedicated instances for the long-tail samples).

  --mode sweep   (2 GPUs) decode T(b) of one TP = 2 instance at a context,
                 prompts admitted without prefill (SGS_F_SKIP_PREFILL)
  --mode tail    (4 GPUs) one RL batch two ways: (A) the tail group (top
                 alpha% by hint) on a TP = 2 instance over GPUs 0-1 and the
                 rest round-robin on two DP instances (GPUs 2, 3); (B) four DP
                 instances, round-robin over the whole batch (the best policy
                 of config 3).  Makespan = max over instances (device time).

    torchrun --nproc-per-node 2 tools/tp_experiment.py --mode sweep --out gpurun_out/tp_sweep.json
    torchrun --nproc-per-node 4 tools/tp_experiment.py --mode tail --out gpurun_out/tp_tail.json
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
    ap.add_argument("--mode", default="sweep", choices=["sweep", "tail"])
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--b", type=int, nargs="*", default=[1, 2, 4, 8, 16, 32, 64, 128, 256])
    ap.add_argument("--prompts", type=int, default=1024)
    ap.add_argument("--alpha-pct", type=int, default=20, help="< 0: sgs_tp_tail_plan chooses the split")
    ap.add_argument("--phases", default="A_tp2_tail,B_dp4_round_robin")
    ap.add_argument("--dp-prof", default=None, help="t0_ns,k0_ps,b_star,k1_ps of one GPU (planner; else fitted)")
    ap.add_argument("--tp-prof", default=None, help="the same for the TP pair")
    ap.add_argument("--dp-kv", type=int, default=0, help="ps per cached context token per iteration, one GPU")
    ap.add_argument("--tp-kv", type=int, default=0, help="the same for the TP pair")
    ap.add_argument("--dp-pf", type=int, default=0, help="ps per prefilled prompt token, one GPU")
    ap.add_argument("--tp-pf", type=int, default=0, help="the same for the TP pair")
    ap.add_argument("--dp-ctx", type=int, default=2048, help="context of the DP side's T(b) points (planner)")
    ap.add_argument("--tp-ctx", type=int, default=2048, help="context of the TP side's T(b) points (planner)")
    ap.add_argument("--dp-pool", type=int, default=150000, help="KV pages of one DP instance (planner)")
    ap.add_argument("--tp-pool", type=int, default=300000, help="KV pages of one TP shard (planner)")
    ap.add_argument("--dp-profile-file", default="profiles/r02/tb_layout_tiles.json",
                    help="T(b) points of one GPU (ctx 2048 used) for the planner's DP side")
    ap.add_argument("--tp-profile-file", default="profiles/r02/tp/tp2_sweep_ll_ctx2048.json",
                    help="T(b) points of the TP pair (ctx 2048, p2p exchange) for the planner's TP side")
    ap.add_argument("--ar", nargs="*", default=["p2p", "nccl"], choices=["p2p", "nccl"])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    import paper_2504_15930_b200 as sgs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(rank)
    dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", rank))
    shape = workload.MODELS[a.model]
    out = {"mode": a.mode, "model": a.model}

    def tp_pair(ranks, **kw):
        """A TP = len(ranks) instance over `ranks` (this rank must be in it)."""
        r = ranks.index(rank)
        inst = sgs.Instance(shape, kw.pop("B"), kw.pop("max_ctx"), device=rank, tp_size=len(ranks), tp_rank=r,
                            trace=False, **kw)
        return inst

    if a.mode == "sweep":
        assert world in (2, 4)
        pts, nid = [], 0
        for ar in a.ar:
            # exchange of the partials: NVLink peer memory (tp_comm.cu) or NCCL all-reduces
            os.environ["SGS_TP_NCCL_AR"] = "1" if ar == "nccl" else "0"
            inst = tp_pair(list(range(world)), B=max(a.b), max_ctx=a.ctx + 16, weight_seed=5, flags=sgs.sgs.F_SKIP_PREFILL,
                           max_prefill_tokens=max(16384, a.ctx))
            uid = [sgs.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            inst.tp_comm_init(uid[0])
            for b in a.b:
                tr = workload.make_trace(b, a.ctx, 7, 0.0, 7, shape.vocab, seed=b, id_base=nid)
                nid += b
                n0 = len(inst.iter_log())
                inst.submit_trace(tr)
                inst.run()
                log = inst.iter_log()[n0:]
                dec = log[(log[:, 3] == 0) & (log[:, 1] == b)]
                t = torch.tensor([float(np.median(dec[:, 5])) if len(dec) else 0.0], dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                pts.append({"b": b, "ctx": a.ctx, "exchange": ar, "tp": world, "T_us_tp2": float(t[0])})
                if rank == 0:
                    print(json.dumps(pts[-1]), flush=True)
            inst.close()
            del inst
            torch.cuda.empty_cache()
            dist.barrier()
        out["points"] = pts
    else:
        assert world == 4
        tr = workload.make_trace(a.prompts, 512, 1024, 1.0, 8192, shape.vocab, seed=1234)
        order = sorted(range(len(tr)), key=lambda i: (-int(tr.hint[i]), int(tr.ids[i])))
        if a.alpha_pct >= 0:
            n_tail = a.alpha_pct * len(tr) // 100
        else:
            # two-dimensional dispatch (sgs_tp_tail_plan, R27) with T(b) fits of the committed ctx-2048
            # sweeps: one GPU (tiled weights) for the DP side, the TP = 2 pair (peer-memory exchange)
            def fit(path, keep=lambda p: True):
                pts = [p for p in json.load(open(os.path.join(ROOT, path)))["points"] if keep(p)]
                return tuple(sgs.fit_profile(np.array([p["b"] for p in pts], float),
                                             np.array([p.get("T_us", p.get("T_us_tp2")) * 1e3 for p in pts],
                                                      float))["profile"])
            if a.dp_prof:  # fixed profiles (e.g. tools/fit_kv_profile.py over several contexts)
                dp_prof = tuple(int(x) for x in a.dp_prof.split(","))
                tp_prof = tuple(int(x) for x in a.tp_prof.split(","))
            else:
                dp_prof = fit(a.dp_profile_file, lambda p: p.get("ctx", 2048) == a.dp_ctx)
                tp_prof = fit(a.tp_profile_file,
                              lambda p: p.get("exchange") == "p2p" and p.get("ctx", 2048) == a.tp_ctx)
            plan = sgs.tp_tail_plan(tr.ids, tr.prompt_len, tr.hint, 2, 256, 16, a.dp_pool, dp_prof, 2, 256, a.tp_pool,
                                    tp_prof, dispatch="round_robin", kv_ps=a.dp_kv, tp_kv_ps=a.tp_kv, pf_ps=a.dp_pf,
                                    tp_pf_ps=a.tp_pf)
            n_tail = plan["n_tail"]
            out["plan"] = {**plan, "dp_profile": dp_prof, "tp_profile": tp_prof, "dp_ctx": a.dp_ctx, "tp_ctx": a.tp_ctx,
                           "dp_pool": a.dp_pool, "tp_pool": a.tp_pool, "dp_kv": a.dp_kv, "tp_kv": a.tp_kv,
                           "dp_pf": a.dp_pf, "tp_pf": a.tp_pf}
            if rank == 0:
                print(json.dumps({"plan": out["plan"]}), flush=True)
        tail, reg = tr.subset(order[:n_tail]), tr.subset(order[n_tail:])
        res = {}
        for phase in a.phases.split(","):
            torch.cuda.empty_cache()
            if phase.startswith("A"):
                if rank < 2:
                    inst = tp_pair([0, 1], B=256, max_ctx=512 + 8192, weight_seed=5)
                    uid = [sgs.comm_unique_id() if rank == 0 else None]
                else:
                    inst = sgs.Instance(shape, 256, 512 + 8192, device=rank, n_instances=2, instance_rank=rank - 2,
                                        dispatch="round_robin", weight_seed=5, trace=False)
                    uid = [None]
                objs = [uid[0] if rank == 0 else None]
                dist.broadcast_object_list(objs, src=0)
                if rank < 2:
                    inst.tp_comm_init(objs[0])
                mine = tail if rank < 2 else reg
            else:
                inst = sgs.Instance(shape, 256, 512 + 8192, device=rank, n_instances=4, instance_rank=rank,
                                    dispatch="round_robin", weight_seed=5, trace=False)
                mine = tr
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(inst.stream)
            kept = inst.submit_trace(mine)
            comps = inst.run()
            e1.record(inst.stream)
            torch.cuda.synchronize()
            rec = {"rank": rank, "samples": kept, "tokens": int(sum(len(c["tokens"]) for c in comps)),
                   "dev_s": e0.elapsed_time(e1) / 1e3}
            g = [None] * world
            dist.all_gather_object(g, rec)
            if rank == 0:
                span = max(x["dev_s"] for x in g)
                # a TP pair generates one set of tokens: count rank 0's, not rank 1's
                tok = sum(x["tokens"] for x in g if not (phase.startswith("A") and x["rank"] == 1))
                res[phase] = {"makespan_s": round(span, 3), "tokens": tok, "tokens_per_s": round(tok / span, 1),
                              "per_rank": g}
                print(json.dumps({phase: res[phase]}), flush=True)
            inst.close()
            del inst
            dist.barrier()
        out["alpha_pct"] = a.alpha_pct
        out["n_tail"] = n_tail
        out["results"] = res
    if rank == 0 and a.out:
        json.dump(out, open(a.out, "w"), indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
