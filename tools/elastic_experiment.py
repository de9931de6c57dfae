"""NEXT-4 on hardware: elastic data-parallel scale-out of the generation stage
(§4.2 "Dynamic adjustment").  RL steps whose output lengths grow
step by step ("the generation length of LLMs increases progressively during
RL training") run on N active instances out of the torchrun world;
after each step the measured gap delta = T_gen - T_train is compared with
delta' = T_gen(N) - T_gen(N + 1) predicted by sgs_elastic_plan on the current
batch (Alg. 2 + longest-first schedule timed with the T(b) profile, R25); when
delta >= delta' one more DP unit joins (sgs_set_instances) for the next step.

Trainer stand-in (the trainer is out of scope): T_train = c * (prompt + output
tokens of the batch), c calibrated so that step 0 on one instance is balanced
(training time grows with total tokens, generation with the longest sample).

    torchrun --nproc-per-node 4 tools/elastic_experiment.py --steps 6 --out gpurun_out/elastic.json
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
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--prompts", type=int, default=256)
    ap.add_argument("--prompt-len", type=int, default=512)
    ap.add_argument("--median0", type=int, default=256)
    ap.add_argument("--growth", type=float, default=1.5)
    ap.add_argument("--cap", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--B", type=int, default=256)
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
    shape = workload.MODELS[a.model]
    prof = bench.DEFAULT_PROFILES[a.model]
    inst = sgs.Instance(shape, a.B, a.prompt_len + a.cap, device=local, n_instances=1, instance_rank=0,
                        weight_seed=7, profile=prof, trace=False)
    N, c_train, log = 1, None, []
    for s in range(a.steps):
        med = int(a.median0 * a.growth ** s)
        tr = workload.make_trace(a.prompts, a.prompt_len, med, 1.0, a.cap, shape.vocab, seed=100 + s,
                                 id_base=s * 1_000_000)
        dev = 0.0
        if rank < N:
            inst.set_instances(N, rank)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(inst.stream)
            inst.submit_trace(tr)
            inst.run()
            ev1.record(inst.stream)
            torch.cuda.synchronize()
            dev = ev0.elapsed_time(ev1) / 1e3
        t = torch.tensor([dev], dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_gen = float(t[0])
        tokens = int(tr.prompt_len.sum() + tr.forced_len.sum())
        if c_train is None:
            c_train = t_gen / tokens  # step 0 on one instance is balanced
        t_train = c_train * tokens
        delta_ps = int((t_gen - t_train) * 1e12)
        plan = sgs.elastic_plan(tr.ids, tr.prompt_len, tr.hint, N, a.B, 16, inst.n_pages, prof, delta_ps)
        rec = {"step": s, "N": N, "median_out": med, "max_out": int(tr.forced_len.max()), "tokens": tokens,
               "T_gen_s": round(t_gen, 3), "T_train_s": round(t_train, 3), "delta_s": round(t_gen - t_train, 3),
               "pred_T_gen_N_s": round(plan["t_gen_ps"][0] / 1e12, 3),
               "pred_T_gen_N1_s": round(plan["t_gen_ps"][1] / 1e12, 3),
               "delta_prime_s": round(plan["delta_prime_ps"] / 1e12, 3), "scale_out": plan["scale_out"]}
        if rank == 0:
            print(json.dumps(rec), flush=True)
        log.append(rec)
        if plan["scale_out"] and N < world:
            N += 1
        if world > 1:
            dist.barrier()
    if rank == 0 and a.out:
        json.dump({"model": a.model, "world": world, "profile": list(prof), "steps": log,
                   "trainer": "T_train = c * tokens, c from step 0 at N = 1"}, open(a.out, "w"), indent=1)
    inst.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
