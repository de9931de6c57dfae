"""NEXT-2 host logic at N > 1 on CPU (gloo, world size 4): the layout of the
tail experiment -- ranks 0-1 one tensor-parallel instance for the longest
samples, ranks 2-3 two DP instances for the rest -- with every rank computing
the split from the same batch through sgs_tp_tail_plan (no communication on
the data path).  Null-device instances stand in for the GPU ones (the TP pair's
two shards run the same scheduler on the same samples).  Checks: all ranks
agree on the split, it equals the oracle's (R27), the shares partition the
batch, and every rank's schedule is bit-exact against the oracle simulator."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workload

PROF_DP = (2_800_000, 13_500_000, 16, 21_800_000)
PROF_TP = (2_080_000, 9_500_000, 16, 15_300_000)
B, POOL = 64, 30000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch():
    return workload.make_trace(160, 64, 256, 1.0, 2048, 1024, seed=77)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2504_15930_b200 as sgs
        shape = workload.MODELS["qwen2.5-7b"]
        tr = _batch()
        plan = sgs.tp_tail_plan(tr.ids, tr.prompt_len, tr.hint, 2, B, 16, POOL, PROF_DP, 2, B, POOL, PROF_TP,
                                dispatch="round_robin")
        order = sorted(range(len(tr)), key=lambda i: (-int(tr.hint[i]), int(tr.ids[i])))
        k = plan["n_tail"]
        share = tr.subset(order[:k]) if rank < 2 else tr.subset(order[k:])
        if rank < 2:  # one shard of the TP instance: the whole tail on one scheduler
            inst = sgs.Instance(shape, B, 64 + 2048, device=None, n_pages=POOL, profile=PROF_TP)
        else:
            inst = sgs.Instance(shape, B, 64 + 2048, device=None, n_pages=POOL, n_instances=2, instance_rank=rank - 2,
                                dispatch="round_robin", profile=PROF_DP)
        mine = inst.submit_trace(share)
        comps = inst.run()
        out = [None] * world
        dist.all_gather_object(out, dict(rank=rank, plan=plan, mine=mine, ids=sorted(c["id"] for c in comps),
                                         trace=inst.trace(0).tolist()))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_tail_split_on_four_ranks():
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tr = _batch()
    o = oracle.tp_tail_plan(tr.ids, tr.prompt_len, tr.hint, 2, B, 16, POOL, PROF_DP, 2, B, POOL, PROF_TP)
    for r in res:  # every rank took the same split, the oracle's
        assert (r["plan"]["n_tail"], r["plan"]["t_tp_ps"], r["plan"]["t_dp_ps"], r["plan"]["t_all_ps"]) == \
            (o["n_tail"], o["t_tp_ps"], o["t_dp_ps"], o["t_all_ps"])
    k = o["n_tail"]
    order = sorted(range(len(tr)), key=lambda i: (-int(tr.hint[i]), int(tr.ids[i])))
    tail, rest = order[:k], order[k:]
    # the TP pair's two shards: the whole tail, identical schedules, equal to the oracle's
    sub = tr.subset(tail)
    ot = oracle.sched_sim(sub.ids, sub.prompt_len, sub.forced_len, sub.hint, B, 16, POOL)
    assert res[0]["ids"] == res[1]["ids"] == sorted(sub.ids.tolist())
    assert res[0]["trace"] == res[1]["trace"] == ot["iter_blob"].tolist()
    # the DP ranks: round robin over the rest in (hint desc, id asc) order
    all_ids = list(res[0]["ids"])
    for j, r in enumerate(res[2:]):
        sel = [rest[x] for x in range(j, len(rest), 2)]
        s = tr.subset(sel)
        od = oracle.sched_sim(s.ids, s.prompt_len, s.forced_len, s.hint, B, 16, POOL)
        assert r["ids"] == sorted(s.ids.tolist())
        assert r["trace"] == od["iter_blob"].tolist()
        all_ids += r["ids"]
    assert sorted(all_ids) == sorted(tr.ids.tolist())
    assert 0 < k < len(tr)
