"""N > 1 host logic on CPU: two ranks (gloo, world size 2) each run a null-device
instance; every rank submits the same RL batch, Alg. 2 keeps its share, the
ranks exchange nothing on the data path.  Checks: the shares partition the
batch exactly as the oracle's dispatch says, each rank's schedule is bit-exact
against the oracle simulator on its share, and the weight version advances in
lock step."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workload

PROF = (20000, 500, 128, 2000)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_15930_b200 import Instance
        shape = workload.MODELS["qwen2.5-14b"]
        tr = workload.config_trace("c3_14b_2", n=200)
        inst = Instance(shape, 64, 20000, device=None, n_pages=30000, n_instances=world, instance_rank=rank,
                        profile=PROF)
        mine = inst.submit_trace(tr)
        comps = inst.run()
        inst.update_weights(0)
        ids = sorted(c["id"] for c in comps)
        gathered = [None] * world
        dist.all_gather_object(gathered, dict(rank=rank, ids=ids, mine=mine, trace=inst.trace(0).tolist(),
                                              version=inst.weight_version()))
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


def test_two_ranks_partition_and_schedules():
    world = 2
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
    tr = workload.config_trace("c3_14b_2", n=200)
    exp = oracle.dispatch(tr.ids, tr.prompt_len, tr.hint, world, 64, 16, 30000, PROF)["instance"]
    all_ids = []
    for r in res:
        assert r["ids"] == sorted(tr.ids[exp == r["rank"]].tolist())
        assert r["mine"] == len(r["ids"])
        sub = tr.subset(np.flatnonzero(exp == r["rank"]))
        o = oracle.sched_sim(sub.ids, sub.prompt_len, sub.forced_len, sub.hint, 64, 16, 30000)
        assert np.array_equal(np.array(r["trace"], np.int64), o["iter_blob"])
        assert r["version"] == 1
        all_ids += r["ids"]
    assert sorted(all_ids) == tr.ids.tolist()
