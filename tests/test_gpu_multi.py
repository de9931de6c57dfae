"""Weight sync over NCCL (a15) on 2 GPUs: rank 0 (trainer proxy)
regenerates its weights from a new seed, sgs_update_weights broadcasts them,
and every rank's weights are then bit-identical to the oracle generator with
that seed (64-bit checksums).  Needs >= 2 GPUs (gpurun --gpus 2)."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

import oracle
import workload

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2504_15930_b200 as sgs
        shape = workload.MODELS["tiny"]
        inst = sgs.Instance(shape, 8, 128, device=rank, n_pages=64, n_instances=world, instance_rank=rank,
                            weight_seed=1000 + rank)
        uid = [sgs.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        inst.comm_init(uid[0], rank, world)
        if rank == 0:
            inst.load_weights_seed(4242)
        inst.update_weights(0)
        sums = {tid: inst.checksum(tid) for tid in (0, 1, 2, 16, 23, 24, 27, 32 + 9)}
        out = [None] * world
        dist.all_gather_object(out, dict(rank=rank, sums=sums, version=inst.weight_version()))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_weight_sync_broadcast_bit_identical():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (run with gpurun --gpus 2)")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    shape = workload.MODELS["tiny"]
    sizes = {0: shape.vocab * shape.d_model, 1: shape.vocab * shape.d_model, 2: shape.d_model,
             16: shape.n_q_heads * shape.head_dim * shape.d_model, 23: shape.d_ffn * shape.d_model,
             24: shape.d_ffn * shape.d_model, 27: shape.d_model, 41: shape.d_model * shape.d_ffn}
    norm = {2, 27}
    for r in res:
        assert r["version"] == 1
        for tid, v in r["sums"].items():
            assert v == oracle.tensor_checksum(4242, tid, sizes[tid], tid in norm), (r["rank"], tid)
