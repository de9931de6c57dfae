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


def _async_worker(rank, world, port, q):
    # NEXT-1: the broadcast of the next weights overlaps generation of the
    # current batch; the batch completes on the old weights (old checksums,
    # old version), the commit at the batch boundary installs the new ones
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2504_15930_b200 as sgs
        shape = workload.MODELS["tiny"]
        inst = sgs.Instance(shape, 8, 128, device=rank, n_pages=64, n_instances=world, instance_rank=rank,
                            weight_seed=77, flags=sgs.sgs.F_SHADOW_WEIGHTS)
        uid = [sgs.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        inst.comm_init(uid[0], rank, world)
        tr = workload.make_trace(16, 12, 30, 0.5, 40, shape.vocab, seed=5)
        inst.submit_trace(tr)
        inst.step()
        if rank == 0:
            inst.stage_weights_seed(4242)  # trainer proxy writes the next weights into its shadow buffer
        inst.update_weights_begin(0)
        done = inst.run()  # generation continues while the broadcast runs on the side stream
        old = {tid: inst.checksum(tid) for tid in (0, 16, 27)}
        inst.update_weights_commit()
        new = {tid: inst.checksum(tid) for tid in (0, 16, 27)}
        tr2 = workload.make_trace(4, 12, 5, 0.5, 5, shape.vocab, seed=6, id_base=1000)
        inst.submit_trace(tr2)
        done2 = inst.run()
        out = [None] * world
        dist.all_gather_object(out, dict(rank=rank, old=old, new=new, v1={c["weight_version"] for c in done},
                                         v2={c["weight_version"] for c in done2}, version=inst.weight_version()))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def _spawn(target, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_async_weight_sync_overlaps_generation():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (run with gpurun --gpus 2)")
    res = _spawn(_async_worker, 2)
    shape = workload.MODELS["tiny"]
    sizes = {0: shape.vocab * shape.d_model, 16: shape.n_q_heads * shape.head_dim * shape.d_model,
             27: shape.d_model}
    for r in res:
        assert r["v1"] == {0} and r["v2"] == {1} and r["version"] == 1
        for tid, n in sizes.items():
            assert r["old"][tid] == oracle.tensor_checksum(77, tid, n, tid == 27), (r["rank"], tid)
            assert r["new"][tid] == oracle.tensor_checksum(4242, tid, n, tid == 27), (r["rank"], tid)


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


def _src_worker(rank, world, port, q):
    # the trainer path of sgs_update_weights (P:595-596 update(weights)): the root
    # passes the new weights (host tensors, canonical order) and every rank ends
    # with them bit for bit; non-root ranks pass no source
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2504_15930_b200 as sgs
        shape = workload.MODELS["tiny"]
        inst = sgs.Instance(shape, 8, 128, device=rank, n_pages=64, n_instances=world, instance_rank=rank,
                            weight_seed=3000 + rank)
        uid = [sgs.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        inst.comm_init(uid[0], rank, world)
        w = None
        if rank == 0:
            w = []
            for tid, rows, cols in sgs.weight_tensors(shape):
                norm = tid == 2 or (tid >= 16 and (tid - 16) % 16 >= 10)
                w.append(torch.from_numpy(oracle.gen_tensor(555, tid, rows * cols, norm)).to(torch.bfloat16))
        inst.update_weights(0, weights=w)
        sums = {tid: inst.checksum(tid) for tid in (0, 1, 2, 16, 23, 24, 27, 32 + 9)}
        out = [None] * world
        dist.all_gather_object(out, dict(rank=rank, sums=sums, version=inst.weight_version()))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_weight_sync_from_trainer_source():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (run with gpurun --gpus 2)")
    res = _spawn(_src_worker, 2)
    shape = workload.MODELS["tiny"]
    sizes = {0: shape.vocab * shape.d_model, 1: shape.vocab * shape.d_model, 2: shape.d_model,
             16: shape.n_q_heads * shape.head_dim * shape.d_model, 23: shape.d_ffn * shape.d_model,
             24: shape.d_ffn * shape.d_model, 27: shape.d_model, 41: shape.d_model * shape.d_ffn}
    for r in res:
        assert r["version"] == 1
        for tid, v in r["sums"].items():
            assert v == oracle.tensor_checksum(555, tid, sizes[tid], tid in {2, 27}), (r["rank"], tid)


def _tp_worker(rank, world, port, q, model, ar):
    # NEXT-2: one tensor-parallel instance over `world` GPUs --
    # q/kv heads, FFN columns and vocabulary rows split, O / down partial sums
    # and the LM-head argmax combined over NVLink peer memory (tp_comm.cu) or
    # with NCCL all-reduces (SGS_TP_NCCL_AR=1)
    import torch.distributed as dist
    os.environ["SGS_TP_NCCL_AR"] = "1" if ar == "nccl" else "0"
    import faulthandler
    faulthandler.dump_traceback_later(float(os.environ.get("SGS_TEST_STACK_DUMP_S", "600")), exit=False)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        import paper_2504_15930_b200 as sgs
        shape = workload.MODELS[model]
        n, P, med, cap = (16, 16, 10, 30) if model == "tiny" else (3, 20, 6, 10)
        tr = workload.make_trace(n, P, med, 0.8, cap, shape.vocab, seed=13, prompt_len_jitter=6)
        inst = sgs.Instance(shape, 4, P + 64, device=rank, n_pages=96, weight_seed=808, tp_size=world, tp_rank=rank,
                            flags=sgs.sgs.F_KEEP_LOGITS)
        uid = [sgs.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        inst.tp_comm_init(uid[0])
        inst.submit_trace(tr)
        rows, comps = {}, []
        while True:
            qd, a = inst.pending()
            if qd == 0 and a == 0:
                break
            comps += inst.step()
            lg, ids, tk = inst.last_logits()
            for r in range(len(ids)):
                rows[(int(ids[r]), int(tk[r]))] = lg[r].copy()
        out = [None] * world
        dist.all_gather_object(out, dict(rank=rank, rows=rows, toks={c["id"]: c["tokens"].tolist() for c in comps},
                                         trace=inst.trace(0).tolist(), strace=inst.trace(1).tolist()))
        if rank == 0:
            q.put((tr, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("model,ar,tp", [("tiny", "p2p", 2), ("tiny", "nccl", 2), ("qwen2.5-7b", "p2p", 2),
                                         ("qwen2.5-7b", "p2p", 4)])
def test_tensor_parallel_instance_vs_oracle(model, ar, tp):
    if torch.cuda.device_count() < tp:
        pytest.skip(f"needs {tp} GPUs (run with gpurun --gpus {tp})")
    import numpy as np
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_worker, args=(r, tp, port, q, model, ar)) for r in range(tp)]
    for p in procs:
        p.start()
    tr, res = q.get(timeout=900)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    shape = workload.MODELS[model]
    # every shard ran the same schedule, equal to the oracle's, and emitted the same tokens
    o = oracle.sched_sim(tr.ids, tr.prompt_len, tr.forced_len, tr.hint, 4, 16, 96)
    for r in res:
        assert r["trace"] == o["iter_blob"].tolist()
        assert r["toks"] == res[0]["toks"]
    tol = 2e-2 if model == "tiny" else 0.25  # DESIGN.md R17 for the 28-layer 7B shape
    check = tr.ids.tolist() if model == "tiny" else tr.ids[:2].tolist()
    for sid in check:
        i = int(np.flatnonzero(tr.ids == sid)[0])
        prompt = tr.tokens[tr.offsets[i]:tr.offsets[i + 1]]
        gen = np.array(res[0]["toks"][sid])
        # the shards' vocabulary rows, concatenated in shard order
        got = np.stack([np.concatenate([r["rows"][(sid, j)] for r in res]) for j in range(len(gen))])
        ref = oracle.decoder_forward(shape, 808, np.concatenate([prompt, gen[:-1]]).astype(np.int32),
                                     first_row=len(prompt) - 1)
        err = np.abs(got - ref).max()
        assert err <= tol, (sid, err)
        assert np.array_equal(got.argmax(1), gen)
