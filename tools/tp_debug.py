"""Debug driver for the 2-GPU TP test (progress to files, per-stage)."""
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import multiprocessing as mp  # noqa: E402


def worker(rank, world, port, q, model, ar, outdir):
    log = open(os.path.join(outdir, f"w{rank}_{ar}.log"), "w", buffering=1)
    faulthandler.dump_traceback_later(90, exit=True, file=log)
    t0 = time.time()

    def P(*a):
        print(f"[{time.time() - t0:7.2f}]", *a, file=log, flush=True)
    P("start")
    os.environ["SGS_TP_NCCL_AR"] = "1" if ar == "nccl" else "0"
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P("pg up")
    import paper_2504_15930_b200 as sgs
    import workload
    shape = workload.MODELS[model]
    n, Pl, med, cap = (16, 16, 10, 30)
    tr = workload.make_trace(n, Pl, med, 0.8, cap, shape.vocab, seed=13, prompt_len_jitter=6)
    inst = sgs.Instance(shape, 4, Pl + 64, device=rank, n_pages=96, weight_seed=808, tp_size=world, tp_rank=rank,
                        flags=sgs.sgs.F_KEEP_LOGITS)
    P("instance")
    uid = [sgs.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    P("uid")
    inst.tp_comm_init(uid[0])
    P("tp_comm_init")
    inst.submit_trace(tr)
    P("submitted")
    k = 0
    while True:
        qd, a = inst.pending()
        if qd == 0 and a == 0:
            break
        c = inst.step()
        lg, ids, tk = inst.last_logits()
        k += 1
        P("step", k, "q", qd, "a", a, "comps", len(c), "rows", len(ids))
    P("done")
    dist.barrier()
    q.put(rank)
    dist.destroy_process_group()


if __name__ == "__main__":
    outdir = sys.argv[1]
    os.makedirs(outdir, exist_ok=True)
    for ar in sys.argv[2:]:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        ps = [ctx.Process(target=worker, args=(r, 2, 29700 + len(ar), q, "tiny", ar, outdir)) for r in range(2)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(150)
            print(ar, "exit", p.exitcode, flush=True)
            if p.exitcode is None:
                p.kill()
