"""Per-position teacher-forced logits error of the engine vs the oracle (debug aid).
usage: debug_e2e.py MODEL [field=value ...]   e.g. debug_e2e.py tiny n_layers=1 d_model=3584"""
import dataclasses
import sys
import numpy as np
import oracle, workload
import paper_2504_15930_b200 as sgs

name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
shape = workload.MODELS[name]
over = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
shape = dataclasses.replace(shape, **over)
tr = workload.make_trace(4, 20, 6, 0.5, 10, shape.vocab, seed=2, prompt_len_jitter=12)
inst = sgs.Instance(shape, 2, 64, device=0, n_pages=64, weight_seed=4321, flags=sgs.sgs.F_KEEP_LOGITS)
inst.submit_trace(tr)
rows, comps = {}, []
while True:
    q, a = inst.pending()
    if q == 0 and a == 0:
        break
    comps += inst.step()
    lg, ids, tk = inst.last_logits()
    for r in range(len(ids)):
        rows[(int(ids[r]), int(tk[r]))] = lg[r].copy()
toks = {c["id"]: c["tokens"] for c in comps}
errs = []
for sid in tr.ids.tolist()[:2]:
    i = int(np.flatnonzero(tr.ids == sid)[0])
    prompt = tr.tokens[tr.offsets[i]:tr.offsets[i + 1]]
    seq = np.concatenate([prompt, toks[sid][:-1]]).astype(np.int32)
    ref = oracle.decoder_forward(shape, 4321, seq, first_row=len(prompt) - 1)
    got = np.stack([rows[(sid, j)] for j in range(len(toks[sid]))])
    errs.append(np.abs(got - ref).max(1))
e = np.concatenate(errs)
print(over, "max err %.4f  median %.4f" % (e.max(), np.median(e)), "ref std %.3f" % ref.std())
