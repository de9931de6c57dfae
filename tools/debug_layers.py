"""Layer-by-layer residual-stream parity of the engine's prefill vs the oracle (debug aid).
usage: debug_layers.py MODEL [field=value ...]"""
import dataclasses, sys
import numpy as np
import oracle, workload
import paper_2504_15930_b200 as sgs

shape = workload.MODELS[sys.argv[1] if len(sys.argv) > 1 else "tiny"]
shape = dataclasses.replace(shape, **{k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])})
toks = np.random.default_rng(1).integers(0, shape.vocab, size=24).astype(np.int32)
inst = sgs.Instance(shape, 2, 64, device=0, n_pages=16, weight_seed=4321)
g = inst.debug_forward(toks)
o = oracle.decoder_dump(shape, 4321, toks)
for k in range(g.shape[0]):
    e = np.abs(g[k] - o[k])
    print("stage %2d (%s) max|h| %.3f  max err %.2e  rel %.2e" % (k, "emb" if k == 0 else ("attn" if k % 2 else "mlp"),
          np.abs(o[k]).max(), e.max(), e.max() / np.abs(o[k]).max()))
