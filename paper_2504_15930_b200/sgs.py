"""Thin ctypes binding of libsgs.so (include/sgs.h).  Argument marshalling only:
every step of the hot path runs in the library's sm_100a kernels.  PyTorch is
used for device memory (the arena), streams and process groups."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SGS_LIB_PATH: an alternative in-tree build of the same library (A/B timing in tools/ab.sh)
LIB_PATH = os.environ.get("SGS_LIB_PATH") or os.path.join(_HERE, "libsgs.so")

SGS_OK = 0
STATUS = {0: "SGS_OK", -1: "SGS_E_INVAL", -2: "SGS_E_NOMEM", -3: "SGS_E_STATE", -4: "SGS_E_CAPACITY",
          -5: "SGS_E_CUDA", -6: "SGS_E_NCCL", -7: "SGS_E_UNSUPPORTED"}
DISPATCH = {"skew": 0, "round_robin": 1, "random": 2}
F_KEEP_LOGITS = 1
F_NO_GRAPHS = 2
F_KERNEL_TIMING = 4
F_SHADOW_WEIGHTS = 8
F_TRACE = 16
F_DETERMINISTIC = 32
F_SKIP_PREFILL = 64
F_PREFIX_SHARING = 128

# every symbol include/sgs.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = [
    "sgs_arena_bytes", "sgs_init", "sgs_destroy", "sgs_last_error", "sgs_submit", "sgs_step", "sgs_pending",
    "sgs_comm_unique_id", "sgs_comm_init", "sgs_update_weights", "sgs_load_weights_seed", "sgs_weight_checksum",
    "sgs_shadow_weights", "sgs_stage_weights_seed", "sgs_update_weights_begin", "sgs_update_weights_ready",
    "sgs_update_weights_commit",
    "sgs_weight_version", "sgs_trace", "sgs_trace_clear", "sgs_last_logits", "sgs_last_iter_ms",
    "sgs_kernel_launches", "sgs_fit_profile", "sgs_dispatch_plan", "sgs_attn_workspace_bytes",
    "sgs_op_decode_attention", "sgs_op_gemm", "sgs_op_rmsnorm", "sgs_op_rope_append", "sgs_rope_table",
    "sgs_op_argmax", "sgs_op_prefill_attention", "sgs_debug_forward", "sgs_op_silu_mul", "sgs_kernel_stats", "sgs_io_bytes",
    "sgs_set_roofline", "sgs_kernel_roofline_ms", "sgs_iter_log", "sgs_debug_layer", "sgs_op_sample_top_p",
    "sgs_weight_tensors", "sgs_stage_weights", "sgs_prefill_workspace_bytes", "sgs_host_state",
    "sgs_op_decode_attention_timed", "sgs_elastic_plan", "sgs_set_instances", "sgs_tp_comm_init",
    "sgs_tp_tail_plan",
]


class SgsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class ModelCfg(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("d_model", ctypes.c_int32), ("n_q_heads", ctypes.c_int32),
                ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("d_ffn", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("rms_eps", ctypes.c_float), ("rope_theta", ctypes.c_double)]


class TbProfile(ctypes.Structure):
    _fields_ = [("t0_ns", ctypes.c_int64), ("k0_ps", ctypes.c_int64), ("b_star", ctypes.c_int64),
                ("k1_ps", ctypes.c_int64)]


class EngineCfg(ctypes.Structure):
    _fields_ = [("max_batch", ctypes.c_int32), ("page_size", ctypes.c_int32), ("max_ctx", ctypes.c_int32),
                ("max_prefill_tokens", ctypes.c_int32), ("n_pages", ctypes.c_int64), ("arena", ctypes.c_void_p),
                ("arena_bytes", ctypes.c_int64), ("stream", ctypes.c_void_p), ("device", ctypes.c_int32),
                ("n_instances", ctypes.c_int32), ("instance_rank", ctypes.c_int32), ("dispatch", ctypes.c_int32),
                ("alpha_pct", ctypes.c_int32), ("score", ctypes.c_int32), ("tail_ceil", ctypes.c_int32),
                ("profile", TbProfile), ("sampling", ctypes.c_int32), ("temperature", ctypes.c_float),
                ("top_p", ctypes.c_float), ("sample_seed", ctypes.c_uint64), ("weight_seed", ctypes.c_uint64),
                ("flags", ctypes.c_int32), ("tp_size", ctypes.c_int32), ("tp_rank", ctypes.c_int32)]


class Weights(ctypes.Structure):
    _fields_ = [("ptrs", ctypes.POINTER(ctypes.c_void_p)), ("n", ctypes.c_int32)]


class Prompt(ctypes.Structure):
    _fields_ = [("id", ctypes.c_uint64), ("tokens", ctypes.POINTER(ctypes.c_int32)), ("len", ctypes.c_int32)]


class Completion(ctypes.Structure):
    _fields_ = [("id", ctypes.c_uint64), ("instance", ctypes.c_int32), ("n_tokens", ctypes.c_int32),
                ("tokens", ctypes.POINTER(ctypes.c_int32)), ("admit_iter", ctypes.c_int64),
                ("finish_iter", ctypes.c_int64), ("weight_version", ctypes.c_int32), ("slot", ctypes.c_int32)]


_lib = None


def lib():
    """Load libsgs.so; fail loudly when it is missing (there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2504_15930_b200.build`")
        _lib = ctypes.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def _declare(L):
    vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    P = ctypes.POINTER
    L.sgs_arena_bytes.argtypes = [P(ModelCfg), P(EngineCfg), i64, P(i64), P(i64)]
    L.sgs_init.argtypes = [P(ModelCfg), P(EngineCfg), P(Weights), P(vp)]
    L.sgs_weight_tensors.argtypes = [P(ModelCfg), P(i64), P(i64), P(i64), i32, P(i32)]
    L.sgs_stage_weights.argtypes = [vp, P(Weights)]
    L.sgs_host_state.argtypes = [vp, P(i64), P(i64), P(i64)]
    L.sgs_elastic_plan.argtypes = [P(EngineCfg), i32, P(u64), P(i32), P(i32), i64, i64, P(i64), P(i64), P(i32)]
    L.sgs_set_instances.argtypes = [vp, i32, i32]
    L.sgs_tp_tail_plan.argtypes = [P(EngineCfg), i64, i32, i32, i64, P(TbProfile), i64, i64, i64, i64, i32, P(u64),
                                   P(i32), P(i32), P(i32), P(i64)]
    L.sgs_tp_comm_init.argtypes = [vp, P(ctypes.c_uint8)]
    L.sgs_prefill_workspace_bytes.argtypes = [i32, i32, i32, i32]
    L.sgs_prefill_workspace_bytes.restype = i64
    L.sgs_destroy.argtypes = [vp]
    L.sgs_destroy.restype = None
    L.sgs_last_error.argtypes = [vp]
    L.sgs_last_error.restype = ctypes.c_char_p
    L.sgs_submit.argtypes = [vp, P(Prompt), i32, P(i32), P(i32), P(i32)]
    L.sgs_step.argtypes = [vp, P(Completion), i32, P(i32)]
    L.sgs_pending.argtypes = [vp, P(i64), P(i64)]
    L.sgs_comm_unique_id.argtypes = [P(ctypes.c_uint8)]
    L.sgs_comm_init.argtypes = [vp, P(ctypes.c_uint8), i32, i32]
    L.sgs_update_weights.argtypes = [vp, P(Weights), i32]
    L.sgs_shadow_weights.argtypes = [vp, P(vp), P(i64)]
    L.sgs_stage_weights_seed.argtypes = [vp, u64]
    L.sgs_update_weights_begin.argtypes = [vp, i32]
    L.sgs_update_weights_ready.argtypes = [vp, P(i32)]
    L.sgs_update_weights_commit.argtypes = [vp]
    L.sgs_load_weights_seed.argtypes = [vp, u64]
    L.sgs_weight_checksum.argtypes = [vp, i64, P(u64)]
    L.sgs_weight_version.argtypes = [vp, P(i32)]
    L.sgs_trace.argtypes = [vp, i32, P(i64), i64, P(i64)]
    L.sgs_trace_clear.argtypes = [vp]
    L.sgs_last_logits.argtypes = [vp, P(ctypes.c_float), P(u64), P(i32), i32, P(i32)]
    L.sgs_last_iter_ms.argtypes = [vp, P(ctypes.c_float)]
    L.sgs_kernel_launches.argtypes = [vp, P(i64)]
    L.sgs_fit_profile.argtypes = [i32, P(ctypes.c_double), P(ctypes.c_double), P(ctypes.c_double), P(TbProfile)]
    L.sgs_dispatch_plan.argtypes = [P(EngineCfg), i32, P(u64), P(i32), P(i32), i64, P(i32), P(i32)]
    L.sgs_attn_workspace_bytes.argtypes = [i32, i32, i32, i32, i32]
    L.sgs_attn_workspace_bytes.restype = i64
    L.sgs_op_decode_attention.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, vp, i32, vp, i64, i32,
                                          vp]
    L.sgs_op_decode_attention_timed.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, vp, vp, i64, i32, vp,
                                                i64, P(ctypes.c_float), vp]
    L.sgs_op_gemm.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, i32, vp]
    L.sgs_op_rmsnorm.argtypes = [vp, vp, vp, i32, i32, ctypes.c_float, vp]
    L.sgs_op_rope_append.argtypes = [vp, vp, vp, vp, vp, i32, vp, vp, vp, i32, i32, i32, i32, i32, vp]
    L.sgs_rope_table.argtypes = [P(ctypes.c_float), i32, i32, ctypes.c_double]
    L.sgs_op_argmax.argtypes = [vp, i32, i32, vp, vp]
    L.sgs_kernel_stats.argtypes = [vp, i32, P(ctypes.c_double), P(ctypes.c_double), P(ctypes.c_double), P(i64), i32]
    L.sgs_io_bytes.argtypes = [vp, P(i64), P(i64)]
    L.sgs_set_roofline.argtypes = [vp, ctypes.c_double, ctypes.c_double]
    L.sgs_kernel_roofline_ms.argtypes = [vp, i32, P(ctypes.c_double)]
    L.sgs_iter_log.argtypes = [vp, P(i64), i64, P(i64)]
    L.sgs_debug_layer.argtypes = [vp, i32, P(ctypes.c_float), i32, P(ctypes.c_float)]
    L.sgs_op_sample_top_p.argtypes = [vp, i32, i32, ctypes.c_float, ctypes.c_float, u64, vp, vp, vp, vp]
    L.sgs_op_silu_mul.argtypes = [vp, vp, i32, i32, vp]
    L.sgs_debug_forward.argtypes = [vp, P(i32), i32, P(ctypes.c_float)]
    L.sgs_op_prefill_attention.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, vp, vp, i64, vp]
    for name in EXPORTS:
        f = getattr(L, name)
        if name not in ("sgs_destroy", "sgs_last_error", "sgs_attn_workspace_bytes", "sgs_prefill_workspace_bytes"):
            f.restype = ctypes.c_int


def _check(rc, h=None):
    if rc != SGS_OK:
        raise SgsError(rc, lib().sgs_last_error(h).decode(errors="replace"))


def _i32p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def model_cfg(shape) -> ModelCfg:
    return ModelCfg(shape.n_layers, shape.d_model, shape.n_q_heads, shape.n_kv_heads, shape.head_dim, shape.d_ffn,
                    shape.vocab, shape.rms_eps, shape.rope_theta)


def weight_tensors(shape):
    """Canonical weight order of a model: list of (tensor id, rows, cols) (sgs_weight_tensors)."""
    m = model_cfg(shape)
    n = ctypes.c_int32()
    _check(lib().sgs_weight_tensors(ctypes.byref(m), None, None, None, 0, ctypes.byref(n)))
    ids, rows, cols = (np.zeros(n.value, np.int64) for _ in range(3))
    P = ctypes.POINTER(ctypes.c_int64)
    _check(lib().sgs_weight_tensors(ctypes.byref(m), ids.ctypes.data_as(P), rows.ctypes.data_as(P),
                                    cols.ctypes.data_as(P), n.value, ctypes.byref(n)))
    return [(int(a), int(b), int(c)) for a, b, c in zip(ids, rows, cols)]


def make_weights(tensors):
    """sgs_weights over a list of bf16 tensors (torch CPU/CUDA or numpy uint16 views) in canonical
    order; the returned object keeps the pointer array alive."""
    ptrs = (ctypes.c_void_p * max(len(tensors), 1))()
    for i, t in enumerate(tensors):
        ptrs[i] = t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data
    w = Weights(ctypes.cast(ptrs, ctypes.POINTER(ctypes.c_void_p)), len(tensors))
    w._keep = (ptrs, tensors)
    return w


def _stream_ptr(stream):
    if stream is None:
        return None
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


class Instance:
    """One generation instance (one GPU, or null-device mode when device is None)."""

    def __init__(self, shape, max_batch: int, max_ctx: int, device: int | None = 0, page_size: int = 16,
                 n_pages: int | None = None, mem_fraction: float = 0.92, n_instances: int = 1,
                 instance_rank: int = 0, dispatch: str = "skew", alpha_pct: int = 20, score: int = 0,
                 tail_ceil: int = 0, profile=(2000, 1000, 208, 5000), weight_seed: int = 1234,
                 sample_seed: int = 0, flags: int = 0, max_prefill_tokens: int = 16384, stream=None,
                 top_p: float | None = None, temperature: float = 1.0, trace: bool = True, weights=None,
                 tp_size: int = 1, tp_rank: int = 0):
        """weights: None (hash-init from weight_seed) or a list of bf16 tensors in the
        canonical order of weight_tensors(shape).  trace: keep the schedule trace
        (SGS_F_TRACE; the C default is off, bench.py turns it off)."""
        L = lib()
        self.shape = shape
        self.m = model_cfg(shape)
        e = EngineCfg()
        e.max_batch, e.page_size, e.max_ctx, e.max_prefill_tokens = max_batch, page_size, max_ctx, max_prefill_tokens
        e.device = -1 if device is None else int(device)
        e.n_instances, e.instance_rank = n_instances, instance_rank
        e.dispatch, e.alpha_pct, e.score, e.tail_ceil = DISPATCH[dispatch], alpha_pct, score, tail_ceil
        e.profile = TbProfile(*profile)
        e.sampling, e.temperature, e.top_p = (1 if top_p is not None else 0), temperature, (top_p or 1.0)
        e.sample_seed, e.weight_seed, e.flags = sample_seed, weight_seed, flags | (F_TRACE if trace else 0)
        e.tp_size, e.tp_rank = tp_size, tp_rank
        self.tp_size = max(1, tp_size)
        self.arena = None
        self.stream = None
        if device is None:
            if not n_pages:
                raise ValueError("null-device mode needs n_pages")
            e.n_pages = n_pages
        else:
            import torch
            torch.cuda.set_device(device)
            self.stream = stream if stream is not None else torch.cuda.Stream(device=device)
            fixed, page_bytes = ctypes.c_int64(), ctypes.c_int64()
            _check(L.sgs_arena_bytes(ctypes.byref(self.m), ctypes.byref(e), 0, ctypes.byref(fixed),
                                     ctypes.byref(page_bytes)))
            free, _ = torch.cuda.mem_get_info(device)
            budget = int(free * mem_fraction) - fixed.value
            fit = budget // page_bytes.value
            if n_pages is None:
                n_pages = fit
            if n_pages < 1 or n_pages > fit:
                raise SgsError(-2, f"KV pool of {n_pages} pages does not fit ({fit} possible)")
            total = fixed.value + n_pages * page_bytes.value
            self.arena = torch.empty(total, dtype=torch.uint8, device=f"cuda:{device}")
            e.n_pages = n_pages
            e.arena = ctypes.c_void_p(self.arena.data_ptr())
            e.arena_bytes = total
            e.stream = _stream_ptr(self.stream)
        self.n_pages = e.n_pages
        self.e = e
        h = ctypes.c_void_p()
        wts = make_weights(weights) if weights is not None else None
        _check(L.sgs_init(ctypes.byref(self.m), ctypes.byref(e), ctypes.byref(wts) if wts is not None else None,
                          ctypes.byref(h)))
        self.h = h
        self._cap = max(64, max_batch * 2)
        self._comp = (Completion * self._cap)()

    def close(self):
        if getattr(self, "h", None):
            lib().sgs_destroy(self.h)
            self.h = None
        self.arena = None  # the device arena goes back to PyTorch's allocator

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- service API
    def submit(self, ids, tokens, offsets, hint, forced) -> int:
        n = len(ids)
        toks = np.ascontiguousarray(tokens, dtype=np.int32)
        offs = np.asarray(offsets, dtype=np.int64)
        prompts = (Prompt * max(n, 1))()
        base = toks.ctypes.data
        for i in range(n):
            prompts[i].id = int(ids[i])
            prompts[i].tokens = ctypes.cast(base + 4 * int(offs[i]), ctypes.POINTER(ctypes.c_int32))
            prompts[i].len = int(offs[i + 1] - offs[i])
        hint = np.ascontiguousarray(hint, dtype=np.int32)
        forced = np.ascontiguousarray(forced, dtype=np.int32)
        mine = ctypes.c_int32()
        _check(lib().sgs_submit(self.h, prompts, n, _i32p(hint), _i32p(forced), ctypes.byref(mine)), self.h)
        return mine.value

    def submit_trace(self, tr) -> int:
        return self.submit(tr.ids, tr.tokens, tr.offsets, tr.hint, tr.forced_len)

    def step(self, cap: int | None = None):
        """One iteration; returns a list of completion dicts (ascending id)."""
        cap = self._cap if cap is None else min(int(cap), self._cap)  # the C side writes <= cap records
        n = ctypes.c_int32()
        _check(lib().sgs_step(self.h, self._comp, cap, ctypes.byref(n)), self.h)
        out = []
        for i in range(n.value):
            c = self._comp[i]
            toks = np.ctypeslib.as_array(c.tokens, shape=(c.n_tokens,)).copy() if c.n_tokens else np.zeros(0, np.int32)
            out.append(dict(id=int(c.id), instance=c.instance, tokens=toks, admit_iter=c.admit_iter,
                            finish_iter=c.finish_iter, weight_version=c.weight_version, slot=c.slot))
        return out

    def host_state(self):
        """(sample records, queue entries, live ids) held on the host."""
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().sgs_host_state(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), self.h)
        return a.value, b.value, c.value

    def set_instances(self, n_instances: int, instance_rank: int):
        """Elastic DP (NEXT-4): change the data-parallel layout between RL batches."""
        _check(lib().sgs_set_instances(self.h, n_instances, instance_rank), self.h)

    def pending(self):
        q, a = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().sgs_pending(self.h, ctypes.byref(q), ctypes.byref(a)), self.h)
        return q.value, a.value

    def run(self, on_step=None):
        """Step until idle; returns all completions."""
        done = []
        while True:
            q, a = self.pending()
            c = self.step()
            if on_step:
                on_step(c)
            done.extend(c)
            if not c and q == 0 and a == 0:
                return done

    # ---------------------------------------------------------------- weights
    def load_weights_seed(self, seed: int):
        _check(lib().sgs_load_weights_seed(self.h, seed), self.h)

    def checksum(self, tensor_id: int) -> int:
        v = ctypes.c_uint64()
        _check(lib().sgs_weight_checksum(self.h, tensor_id, ctypes.byref(v)), self.h)
        return v.value

    def comm_init(self, uid: bytes, rank: int, world: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().sgs_comm_init(self.h, buf, rank, world), self.h)

    def tp_comm_init(self, uid: bytes):
        """NEXT-2: the tensor-parallel communicator (uid from comm_unique_id on shard 0)."""
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().sgs_tp_comm_init(self.h, buf), self.h)

    def update_weights(self, root: int = 0, weights=None):
        """Weight sync: the root copies `weights` (canonical order, or None = keep its
        current weights) and broadcasts; other ranks pass None."""
        wts = make_weights(weights) if weights is not None else None
        _check(lib().sgs_update_weights(self.h, ctypes.byref(wts) if wts is not None else None, root), self.h)

    def stage_weights(self, weights):
        """Asynchronous sync, trainer path: copy weights into the shadow buffer (side stream)."""
        wts = make_weights(weights)
        _check(lib().sgs_stage_weights(self.h, ctypes.byref(wts)), self.h)

    # ---- asynchronous weight sync (flags |= F_SHADOW_WEIGHTS)
    def shadow_weights(self):
        """(device pointer, bytes) of the shadow weight buffer a trainer writes the next weights into."""
        p, n = ctypes.c_void_p(), ctypes.c_int64()
        _check(lib().sgs_shadow_weights(self.h, ctypes.byref(p), ctypes.byref(n)), self.h)
        return p.value, n.value

    def stage_weights_seed(self, seed: int):
        _check(lib().sgs_stage_weights_seed(self.h, seed), self.h)

    def update_weights_begin(self, root: int = 0):
        _check(lib().sgs_update_weights_begin(self.h, root), self.h)

    def update_weights_ready(self) -> bool:
        r = ctypes.c_int32()
        _check(lib().sgs_update_weights_ready(self.h, ctypes.byref(r)), self.h)
        return bool(r.value)

    def update_weights_commit(self):
        _check(lib().sgs_update_weights_commit(self.h), self.h)

    def weight_version(self) -> int:
        v = ctypes.c_int32()
        _check(lib().sgs_weight_version(self.h, ctypes.byref(v)), self.h)
        return v.value

    # ---------------------------------------------------------------- introspection
    def trace(self, which: int = 0) -> np.ndarray:
        n = ctypes.c_int64()
        _check(lib().sgs_trace(self.h, which, None, 0, ctypes.byref(n)), self.h)
        buf = np.zeros(n.value, np.int64)
        _check(lib().sgs_trace(self.h, which, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n.value,
                               ctypes.byref(n)), self.h)
        return buf

    def trace_clear(self):
        _check(lib().sgs_trace_clear(self.h), self.h)

    def last_logits(self):
        rows = ctypes.c_int32()
        _check(lib().sgs_last_logits(self.h, None, None, None, 0, ctypes.byref(rows)), self.h)
        r = rows.value
        lg = np.zeros((r, self.shape.vocab // self.tp_size), np.float32)  # a TP shard keeps its vocabulary rows
        ids = np.zeros(r, np.uint64)
        tk = np.zeros(r, np.int32)
        _check(lib().sgs_last_logits(self.h, lg.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                     ids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), _i32p(tk), r,
                                     ctypes.byref(rows)), self.h)
        return lg, ids, tk

    def debug_forward(self, tokens) -> np.ndarray:
        """Residual stream after the embedding and each residual add: [2L+1, T, d] fp32."""
        toks = np.ascontiguousarray(tokens, np.int32)
        out = np.zeros((2 * self.shape.n_layers + 1, len(toks), self.shape.d_model), np.float32)
        _check(lib().sgs_debug_forward(self.h, _i32p(toks), len(toks),
                                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_float))), self.h)
        return out

    def debug_layer(self, layer: int, h_in) -> np.ndarray:
        """Run one decoder layer of the CUDA path on h_in [T, d] (fp32); returns h after the layer."""
        h = np.ascontiguousarray(h_in, np.float32)
        out = np.zeros_like(h)
        _check(lib().sgs_debug_layer(self.h, layer, h.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), h.shape[0],
                                     out.ctypes.data_as(ctypes.POINTER(ctypes.c_float))), self.h)
        return out

    def debug_head(self, h_in) -> np.ndarray:
        """Final RMSNorm + LM head of the CUDA path on h_in [T, d] -> fp32 logits [T, V]."""
        h = np.ascontiguousarray(h_in, np.float32)
        out = np.zeros((h.shape[0], self.shape.vocab), np.float32)
        _check(lib().sgs_debug_layer(self.h, self.shape.n_layers, h.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                     h.shape[0], out.ctypes.data_as(ctypes.POINTER(ctypes.c_float))), self.h)
        return out

    def last_iter_ms(self) -> float:
        v = ctypes.c_float()
        _check(lib().sgs_last_iter_ms(self.h, ctypes.byref(v)), self.h)
        return v.value

    def kernel_stats(self, cls: int, reset: bool = False):
        ms, by, fl, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        _check(lib().sgs_kernel_stats(self.h, cls, ctypes.byref(ms), ctypes.byref(by), ctypes.byref(fl),
                                      ctypes.byref(n), int(reset)), self.h)
        return dict(ms=ms.value, bytes=by.value, flops=fl.value, launches=n.value)

    def set_roofline(self, bw_gbs: float, tflops: float):
        _check(lib().sgs_set_roofline(self.h, bw_gbs, tflops), self.h)

    def kernel_roofline_ms(self, cls: int) -> float:
        v = ctypes.c_double()
        _check(lib().sgs_kernel_roofline_ms(self.h, cls, ctypes.byref(v)), self.h)
        return v.value

    def iter_log(self) -> np.ndarray:
        """[n, 6] int64: t, b, admitted, prefill tokens, sum of contexts, device us."""
        n = ctypes.c_int64()
        _check(lib().sgs_iter_log(self.h, None, 0, ctypes.byref(n)), self.h)
        buf = np.zeros(n.value, np.int64)
        _check(lib().sgs_iter_log(self.h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n.value,
                                  ctypes.byref(n)), self.h)
        return buf.reshape(-1, 6)

    def io_bytes(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().sgs_io_bytes(self.h, ctypes.byref(a), ctypes.byref(b)), self.h)
        return a.value, b.value

    def kernel_launches(self) -> int:
        v = ctypes.c_int64()
        _check(lib().sgs_kernel_launches(self.h, ctypes.byref(v)), self.h)
        return v.value


def comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().sgs_comm_unique_id(buf))
    return bytes(buf)


def fit_profile(b, T_ns):
    b = np.ascontiguousarray(b, np.float64)
    T = np.ascontiguousarray(T_ns, np.float64)
    out = np.zeros(5, np.float64)
    prof = TbProfile()
    _check(lib().sgs_fit_profile(len(b), b.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                 T.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(prof)))
    return dict(t0=out[0], k0=out[1], k1=out[2], t1=out[3], sse=out[4],
                profile=(prof.t0_ns, prof.k0_ps, prof.b_star, prof.k1_ps))


def dispatch_plan(ids, prompt_len, hint, n_instances, max_batch, page, pool_pages, profile, alpha_pct=20, score=0,
                  tail_ceil=0, policy="skew", seed=0):
    e = EngineCfg()
    e.n_instances, e.max_batch, e.page_size = n_instances, max_batch, page
    e.profile = TbProfile(*profile)
    e.alpha_pct, e.score, e.tail_ceil, e.dispatch, e.sample_seed = alpha_pct, score, tail_ceil, DISPATCH[policy], seed
    n = len(ids)
    ids = np.ascontiguousarray(ids, np.uint64)
    P = np.ascontiguousarray(prompt_len, np.int32)
    h = np.ascontiguousarray(hint, np.int32)
    inst = np.zeros(n, np.int32)
    nl = ctypes.c_int32()
    _check(lib().sgs_dispatch_plan(ctypes.byref(e), n, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), _i32p(P),
                                   _i32p(h), pool_pages, _i32p(inst), ctypes.byref(nl)))
    return inst, nl.value


def elastic_plan(ids, prompt_len, hint, n_instances, max_batch, page, pool_pages, profile, delta_ps, alpha_pct=20,
                 score=0, tail_ceil=0):
    """NEXT-4: predicted generation ps on N and N+1 instances, delta' and the decision."""
    e = EngineCfg()
    e.n_instances, e.max_batch, e.page_size = n_instances, max_batch, page
    e.profile = TbProfile(*profile)
    e.alpha_pct, e.score, e.tail_ceil, e.dispatch = alpha_pct, score, tail_ceil, 0
    n = len(ids)
    ids = np.ascontiguousarray(ids, np.uint64)
    P = np.ascontiguousarray(prompt_len, np.int32)
    h = np.ascontiguousarray(hint, np.int32)
    t = np.zeros(2, np.int64)
    dp = ctypes.c_int64()
    so = ctypes.c_int32()
    _check(lib().sgs_elastic_plan(ctypes.byref(e), n, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), _i32p(P),
                                  _i32p(h), pool_pages, int(delta_ps), t.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                  ctypes.byref(dp), ctypes.byref(so)))
    return dict(t_gen_ps=(int(t[0]), int(t[1])), delta_prime_ps=dp.value, scale_out=bool(so.value))


def tp_tail_plan(ids, prompt_len, hint, n_dp, max_batch, page, pool_pages, profile, tp_size, tp_max_batch,
                 tp_pool_pages, tp_profile, dispatch="round_robin", alpha_pct=20, score=0, tail_ceil=0, kv_ps=0,
                 tp_kv_ps=0, pf_ps=0, tp_pf_ps=0):
    """NEXT-2 two-dimensional dispatch (R27): how many of the longest samples go to one
    tensor-parallel instance; predicted ps of the TP instance, of the DP instances, and of DP only."""
    e = EngineCfg()
    e.n_instances, e.max_batch, e.page_size = n_dp, max_batch, page
    e.profile = TbProfile(*profile)
    e.alpha_pct, e.score, e.tail_ceil, e.dispatch = alpha_pct, score, tail_ceil, DISPATCH[dispatch]
    tpp = TbProfile(*tp_profile)
    n = len(ids)
    ids = np.ascontiguousarray(ids, np.uint64)
    P = np.ascontiguousarray(prompt_len, np.int32)
    h = np.ascontiguousarray(hint, np.int32)
    t = np.zeros(3, np.int64)
    k = ctypes.c_int32()
    _check(lib().sgs_tp_tail_plan(ctypes.byref(e), pool_pages, tp_size, tp_max_batch, tp_pool_pages, ctypes.byref(tpp),
                                  int(kv_ps), int(tp_kv_ps), int(pf_ps), int(tp_pf_ps), n, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), _i32p(P), _i32p(h),
                                  ctypes.byref(k), t.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    return dict(n_tail=k.value, t_tp_ps=int(t[0]), t_dp_ps=int(t[1]), t_all_ps=int(t[2]),
                use_tp=bool(max(t[0], t[1]) < t[2]))


def rope_table(max_pos: int, hd: int, theta: float) -> np.ndarray:
    out = np.zeros((max_pos, hd // 2, 2), np.float32)
    _check(lib().sgs_rope_table(out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), max_pos, hd, theta))
    return out


# -------------------------------------------------------------------- kernel-level ops (torch tensors)
def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _cur_stream(t):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def op_gemm(W, X, C, mode: int = 0, splits: int = 1):
    N, K = W.shape
    T = X.shape[0]
    _check(lib().sgs_op_gemm(_ptr(W), _ptr(X), _ptr(C), N, K, T, C.shape[1], mode, splits, _cur_stream(W)))


def op_rmsnorm(x, w, y, eps: float):
    T, d = x.shape
    _check(lib().sgs_op_rmsnorm(_ptr(x), _ptr(w), _ptr(y), T, d, eps, _cur_stream(x)))


def op_rope_append(qkv, bias, pos, slot, block_table, cos_sin, q_out, kv, nq, nkv, hd, page=16):
    T = qkv.shape[0]
    maxp = block_table.shape[1] if block_table is not None else 0
    _check(lib().sgs_op_rope_append(_ptr(qkv), _ptr(bias), _ptr(pos), _ptr(slot), _ptr(block_table), maxp,
                                    _ptr(cos_sin), _ptr(q_out), _ptr(kv), T, nq, nkv, hd, page, _cur_stream(qkv)))


def op_silu_mul(gu, m):
    T, f = m.shape
    _check(lib().sgs_op_silu_mul(_ptr(gu), _ptr(m), T, f, _cur_stream(gu)))


def op_sample_top_p(logits, temperature, top_p, seed, sample_ids, steps, ids):
    rows, V = logits.shape
    _check(lib().sgs_op_sample_top_p(_ptr(logits), rows, V, temperature, top_p, seed, _ptr(sample_ids), _ptr(steps),
                                     _ptr(ids), _cur_stream(logits)))


def op_argmax(logits, ids):
    rows, V = logits.shape
    _check(lib().sgs_op_argmax(_ptr(logits), rows, V, _ptr(ids), _cur_stream(logits)))


def op_prefill_attention(q, k, v, offs, out, workspace=None):
    import torch
    T, nq, hd = q.shape
    nkv = k.shape[1]
    need = lib().sgs_prefill_workspace_bytes(T, offs.numel() - 1, nkv, hd)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=q.device)
    _check(lib().sgs_op_prefill_attention(_ptr(q), _ptr(k), _ptr(v), _ptr(offs), offs.numel() - 1, nq, nkv, hd,
                                          _ptr(out), _ptr(workspace), workspace.numel(), _cur_stream(q)))


def op_decode_attention(q, kv, block_table, ctx, out, page=16, split_pages=0, workspace=None):
    import torch
    b, nq, hd = q.shape
    nkv = kv.shape[1]
    maxp = block_table.shape[1]
    need = lib().sgs_attn_workspace_bytes(b, nq, nkv, hd, maxp)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=q.device)
    out_fp32 = 1 if out.dtype == torch.float32 else 0
    _check(lib().sgs_op_decode_attention(_ptr(q), _ptr(kv), _ptr(block_table), _ptr(ctx), b, nq, nkv, hd, page, maxp,
                                         0, _ptr(out), out_fp32, _ptr(workspace), workspace.numel(), split_pages,
                                         _cur_stream(q)))


def op_decode_attention_timed(q, kv, block_table, ctx, out, reps=10, l2_flush=None, page=16, workspace=None):
    """Mean device ms per launch of the decode-attention kernel (plan built once)."""
    import torch
    b, nq, hd = q.shape
    nkv = kv.shape[1]
    maxp = block_table.shape[1]
    need = lib().sgs_attn_workspace_bytes(b, nq, nkv, hd, maxp)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=q.device)
    ms = ctypes.c_float()
    _check(lib().sgs_op_decode_attention_timed(_ptr(q), _ptr(kv), _ptr(block_table), _ptr(ctx), b, nq, nkv, hd, page,
                                               maxp, _ptr(out), _ptr(workspace), workspace.numel(), reps,
                                               _ptr(l2_flush), 0 if l2_flush is None else l2_flush.numel(),
                                               ctypes.byref(ms), _cur_stream(q)))
    return ms.value


# -------------------------------------------------------------------- KV page layout
def _swz(r: int, rowchunks: int) -> int:
    return (r & 7) if rowchunks >= 8 else ((r >> 1) & (rowchunks - 1))


def kv_perm(hd: int, page: int = 16):
    """perm[r, e] = physical column of logical element e in row r of a page-head."""
    rc = hd // 8
    e = np.arange(hd)
    return np.stack([(((e // 8) ^ _swz(r, rc)) * 8 + e % 8) for r in range(page)])


def kv_pack(K, V):
    """Logical K/V [n_pages, nkv, page, hd] (torch) -> pool [n_pages, nkv, 2, page, hd] with swizzled rows."""
    import torch
    n_pages, nkv, page, hd = K.shape
    perm = torch.from_numpy(kv_perm(hd, page)).to(K.device)
    pool = torch.empty((n_pages, nkv, 2, page, hd), dtype=K.dtype, device=K.device)
    idx = perm.view(1, 1, page, hd).expand(n_pages, nkv, page, hd)
    pool[:, :, 0].scatter_(3, idx, K)
    pool[:, :, 1].scatter_(3, idx, V)
    return pool


def kv_unpack(pool):
    """Inverse of kv_pack: pool [n_pages, nkv, 2, page, hd] -> (K, V) logical."""
    import torch
    n_pages, nkv, _, page, hd = pool.shape
    perm = torch.from_numpy(kv_perm(hd, page)).to(pool.device)
    idx = perm.view(1, 1, page, hd).expand(n_pages, nkv, page, hd)
    return pool[:, :, 0].gather(3, idx), pool[:, :, 1].gather(3, idx)
