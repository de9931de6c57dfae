"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation (C++ under oracle/src/,
loaded here with ctypes) of what StreamRL's generation stage computes.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package.  It shares no code with paper_2504_15930_b200/.

Functions and the paper passages they follow (PAPER.md line numbers):
  sched_sim        C2  longest-first continuous batching
  dispatch         C5  Alg. 2 + Eq. 2
  tb_fit/T_ps      C3  piecewise-linear T(b), hinge fit
  min_merge_gain   C3  lemma T(x+y) < T(x)+T(y)
  elastic_plan     NEXT-4 delta vs delta' (one more DP unit)
  tp_tail_plan     NEXT-2 long tail on a TP instance (R27)
  brute_force      C4  LF vs all admission orders
  attention        C7  naive softmax attention, fp64
  decoder_layer/head  C6  one layer / final norm + LM head    (chained layer-local parity)
  decoder_forward  C6  teacher-forced Qwen2.5-shaped decoder   P:1032-1049  (parity unpinned end to end;
                                                                              components pinned)
  gen_tensor       K11 counter-based weight generator
  sample_top_p     C8  nucleus sampling with Philox4x32-10     DESIGN.md R18
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "src")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SOURCES = ["sched_sim.cpp", "dispatch.cpp", "tb.cpp", "model.cpp", "elastic.cpp", "capi.cpp"]


def build(force: bool = False) -> str:
    srcs = [os.path.join(_SRC, s) for s in _SOURCES] + [os.path.join(_SRC, "oracle.hpp")]
    if not force and os.path.exists(_LIB_PATH):
        lib_m = os.path.getmtime(_LIB_PATH)
        if all(os.path.getmtime(s) <= lib_m for s in srcs):
            return _LIB_PATH
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-o", _LIB_PATH + ".tmp"] + [os.path.join(_SRC, s) for s in _SOURCES]
    subprocess.run(cmd, check=True)
    os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _declare(_lib)
    return _lib


P_i64 = ctypes.POINTER(ctypes.c_int64)
P_i32 = ctypes.POINTER(ctypes.c_int32)
P_u32 = ctypes.POINTER(ctypes.c_uint32)
P_f32 = ctypes.POINTER(ctypes.c_float)
P_f64 = ctypes.POINTER(ctypes.c_double)


def _declare(L):
    L.oracle_last_error.restype = ctypes.c_char_p
    L.oracle_bf16_round.argtypes = [ctypes.c_float]
    L.oracle_bf16_round.restype = ctypes.c_float
    L.oracle_sched_sim.argtypes = [ctypes.c_int32, P_i64, P_i32, P_i32, P_i32, P_i32, P_i64, ctypes.c_int32,
                                   ctypes.c_int32, ctypes.c_int64, P_i64, P_i64, P_i64]
    L.oracle_sched_sim.restype = ctypes.c_int64
    L.oracle_sched_blob.argtypes = [ctypes.c_int32, P_i64]
    L.oracle_sched_blob.restype = ctypes.c_int64
    L.oracle_dispatch.argtypes = [ctypes.c_int32, P_i64, P_i32, P_i32, ctypes.c_int32, ctypes.c_int32,
                                  ctypes.c_int32, ctypes.c_int64, P_i64, ctypes.c_int32, ctypes.c_int32,
                                  ctypes.c_int32, P_i32, P_i64, P_i64]
    L.oracle_elastic_plan.argtypes = [ctypes.c_int32, P_i64, P_i32, P_i32, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_int64, P_i64, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_int64, P_i64]
    L.oracle_elastic_plan.restype = ctypes.c_int32
    L.oracle_tp_tail_plan.argtypes = [ctypes.c_int32, P_i64, P_i32, P_i32, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_int64, P_i64, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                      P_i64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, P_i64]
    L.oracle_tp_tail_plan.restype = ctypes.c_int32
    L.oracle_nearest_rank.argtypes = [ctypes.c_int32, P_i64, ctypes.c_int32]
    L.oracle_nearest_rank.restype = ctypes.c_int64
    L.oracle_T_ps.argtypes = [P_i64, ctypes.c_int64, P_i64]
    L.oracle_tb_fit.argtypes = [ctypes.c_int32, P_f64, P_f64, P_f64, P_i64]
    L.oracle_tb_min_merge_gain.argtypes = [P_i64, ctypes.c_int64, P_i64]
    L.oracle_brute_force.argtypes = [ctypes.c_int32, P_i32, ctypes.c_int32, P_i64, P_i64]
    L.oracle_run_order.argtypes = [ctypes.c_int32, P_i32, P_i32, ctypes.c_int32, P_i64, P_i64]
    L.oracle_attention.argtypes = [ctypes.c_int32] * 4 + [P_f32, P_f32, P_f32, P_f64]
    L.oracle_gen_tensor.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, P_f32]
    L.oracle_tensor_checksum.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32]
    L.oracle_tensor_checksum.restype = ctypes.c_uint64
    L.oracle_weight_hash.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
    L.oracle_weight_hash.restype = ctypes.c_uint64
    L.oracle_decoder_forward.argtypes = [P_i32, P_f64, ctypes.c_uint64, P_i32, ctypes.c_int32, ctypes.c_int32,
                                         P_f64]
    L.oracle_decoder_forward.restype = ctypes.c_int32
    L.oracle_decoder_dump.argtypes = [P_i32, P_f64, ctypes.c_uint64, P_i32, ctypes.c_int32, P_f64]
    L.oracle_decoder_dump.restype = ctypes.c_int32
    L.oracle_decoder_layer.argtypes = [P_i32, P_f64, ctypes.c_uint64, ctypes.c_int32, P_f64, ctypes.c_int32, P_f64]
    L.oracle_weight_cache.argtypes = [ctypes.c_int32]
    L.oracle_decoder_head.argtypes = [P_i32, P_f64, ctypes.c_uint64, P_f64, ctypes.c_int32, P_f64]
    L.oracle_rmsnorm.argtypes = [P_f64, P_f32, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, P_f64]
    L.oracle_rope.argtypes = [P_f64, ctypes.c_int32, ctypes.c_int32, ctypes.c_double]
    L.oracle_argmax.argtypes = [P_f32, ctypes.c_int64]
    L.oracle_argmax.restype = ctypes.c_int32
    L.oracle_philox.argtypes = [P_u32, P_u32, P_u32]
    L.oracle_sample_top_p.argtypes = [P_f32, ctypes.c_int64, ctypes.c_float, ctypes.c_float, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_uint64]
    L.oracle_sample_top_p.restype = ctypes.c_int32


def _p(a, t):
    return a.ctypes.data_as(t)


def _i128(hi, lo):
    return (int(hi) << 64) + (int(lo) & 0xFFFFFFFFFFFFFFFF)


def _prof(profile):
    return np.asarray(profile, dtype=np.int64)


# ------------------------------------------------------------------ C3
def T_ps(profile, b: int) -> int:
    out = np.zeros(2, np.int64)
    lib().oracle_T_ps(_p(_prof(profile), P_i64), int(b), _p(out, P_i64))
    return _i128(out[0], out[1])


def tb_fit(b, T_ns):
    b = np.ascontiguousarray(b, dtype=np.float64)
    T = np.ascontiguousarray(T_ns, dtype=np.float64)
    od = np.zeros(5, np.float64)
    oi = np.zeros(5, np.int64)
    lib().oracle_tb_fit(len(b), _p(b, P_f64), _p(T, P_f64), _p(od, P_f64), _p(oi, P_i64))
    return dict(ok=bool(oi[0]), b_star=int(oi[1]), t0=od[0], k0=od[1], k1=od[2], t1=od[3], sse=od[4],
                profile=(int(oi[2]), int(oi[3]), int(oi[1]), int(oi[4])))


def min_merge_gain(profile, bmax: int):
    out = np.zeros(4, np.int64)
    lib().oracle_tb_min_merge_gain(_p(_prof(profile), P_i64), int(bmax), _p(out, P_i64))
    return _i128(out[0], out[1]), int(out[2]), int(out[3])


# ------------------------------------------------------------------ C4
def brute_force(d, B: int, profile):
    d = np.ascontiguousarray(d, dtype=np.int32)
    out = np.zeros(6, np.int64)
    lib().oracle_brute_force(len(d), _p(d, P_i32), int(B), _p(_prof(profile), P_i64), _p(out, P_i64))
    return dict(lf_time=_i128(out[0], out[1]), opt_time=_i128(out[2], out[3]), lf_iters=int(out[4]),
                opt_iters_min=int(out[5]))


def run_order(d, order, B: int, profile):
    d = np.ascontiguousarray(d, dtype=np.int32)
    o = np.ascontiguousarray(order, dtype=np.int32)
    out = np.zeros(3, np.int64)
    lib().oracle_run_order(len(d), _p(d, P_i32), _p(o, P_i32), int(B), _p(_prof(profile), P_i64),
                           _p(out, P_i64))
    return _i128(out[0], out[1]), int(out[2])


# ------------------------------------------------------------------ C2
def sched_sim(ids, P, d, hint, B: int, page: int, pool_pages: int, batch=None, arrival_after=None,
              profile=None, group=None):
    """Returns dict(iters=[...], samples={id: {...}}, n_iters, time_ps).  group: prefix-sharing group
    per sample (-1: none; NEXT-3, reading R26)."""
    n = len(ids)
    ids = np.ascontiguousarray(ids, np.int64)
    P = np.ascontiguousarray(P, np.int32)
    d = np.ascontiguousarray(d, np.int32)
    hint = np.ascontiguousarray(hint, np.int32)
    bt = None if batch is None else np.ascontiguousarray(batch, np.int32)
    ar = None if arrival_after is None else np.ascontiguousarray(arrival_after, np.int64)
    tp = np.zeros(2, np.int64)
    prof = None if profile is None else _prof(profile)
    gr = None if group is None else np.ascontiguousarray(group, np.int64)
    L = lib()
    nit = L.oracle_sched_sim(n, _p(ids, P_i64), _p(P, P_i32), _p(d, P_i32), _p(hint, P_i32),
                             None if bt is None else _p(bt, P_i32), None if ar is None else _p(ar, P_i64),
                             int(B), int(page), int(pool_pages), None if prof is None else _p(prof, P_i64),
                             _p(tp, P_i64), None if gr is None else _p(gr, P_i64))
    if nit < 0:
        raise RuntimeError(L.oracle_last_error().decode())
    blobs = []
    for which in (0, 1):
        m = L.oracle_sched_blob(which, None)
        b = np.zeros(m, np.int64)
        L.oracle_sched_blob(which, _p(b, P_i64))
        blobs.append(b)
    return dict(iters=parse_iter_blob(blobs[0]), samples=parse_sample_blob(blobs[1]), n_iters=int(nit),
                time_ps=_i128(tp[0], tp[1]), iter_blob=blobs[0], sample_blob=blobs[1])


def parse_iter_blob(b):
    """Iteration records: t, b, sumctx, nadm, ncomp, nalloc, nfree, adm..., comp..., alloc..., free..."""
    out, i = [], 0
    b = [int(x) for x in b]
    while i < len(b):
        t, bb, sc, na, nc, nal, nfr = b[i:i + 7]
        i += 7
        adm = b[i:i + na]; i += na
        comp = b[i:i + nc]; i += nc
        al = b[i:i + nal]; i += nal
        fr = b[i:i + nfr]; i += nfr
        out.append(dict(t=t, b=bb, sumctx=sc, admitted=adm, completed=comp, alloc=al, freed=fr))
    return out


def parse_sample_blob(b):
    out, i = {}, 0
    b = [int(x) for x in b]
    while i < len(b):
        sid, slot, adm, fin, npg = b[i:i + 5]
        i += 5
        out[sid] = dict(slot=slot, admit=adm, finish=fin, pages=b[i:i + npg])
        i += npg
    return out


# ------------------------------------------------------------------ C5
def dispatch(ids, P, hint, N: int, B: int, page: int, pool_pages: int, profile, alpha_pct=20, score_max=0,
             tail_ceil=0):
    n = len(ids)
    ids = np.ascontiguousarray(ids, np.int64)
    P = np.ascontiguousarray(P, np.int32)
    hint = np.ascontiguousarray(hint, np.int32)
    inst = np.zeros(n, np.int32)
    info = np.zeros(8, np.int64)
    sc = np.zeros(2 * max(N, 1), np.int64)
    lib().oracle_dispatch(n, _p(ids, P_i64), _p(P, P_i32), _p(hint, P_i32), N, B, page, pool_pages,
                          _p(_prof(profile), P_i64), alpha_pct, score_max, tail_ceil, _p(inst, P_i32),
                          _p(info, P_i64), _p(sc, P_i64))
    nsc = int(info[6])
    return dict(instance=inst, n_l=int(info[0]), n_tail=int(info[1]), L_alpha=int(info[2]), L_r=int(info[3]),
                score=_i128(info[4], info[5]), scores=[_i128(sc[2 * i], sc[2 * i + 1]) for i in range(nsc)])


def elastic_plan(ids, P, hint, N: int, B: int, page: int, pool_pages: int, profile, delta_ps: int, alpha_pct=20,
                 score_max=0, tail_ceil=0):
    """NEXT-4: predicted generation ps on N and N+1 instances, delta' and the decision."""
    n = len(ids)
    ids = np.ascontiguousarray(ids, np.int64)
    P = np.ascontiguousarray(P, np.int32)
    hint = np.ascontiguousarray(hint, np.int32)
    out = np.zeros(6, np.int64)
    dec = lib().oracle_elastic_plan(n, _p(ids, P_i64), _p(P, P_i32), _p(hint, P_i32), N, B, page, pool_pages,
                                    _p(_prof(profile), P_i64), alpha_pct, score_max, tail_ceil, int(delta_ps),
                                    _p(out, P_i64))
    return dict(t_gen_ps=(_i128(out[0], out[1]), _i128(out[2], out[3])), delta_prime_ps=_i128(out[4], out[5]),
                scale_out=bool(dec))


def tp_tail_plan(ids, P, hint, N: int, B: int, page: int, pool_pages: int, profile, tp_size: int, tp_B: int,
                 tp_pool_pages: int, tp_profile, policy="round_robin", alpha_pct=20, score_max=0, tail_ceil=0,
                 kv_ps=0, tp_kv_ps=0, pf_ps=0, tp_pf_ps=0):
    """NEXT-2 two-dimensional dispatch (reading R27): k longest to one TP instance, predicted times."""
    n = len(ids)
    ids = np.ascontiguousarray(ids, np.int64)
    P = np.ascontiguousarray(P, np.int32)
    hint = np.ascontiguousarray(hint, np.int32)
    out = np.zeros(6, np.int64)
    k = lib().oracle_tp_tail_plan(n, _p(ids, P_i64), _p(P, P_i32), _p(hint, P_i32), N, B, page, pool_pages,
                                  _p(_prof(profile), P_i64), alpha_pct, score_max, tail_ceil,
                                  {"skew": 0, "round_robin": 1}[policy], tp_size, tp_B, tp_pool_pages,
                                  _p(_prof(tp_profile), P_i64), int(kv_ps), int(tp_kv_ps), int(pf_ps), int(tp_pf_ps),
                                  _p(out, P_i64))
    return dict(n_tail=int(k), t_tp_ps=_i128(out[0], out[1]), t_dp_ps=_i128(out[2], out[3]),
                t_all_ps=_i128(out[4], out[5]))


def nearest_rank(v, q_pct):
    v = np.ascontiguousarray(v, np.int64)
    return int(lib().oracle_nearest_rank(len(v), _p(v, P_i64), int(q_pct)))


# ------------------------------------------------------------------ C6-C8, K11
def bf16_round(x: float) -> float:
    return float(lib().oracle_bf16_round(float(x)))


def attention(q, K, V):
    """q [nq, hd], K/V [ctx, nkv, hd] float32 arrays of bf16 values -> o [nq, hd] float64."""
    q = np.ascontiguousarray(q, np.float32)
    K = np.ascontiguousarray(K, np.float32)
    V = np.ascontiguousarray(V, np.float32)
    nq, hd = q.shape
    ctx, nkv, _ = K.shape
    out = np.zeros((nq, hd), np.float64)
    lib().oracle_attention(nq, nkv, hd, ctx, _p(q, P_f32), _p(K, P_f32), _p(V, P_f32), _p(out, P_f64))
    return out


def gen_tensor(seed: int, tensor_id: int, n: int, is_norm: bool = False):
    out = np.zeros(n, np.float32)
    lib().oracle_gen_tensor(seed, tensor_id, n, int(is_norm), _p(out, P_f32))
    return out


def tensor_checksum(seed: int, tensor_id: int, n: int, is_norm: bool = False) -> int:
    return int(lib().oracle_tensor_checksum(seed, tensor_id, n, int(is_norm)))


def weight_hash(seed, tensor_id, i):
    return int(lib().oracle_weight_hash(seed, tensor_id, i))


def decoder_forward(shape, seed: int, tokens, first_row: int):
    """Teacher-forced logits for rows first_row..T-1 -> float64 [T-first_row, V]."""
    toks = np.ascontiguousarray(tokens, np.int32)
    T = len(toks)
    ci = np.array([shape.n_layers, shape.d_model, shape.n_q_heads, shape.n_kv_heads, shape.head_dim,
                   shape.d_ffn, shape.vocab], np.int32)
    cd = np.array([shape.rms_eps, shape.rope_theta], np.float64)
    out = np.zeros((T - first_row, shape.vocab), np.float64)
    rc = lib().oracle_decoder_forward(_p(ci, P_i32), _p(cd, P_f64), seed, _p(toks, P_i32), T, first_row,
                                      _p(out, P_f64))
    if rc != 0:
        raise RuntimeError(lib().oracle_last_error().decode())
    return out


def rmsnorm(x, w, eps):
    """y = bf16(x / sqrt(mean(x^2) + eps) * w) row-wise; x [T, d] -> float64 [T, d] of bf16 values."""
    x = np.ascontiguousarray(x, np.float64)
    w = np.ascontiguousarray(w, np.float32)
    T, d = x.shape
    y = np.zeros_like(x)
    lib().oracle_rmsnorm(_p(x, P_f64), _p(w, P_f32), T, d, eps, _p(y, P_f64))
    return y


def rope(v, pos: int, theta: float):
    """NeoX rotate-half RoPE of one head vector (fp64)."""
    v = np.array(v, np.float64)
    lib().oracle_rope(_p(v, P_f64), len(v), int(pos), theta)
    return v


def decoder_dump(shape, seed: int, tokens):
    """Residual stream after the embedding and after each residual add: [2L+1, T, d] float64."""
    toks = np.ascontiguousarray(tokens, np.int32)
    T = len(toks)
    ci = np.array([shape.n_layers, shape.d_model, shape.n_q_heads, shape.n_kv_heads, shape.head_dim,
                   shape.d_ffn, shape.vocab], np.int32)
    cd = np.array([shape.rms_eps, shape.rope_theta], np.float64)
    out = np.zeros((2 * shape.n_layers + 1, T, shape.d_model), np.float64)
    if lib().oracle_decoder_dump(_p(ci, P_i32), _p(cd, P_f64), seed, _p(toks, P_i32), T, _p(out, P_f64)) != 0:
        raise RuntimeError(lib().oracle_last_error().decode())
    return out


def decoder_layer(shape, seed: int, layer: int, h_in):
    """One decoder layer on the residual stream h_in [T, d] (positions 0..T-1) -> [T, d] float64."""
    h = np.ascontiguousarray(h_in, np.float64)
    ci = np.array([shape.n_layers, shape.d_model, shape.n_q_heads, shape.n_kv_heads, shape.head_dim,
                   shape.d_ffn, shape.vocab], np.int32)
    cd = np.array([shape.rms_eps, shape.rope_theta], np.float64)
    out = np.zeros_like(h)
    lib().oracle_decoder_layer(_p(ci, P_i32), _p(cd, P_f64), seed, layer, _p(h, P_f64), h.shape[0], _p(out, P_f64))
    return out


def decoder_head(shape, seed: int, h_in):
    """Final RMSNorm + LM head on the residual stream h_in [T, d] -> logits [T, V] float64."""
    h = np.ascontiguousarray(h_in, np.float64)
    ci = np.array([shape.n_layers, shape.d_model, shape.n_q_heads, shape.n_kv_heads, shape.head_dim,
                   shape.d_ffn, shape.vocab], np.int32)
    cd = np.array([shape.rms_eps, shape.rope_theta], np.float64)
    out = np.zeros((h.shape[0], shape.vocab), np.float64)
    lib().oracle_decoder_head(_p(ci, P_i32), _p(cd, P_f64), seed, _p(h, P_f64), h.shape[0], _p(out, P_f64))
    return out


def weight_cache(on: bool):
    """Memoise generated weight tensors (same values; timing runs build the weights once)."""
    lib().oracle_weight_cache(int(on))


def argmax(x) -> int:
    x = np.ascontiguousarray(x, np.float32)
    return int(lib().oracle_argmax(_p(x, P_f32), len(x)))


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().oracle_philox(_p(c, P_u32), _p(k, P_u32), _p(out, P_u32))
    return [int(v) for v in out]


def sample_top_p(logits, temperature, top_p, seed, sample_id, step) -> int:
    x = np.ascontiguousarray(logits, np.float32)
    return int(lib().oracle_sample_top_p(_p(x, P_f32), len(x), temperature, top_p, seed, sample_id, step))
