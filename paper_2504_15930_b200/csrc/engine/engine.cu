// Engine: one SGS generation instance on one B200.
//
// Per iteration (sgs_step): the host scheduler decides admissions (longest
// first), page allocations and completions; the engine stages all
// per-iteration metadata in one pinned buffer (one H2D copy), then runs
//   prefill of the admitted prompts (chunks of <= max_prefill_tokens):
//     embed -> L x [RMSNorm, QKV GEMM, RoPE+KV append, causal attention,
//                   O GEMM (+residual), RMSNorm, gate/up GEMM, SwiGLU,
//                   down GEMM (+residual)] -> final norm on the last token
//     -> LM head -> greedy sample (token 1)
//   decode of the running samples (one token each):
//     same chain with paged split-K decode attention
// and streams the completed samples back.  The residual stream is
// fp32; every other activation is bf16 (R12).
#include "engine.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "nccl.h"

namespace sgs {

static inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// NEXT-2: the dims of tensor-parallel shard (q/kv heads, FFN, vocab rows / tp)
static sgs_model_cfg tp_local(const sgs_model_cfg& m, const sgs_engine_cfg& e) {
  const int tp = e.tp_size > 1 ? e.tp_size : 1;
  sgs_model_cfg l = m;
  l.n_q_heads /= tp, l.n_kv_heads /= tp, l.d_ffn /= tp, l.vocab /= tp;
  return l;
}

sgs_status Engine::layout(const sgs_model_cfg& m_full, const sgs_engine_cfg& e, int64_t n_pages, ArenaLayout* L) {
  const sgs_model_cfg m = tp_local(m_full, e);
  const int64_t d = m.d_model, hd = m.head_dim, nq = m.n_q_heads, nkv = m.n_kv_heads, f = m.d_ffn, V = m.vocab;
  const int64_t V_full = m_full.vocab;
  const int64_t B = e.max_batch;
  const int64_t pf = e.max_prefill_tokens > 0 ? e.max_prefill_tokens : 16384;
  const int64_t tmax = std::max<int64_t>(pf, B);
  const int64_t page = e.page_size;
  const int64_t max_pages = (e.max_ctx + page - 1) / page + 1;
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  // weights (contiguous so the weight sync can broadcast one range)
  const int64_t per_layer = ((nq + 2 * nkv) * hd * d + (nq + 2 * nkv) * hd + d * nq * hd + 2 * f * d + d * f + 2 * d);
  const int64_t wbytes = (m.n_layers * per_layer + (V + V_full) * d + d) * 2;
  take(wbytes + 256 * (8 * m.n_layers + 8));
  L->weights_bytes = o;
  L->kv_page_bytes = m.n_layers * nkv * 2 * page * hd * 2;
  L->off_kv = take(n_pages * L->kv_page_bytes);
  L->kv_bytes = n_pages * L->kv_page_bytes;
  const int64_t s0 = o;
  L->off_h = take(tmax * d * 4);
  L->off_x = take(tmax * d * 2);
  L->off_qkv = take(tmax * (nq + 2 * nkv) * hd * 4);
  L->off_q = take(tmax * nq * hd * 2);
  L->off_kc = take(tmax * nkv * hd * 2);
  L->off_vc = take(tmax * nkv * hd * 2);
  L->off_ao = take(tmax * nq * hd * 2);
  L->off_gu = take(tmax * 2 * f * 4);
  L->off_mm = take(tmax * f * 2);
  {
    const int64_t Bp = (B + 15) / 16 * 16;
    L->off_dh = take(Bp * d * 4);
    L->off_dx = take(Bp * d * 2);
    L->off_dqkv = take(Bp * (nq + 2 * nkv) * hd * 4);
    L->off_dq = take(Bp * nq * hd * 2);
    L->off_dao = take(Bp * nq * hd * 2);
    L->off_dgu = take(Bp * 2 * f * 4);
    L->off_dmm = take(Bp * f * 2);
  }
  // decode rows [0, Bpad) (CUDA-graph buckets pad to 16), prefill rows after them
  const int64_t Bpad = (B + 15) / 16 * 16;
  L->off_logits = take((Bpad + B) * V * 4);
  L->off_rope = take((int64_t)(e.max_ctx + 1) * (hd / 2) * 2 * 4);
  L->off_bt = take(B * max_pages * 4);
  L->off_last = take(B * 4);
  L->off_hist = take(B * (int64_t)(e.max_ctx + 1) * 4);
  // per-iteration metadata: bt deltas, prefill tokens/pos/slot, decode rows, attention work lists
  // attention work list bound of attn_plan: 2*148 + b*nkv (+ slack)
  const int64_t max_items = 2 * 148 + Bpad * nkv + 64;
  // fixed decode region (graph-replayable): counts[4] | slot,pos,ctx,tok [Bpad] | sample id (lo,hi) [Bpad]
  // | combs | items
  L->meta_dec_bytes = align_up(4 * (4 + 6 * Bpad) + max_items * (int64_t)(sizeof(AttnItem) + sizeof(AttnComb)), 256);
  // prefill tokens of one iteration: up to B admitted prompts of <= min(max_ctx, prefill chunk) tokens
  const int64_t adm_tok = B * std::min<int64_t>(e.max_ctx, pf);
  L->meta_bytes = L->meta_dec_bytes +
                  align_up(4 * (3 * (B * max_pages + B) + 3 * adm_tok + 8 * B + 2 * (adm_tok / 64 + 2 * B) + 16 * B) +
                               4096,
                           256);
  L->off_meta = take(L->meta_bytes);
  L->attn_bytes = max_items * (nq / nkv) * (hd + 2) * 4 + max_items * 4;  // partials + arrival counters
  L->off_attn = take(L->attn_bytes);
  L->off_cksum = take(64);
  L->off_amax = take(((B + 15) / 16 * 16) * 8 + 64 + B * 8);
  L->off_nbar = take((2 * m.n_layers + 1) * 2 * 4 + 64);
  L->scratch_bytes = o - s0;
  L->off_shadow = (e.flags & SGS_F_SHADOW_WEIGHTS) ? take(L->weights_bytes) : -1;
  L->total = o;
  L->tmax = (int)tmax;
  L->max_pages = (int)max_pages;
  L->max_items = (int)max_items;
  return SGS_OK;
}

sgs_status Engine::cuda_fail(cudaError_t e, const char* what) {
  err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  poisoned = true;
  return SGS_E_CUDA;
}

#define CK(call, what)                                  \
  do {                                                  \
    cudaError_t e__ = (call);                           \
    if (e__ != cudaSuccess) return cuda_fail(e__, what); \
  } while (0)

Engine::~Engine() {
  if (!null_) {
    if (st_) cudaStreamSynchronize(st_);
    for (int k = 0; k < 2; ++k) {
      if (meta_bufs_[k]) cudaFreeHost(meta_bufs_[k]);
      if (tok_bufs_[k]) cudaFreeHost(tok_bufs_[k]);
      if (ev0s_[k]) cudaEventDestroy(ev0s_[k]);
      if (ev1s_[k]) cudaEventDestroy(ev1s_[k]);
    }
    if (st_side_) {
      cudaStreamSynchronize(st_side_);
      cudaStreamDestroy(st_side_);
    }
    if (ev_sync_) cudaEventDestroy(ev_sync_);
    if (ev_commit_) cudaEventDestroy(ev_commit_);
    if (st_pf_) {
      cudaStreamSynchronize(st_pf_);
      cudaStreamDestroy(st_pf_);
    }
    if (ev_meta_) cudaEventDestroy(ev_meta_);
    if (ev_pf_) cudaEventDestroy(ev_pf_);
    for (auto& v : graphs_)
      for (auto& g : v)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto& kv : pgraphs_)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    for (void* p : xch_peer_) cudaIpcCloseMemHandle(p);
    if (xch_) cudaFree(xch_);
  }
}

void Engine::build_tensor_table() {
  tensors_.clear();
  const int64_t d = m_.d_model, hd = m_.head_dim, nq = m_.n_q_heads, nkv = m_.n_kv_heads, f = m_.d_ffn;
  const int64_t r = tp_rank_, tp = tp_;
  // shard windows of the full tensors (identity without TP): rows for the
  // column-parallel QKV / gate / up / LM head, columns for the row-parallel O / down
  auto rows_win = [&](int64_t row0, int64_t cols) { return tp > 1 ? ShardMap{cols, row0, 0, cols} : ShardMap{}; };
  auto cols_win = [&](int64_t src_cols, int64_t col0, int64_t lcols) {
    return tp > 1 ? ShardMap{src_cols, 0, col0, lcols} : ShardMap{};
  };
  tensors_.push_back({0, embed_, vocab_full_ * d, 0});
  // GEMM weights: row-major, or (w_tiled_) the tiled layout of their fused
  // matrix; a tensor at row R0 of a fused matrix is placed with blk = its
  // rows, stride 0, off = R0 (kernels.h weight placement)
  const int tl = w_tiled_;
  auto gemm_w = [&](int64_t id, void* base, int64_t rows, int64_t k, int64_t r0, ShardMap sm) {
    if (tl) return TensorRef{id, base, rows * k, 0, k, (int)rows, 0, (int)r0, sm, 1};
    return TensorRef{id, (void*)((uint16_t*)base + r0 * k), rows * k, 0, 1, 0, 0, 0, sm, 0};
  };
  tensors_.push_back(gemm_w(1, lm_head_, m_.vocab, d, 0, rows_win(r * m_.vocab, d)));
  tensors_.push_back({2, nf_, d, 1});
  for (int l = 0; l < m_.n_layers; ++l) {
    const int64_t b = 16 + 16 * (int64_t)l;
    auto* L = &layers_[l];
    auto at = [](void* p, int64_t elems) { return (void*)((uint16_t*)p + elems); };
    tensors_.push_back(gemm_w(b + 0, L->wqkv, nq * hd, d, 0, rows_win(r * nq * hd, d)));
    tensors_.push_back(gemm_w(b + 1, L->wqkv, nkv * hd, d, nq * hd, rows_win(r * nkv * hd, d)));
    tensors_.push_back(gemm_w(b + 2, L->wqkv, nkv * hd, d, (nq + nkv) * hd, rows_win(r * nkv * hd, d)));
    tensors_.push_back({b + 3, L->bqkv, nq * hd, 0, 1, 0, 0, 0, rows_win(r * nq * hd, 1)});
    tensors_.push_back({b + 4, at(L->bqkv, nq * hd), nkv * hd, 0, 1, 0, 0, 0, rows_win(r * nkv * hd, 1)});
    tensors_.push_back({b + 5, at(L->bqkv, (nq + nkv) * hd), nkv * hd, 0, 1, 0, 0, 0, rows_win(r * nkv * hd, 1)});
    tensors_.push_back(gemm_w(b + 6, L->wo, d, nq * hd, 0, cols_win(nq * hd * tp, r * nq * hd, nq * hd)));
    // gate and up interleave in 64-row blocks: tile i of the fused matrix = 64 gate rows + 64 up rows
    tensors_.push_back({b + 7, L->wgu, f * d, 0, d, 64, 128, 0, rows_win(r * f, d), tl});
    tensors_.push_back({b + 8, L->wgu, f * d, 0, d, 64, 128, 64, rows_win(r * f, d), tl});
    tensors_.push_back(gemm_w(b + 9, L->wd, d, f, 0, cols_win(f * tp, r * f, f)));
    tensors_.push_back({b + 10, L->n1, d, 1});
    tensors_.push_back({b + 11, L->n2, d, 1});
  }
}

sgs_status Engine::init(const sgs_model_cfg& m_full, const sgs_engine_cfg& e, const sgs_weights* w) {
  tp_ = e.tp_size > 1 ? e.tp_size : 1;
  tp_rank_ = tp_ > 1 ? e.tp_rank : 0;
  vocab_full_ = m_full.vocab;
  if (tp_ > 1) {
    if (e.tp_rank < 0 || e.tp_rank >= tp_ || m_full.n_q_heads % tp_ || m_full.n_kv_heads % tp_ ||
        m_full.d_ffn % tp_ || m_full.vocab % tp_) {
      err = "tensor parallelism: tp_rank out of range or heads / FFN / vocab not divisible by tp_size";
      return SGS_E_INVAL;
    }
    if (w || e.sampling != SGS_SAMPLE_GREEDY || e.device < 0) {
      err = "tensor-parallel shards generate their weights (weights == NULL), decode greedily, need a device";
      return SGS_E_UNSUPPORTED;
    }
  }
  const sgs_model_cfg m = tp_local(m_full, e);
  m_ = m;
  e_ = e;
  if (e_.max_prefill_tokens <= 0) e_.max_prefill_tokens = 16384;
  if (m.n_layers <= 0 || m.d_model <= 0 || m.n_q_heads <= 0 || m.n_kv_heads <= 0 || m.head_dim <= 0 ||
      m.d_ffn <= 0 || m.vocab <= 0 || e.max_batch <= 0 || e.page_size <= 0 || e.max_ctx <= 0 ||
      e.n_instances <= 0 || e.instance_rank < 0 || e.instance_rank >= e.n_instances ||
      m.n_q_heads % m.n_kv_heads) {
    err = "invalid model/engine configuration";
    return SGS_E_INVAL;
  }
  null_ = e.device < 0;
  if (const char* sk = std::getenv("SGS_DEBUG_SKIP")) skip_ = std::atoi(sk);
  max_gen_ = e.max_ctx + 1;
  sched.tracing = (e.flags & SGS_F_TRACE) != 0;
  if (null_) {
    n_pages_ = e.n_pages;
    if (n_pages_ <= 0) {
      err = "null-device mode needs n_pages > 0";
      return SGS_E_INVAL;
    }
    sched.init(e.max_batch, e.page_size, n_pages_);
    sched.tracing = (e.flags & SGS_F_TRACE) != 0;
    return SGS_OK;
  }
  // ---- device mode: shape support of the sm_100a kernels
  if (e.page_size != 16 || !(m.head_dim == 32 || m.head_dim == 64 || m.head_dim == 128) ||
      m.n_q_heads / m.n_kv_heads > 8 || m.d_model % 128 || m.d_ffn % 128 || m.vocab % 128 ||
      ((m.n_q_heads + 2 * m.n_kv_heads) * m.head_dim) % 128 || (m.n_q_heads * m.head_dim) % 64) {
    err = "shape not supported by the sm_100a kernels (page 16, hd 32/64/128, GQA group <= 8, dims multiple of 128)";
    return SGS_E_UNSUPPORTED;
  }
  CK(cudaSetDevice(e.device), "cudaSetDevice");
  st_ = reinterpret_cast<cudaStream_t>(e.stream);
  ArenaLayout L0;
  layout(m_full, e_, 0, &L0);  // layout() applies tp_local itself
  n_pages_ = e.n_pages;
  if (n_pages_ <= 0) n_pages_ = (e.arena_bytes - L0.total - 4096) / L0.kv_page_bytes;
  if (n_pages_ <= 0) {
    err = "arena too small for weights + scratch";
    return SGS_E_NOMEM;
  }
  layout(m_full, e_, n_pages_, &L_);
  if (!e.arena || e.arena_bytes < L_.total) {
    err = "arena smaller than sgs_arena_bytes()";
    return SGS_E_NOMEM;
  }
  arena_ = reinterpret_cast<uint8_t*>(e.arena);
  // carve weights
  {
    const int64_t d = m.d_model, hd = m.head_dim, nq = m.n_q_heads, nkv = m.n_kv_heads, f = m.d_ffn;
    int64_t o = 0;
    auto w = [&](int64_t elems) {
      void* p = arena_ + o;
      o = align_up(o + elems * 2, 256);
      return p;
    };
    embed_ = w(vocab_full_ * d);
    lm_head_ = w((int64_t)m.vocab * d);
    nf_ = w(d);
    layers_.resize(m.n_layers);
    for (auto& l : layers_) {
      l.wqkv = w((nq + 2 * nkv) * hd * d);
      l.bqkv = w((nq + 2 * nkv) * hd);
      l.wo = w(d * nq * hd);
      l.wgu = w(2 * f * d);
      l.wd = w(d * f);
      l.n1 = w(d);
      l.n2 = w(d);
    }
    for (int i = 0; i < m.n_layers; ++i)
      layers_[i].kv = arena_ + L_.off_kv + (int64_t)i * n_pages_ * (L_.kv_page_bytes / m.n_layers);
  }
  h_ = reinterpret_cast<float*>(arena_ + L_.off_h);
  x_ = arena_ + L_.off_x;
  qkv_ = reinterpret_cast<float*>(arena_ + L_.off_qkv);
  q_ = arena_ + L_.off_q;
  kc_ = arena_ + L_.off_kc;
  vc_ = arena_ + L_.off_vc;
  ao_ = arena_ + L_.off_ao;
  gu_ = reinterpret_cast<float*>(arena_ + L_.off_gu);
  mm_ = arena_ + L_.off_mm;
  logits_ = reinterpret_cast<float*>(arena_ + L_.off_logits);
  dset_.h = reinterpret_cast<float*>(arena_ + L_.off_dh);
  dset_.x = arena_ + L_.off_dx;
  dset_.qkv = reinterpret_cast<float*>(arena_ + L_.off_dqkv);
  dset_.q = arena_ + L_.off_dq;
  dset_.ao = arena_ + L_.off_dao;
  dset_.gu = reinterpret_cast<float*>(arena_ + L_.off_dgu);
  dset_.mm = arena_ + L_.off_dmm;
  rope_ = reinterpret_cast<float*>(arena_ + L_.off_rope);
  bt_ = reinterpret_cast<int32_t*>(arena_ + L_.off_bt);
  last_tok_ = reinterpret_cast<int32_t*>(arena_ + L_.off_last);
  hist_ = reinterpret_cast<int32_t*>(arena_ + L_.off_hist);
  meta_dev_ = arena_ + L_.off_meta;
  attn_ws_ = arena_ + L_.off_attn;
  cksum_dev_ = reinterpret_cast<unsigned long long*>(arena_ + L_.off_cksum);
  amax_keys_ = reinterpret_cast<unsigned long long*>(arena_ + L_.off_amax);
  amax_keys_pf_ = amax_keys_ + ((e.max_batch + 15) / 16 * 16) + 8;
  norm_bar_ = reinterpret_cast<unsigned int*>(arena_ + L_.off_nbar);
  // PreNorm is off by default: measured slower than the rmsnorm kernel + PDL
  // (profiles/README.md r02: the norm and the grid barrier stay on the
  // critical path, only the launch is saved); SGS_FUSED_NORM=1 turns it on
  if (const char* nf = std::getenv("SGS_FUSED_NORM")) fused_norm_ = std::atoi(nf) != 0;
  // prefill attention: the tcgen05 kernel for hd 128 (128-query blocks), the
  // mma.sync kernel otherwise or with SGS_PREFILL_LEGACY=1 (64-query blocks)
  qblk_ = (m.head_dim == 128 && !(std::getenv("SGS_PREFILL_LEGACY") && std::atoi(std::getenv("SGS_PREFILL_LEGACY"))))
              ? 128
              : 64;
  tok_host_cap_ = (int64_t)e.max_batch * max_gen_;
  for (int k = 0; k < 2; ++k) {
    CK(cudaMallocHost(&meta_bufs_[k], L_.meta_bytes), "cudaMallocHost(meta)");
    CK(cudaMallocHost(&tok_bufs_[k], tok_host_cap_ * 4), "cudaMallocHost(tokens)");
    CK(cudaEventCreate(&ev0s_[k]), "event");
    CK(cudaEventCreate(&ev1s_[k]), "event");
  }
  meta_host_ = meta_bufs_[0], tok_host_ = tok_bufs_[0], ev0_ = ev0s_[0], ev1_ = ev1s_[0];
  if (L_.off_shadow >= 0) {
    shadow_ = arena_ + L_.off_shadow;
    CK(cudaStreamCreateWithFlags(&st_side_, cudaStreamNonBlocking), "side stream");
    CK(cudaEventCreateWithFlags(&ev_sync_, cudaEventDisableTiming), "event");
    CK(cudaEventCreateWithFlags(&ev_commit_, cudaEventDisableTiming), "event");
  }
  // zero the KV pool (finite garbage only beyond ctx) and the small state
  CK(cudaMemsetAsync(arena_ + L_.off_kv, 0, L_.kv_bytes, st_), "memset kv");
  CK(cudaMemsetAsync(bt_, 0, (size_t)e.max_batch * L_.max_pages * 4, st_), "memset bt");
  CK(cudaMemsetAsync(last_tok_, 0, (size_t)e.max_batch * 4, st_), "memset last");
  // split-K accumulators (kept zeroed by their consumers) and the residual scratch
  CK(cudaMemsetAsync(arena_ + L_.off_h, 0, L_.off_mm - L_.off_h, st_), "memset scratch");
  CK(cudaMemsetAsync(arena_ + L_.off_dh, 0, L_.off_dmm - L_.off_dh, st_), "memset decode scratch");
  CK(cudaStreamCreateWithFlags(&st_pf_, cudaStreamNonBlocking), "prefill stream");
  CK(cudaEventCreateWithFlags(&ev_meta_, cudaEventDisableTiming), "event");
  CK(cudaEventCreateWithFlags(&ev_pf_, cudaEventDisableTiming), "event");
  CK(cudaMemsetAsync(attn_ws_, 0, L_.attn_bytes, st_), "memset attention workspace");
  CK(cudaMemsetAsync(amax_keys_, 0, ((e.max_batch + 15) / 16 * 16) * 8 + 64 + e.max_batch * 8, st_),
     "memset argmax keys");
  CK(cudaMemsetAsync(norm_bar_, 0, (2 * m.n_layers + 1) * 2 * 4 + 64, st_), "memset norm barriers");
  // RoPE table: cos/sin of pos * theta^(-2i/hd) computed in fp64 on the host, stored fp32
  {
    const int half = m.head_dim / 2;
    std::vector<float> tab((size_t)(e.max_ctx + 1) * half * 2);
    sgs_rope_table(tab.data(), e.max_ctx + 1, m.head_dim, m.rope_theta);
    CK(cudaMemcpy(rope_, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice), "rope table");
  }
  // GEMM weight layout: row-major, or (SGS_WEIGHT_LAYOUT=tiles) tiled 16 KB
  // blocks, one contiguous 4-D TMA box each -- ~1% faster decode, but a decode
  // step stalled under torch.profiler (CUPTI) with it and never with row-major
  // weights, so it stays opt-in
  if (const char* wl = std::getenv("SGS_WEIGHT_LAYOUT")) w_tiled_ = std::string(wl) == "tiles" ? 1 : 0;
  build_tensor_table();
  sgs_status s = w ? load_weights(w, arena_, st_) : load_weights_seed(e.weight_seed);
  if (s != SGS_OK) return s;
  CK(cudaStreamSynchronize(st_), "init sync");
  sched.init(e.max_batch, e.page_size, n_pages_);
  sched.tracing = (e.flags & SGS_F_TRACE) != 0;
  return SGS_OK;
}

// Canonical order (sgs.h): embed, lm_head, final norm, then per layer Wq, Wk,
// Wv, bq, bk, bv, Wo, Wgate, Wup, Wdown, attention norm, MLP norm -- exactly
// the order of tensors_ (build_tensor_table).
sgs_status Engine::load_weights(const sgs_weights* w, uint8_t* base, cudaStream_t st) {
  if (null_) return SGS_OK;
  if (!w || !w->ptrs || w->n != (int32_t)tensors_.size()) {
    err = "sgs_weights: expected " + std::to_string(tensors_.size()) + " tensors in canonical order";
    return SGS_E_INVAL;
  }
  for (size_t i = 0; i < tensors_.size(); ++i)
    if (!w->ptrs[i]) {
      err = "sgs_weights: null tensor pointer at index " + std::to_string(i);
      return SGS_E_INVAL;
    }
  for (size_t i = 0; i < tensors_.size(); ++i) {
    const TensorRef& t = tensors_[i];
    uint8_t* dst = base + (reinterpret_cast<uint8_t*>(t.ptr) - arena_);
    if (t.tiled) {
      // canonical row-major source -> tiled placement by a kernel that reads the
      // source directly: device memory, or host memory page-locked for the copy
      const void* src = w->ptrs[i];
      const size_t bytes = (size_t)t.n * 2;
      cudaPointerAttributes pa{};
      bool reg = false;
      if (cudaPointerGetAttributes(&pa, src) != cudaSuccess) cudaGetLastError();
      if (pa.type == cudaMemoryTypeUnregistered) {
        CK(cudaHostRegister(const_cast<void*>(src), bytes, cudaHostRegisterMapped), "cudaHostRegister(weights)");
        reg = true;
      }
      void* dsrc = const_cast<void*>(src);
      if (pa.type == cudaMemoryTypeHost || reg) CK(cudaHostGetDevicePointer(&dsrc, const_cast<void*>(src), 0), "host pointer");
      CK(relayout_bf16(dsrc, dst, t.n, t.cols, t.blk, t.stride, t.off, 1, st), "weight relayout");
      if (reg) {
        CK(cudaStreamSynchronize(st), "weight relayout sync");
        CK(cudaHostUnregister(const_cast<void*>(src)), "cudaHostUnregister(weights)");
      }
    } else if (t.blk == 0) {
      CK(cudaMemcpyAsync(dst, w->ptrs[i], (size_t)t.n * 2, cudaMemcpyDefault, st), "weight copy");
    } else {
      // rows of 64 gate (or up) rows land every 128 rows of the fused matrix
      const size_t rowb = (size_t)t.cols * 2, rows = (size_t)(t.n / t.cols);
      CK(cudaMemcpy2DAsync(dst + (size_t)t.off * rowb, (size_t)t.stride * rowb, w->ptrs[i], (size_t)t.blk * rowb,
                           (size_t)t.blk * rowb, rows / t.blk, cudaMemcpyDefault, st),
         "weight copy (gate/up)");
    }
  }
  CK(cudaStreamSynchronize(st), "weight copy sync");  // the caller may free its buffers on return
  return SGS_OK;
}

sgs_status Engine::set_instances(int32_t n_instances, int32_t instance_rank) {
  if (!sched.idle() || !infl_.empty() || !ready_.empty()) {
    err = "the DP layout changes only between RL batches (nothing queued, in flight or unreturned)";
    return SGS_E_STATE;
  }
  e_.n_instances = n_instances;
  e_.instance_rank = instance_rank;
  return SGS_OK;
}

sgs_status Engine::load_weights_seed(uint64_t seed) {
  if (null_) return SGS_OK;
  for (const auto& t : tensors_) {
    CK(hash_init(t.ptr, seed, (uint64_t)t.id, t.n, t.is_norm, st_, t.cols, t.blk, t.stride, t.off, t.shard, t.tiled),
       "hash_init");
    ++launches;
  }
  CK(cudaStreamSynchronize(st_), "hash_init sync");
  return SGS_OK;
}

sgs_status Engine::checksum(int64_t tensor_id, uint64_t* out) {
  if (null_) {
    err = "no weights in null-device mode";
    return SGS_E_STATE;
  }
  for (const auto& t : tensors_)
    if (t.id == tensor_id) {
      CK(cudaMemsetAsync(cksum_dev_, 0, 8, st_), "memset");
      CK(checksum_bf16(t.ptr, t.n, cksum_dev_, st_, t.cols, t.blk, t.stride, t.off, t.tiled), "checksum");
      unsigned long long v = 0;
      CK(cudaMemcpyAsync(&v, cksum_dev_, 8, cudaMemcpyDeviceToHost, st_), "checksum d2h");
      CK(cudaStreamSynchronize(st_), "checksum sync");
      *out = v;
      return SGS_OK;
    }
  err = "unknown tensor id";
  return SGS_E_INVAL;
}

// ------------------------------------------------------------------ submit
sgs_status Engine::submit(const sgs_prompt* prompts, int32_t n, const int32_t* hint, const int32_t* forced,
                          int32_t* n_mine) {
  if (poisoned) {
    err = "handle poisoned by an earlier error";
    return SGS_E_STATE;
  }
  if (n < 0 || (n > 0 && (!prompts || !hint || !forced))) {
    err = "null arrays";
    return SGS_E_INVAL;
  }
  std::vector<uint64_t> ids(n);
  std::vector<int32_t> P(n);
  for (int i = 0; i < n; ++i) {
    const sgs_prompt& p = prompts[i];
    if (p.len < 1 || !p.tokens || hint[i] < 1 || forced[i] < 1) {
      err = "prompt length, hint and forced length must be >= 1";
      return SGS_E_INVAL;
    }
    for (int j = 0; j < p.len; ++j)
      if (p.tokens[j] < 0 || p.tokens[j] >= vocab_full_) {
        err = "token id out of range";
        return SGS_E_INVAL;
      }
    ids[i] = p.id;
    P[i] = p.len;
  }
  {
    std::vector<uint64_t> s(ids);
    std::sort(s.begin(), s.end());
    if (std::adjacent_find(s.begin(), s.end()) != s.end()) {
      err = "duplicate ids in batch";
      return SGS_E_INVAL;
    }
    for (uint64_t id : s)
      if (live_ids_.count(id)) {
        err = "id of a sample still queued or active on this handle";
        return SGS_E_INVAL;
      }
  }
  for (int i = 0; i < n; ++i) {
    const int64_t need = ((int64_t)P[i] + forced[i] - 1 + e_.page_size - 1) / e_.page_size;
    if ((int64_t)P[i] + forced[i] - 1 > e_.max_ctx || need > n_pages_ ||
        (!null_ && P[i] > e_.max_prefill_tokens)) {
      err = "sample can never fit (max_ctx, page pool or prefill chunk)";
      return SGS_E_CAPACITY;
    }
  }
  // Alg. 2 dispatch, identical on every instance (no communication)
  std::vector<int32_t> inst(n, 0);
  DispatchCfg dc{e_.n_instances, e_.max_batch, e_.page_size, n_pages_, e_.profile.t0_ns, e_.profile.k0_ps,
                 e_.profile.b_star, e_.profile.k1_ps, e_.alpha_pct, e_.score, e_.tail_ceil, e_.dispatch,
                 e_.sample_seed + (uint64_t)batch_counter_};
  dispatch_alg2(dc, n, ids.data(), P.data(), hint, inst.data());
  std::vector<Sample> mine;
  // NEXT-3: identical prompts of this batch on this instance form a prefix group
  std::map<std::vector<int32_t>, std::vector<int>> same_prompt;
  if (e_.flags & SGS_F_PREFIX_SHARING)
    for (int i = 0; i < n; ++i)
      if (inst[i] == e_.instance_rank)
        same_prompt[std::vector<int32_t>(prompts[i].tokens, prompts[i].tokens + P[i])].push_back(i);
  std::vector<int64_t> group_of(n, -1);
  {
    int64_t gi = 0;
    for (const auto& kv : same_prompt) {
      if (kv.second.size() >= 2)
        for (int i : kv.second) group_of[i] = ((int64_t)batch_counter_ << 32) | gi;
      ++gi;
    }
  }
  for (int i = 0; i < n; ++i) {
    if (inst[i] != e_.instance_rank) continue;
    Sample s;
    s.id = ids[i];
    s.P = P[i];
    s.d = forced[i];
    s.hint = hint[i];
    s.batch = batch_counter_;
    s.prompt.assign(prompts[i].tokens, prompts[i].tokens + P[i]);
    s.group = group_of[i];
    live_ids_.insert(s.id);
    mine.push_back(std::move(s));
  }
  if (n_mine) *n_mine = (int32_t)mine.size();
  sched.submit(std::move(mine));
  ++batch_counter_;
  return SGS_OK;
}

// ------------------------------------------------------------------ step
sgs_status Engine::step(sgs_completion* out, int32_t cap, int32_t* n_out) {
  *n_out = 0;
  if (poisoned) {
    err = "handle poisoned by an earlier error";
    return SGS_E_STATE;
  }
  if (tp_ > 1 && !tp_comm_) {
    err = "tensor-parallel handle without sgs_tp_comm_init";
    return SGS_E_STATE;
  }
  handed_.clear();
  if (ready_.empty()) {
    IterPlan plan;
    bool ran;
    try {
      ran = sched.plan(&plan);
    } catch (const std::exception& ex) {
      err = ex.what();
      poisoned = true;
      return SGS_E_STATE;
    }
    if (ran) {
      sgs_status s = run_iteration(plan);  // launches; finalizes it too unless pipelined
      if (s != SGS_OK) return s;
    }
    // the previous iteration (launched by the last call) is waited for only now,
    // while the GPU already runs this one; with nothing new to run, drain
    while (infl_.size() > (ran ? 1u : 0u)) {
      sgs_status s = finalize_front();
      if (s != SGS_OK) return s;
    }
  }
  int k = 0;
  while (k < cap && !ready_.empty()) {
    handed_.push_back(std::move(ready_.front()));
    ready_.pop_front();
    ++k;
  }
  for (int i = 0; i < k; ++i) {
    const Completion& c = handed_[i];
    out[i].id = c.id;
    out[i].instance = e_.instance_rank;
    out[i].n_tokens = (int32_t)c.tokens.size();
    out[i].tokens = c.tokens.data();
    out[i].admit_iter = c.admit_iter;
    out[i].finish_iter = c.finish_iter;
    out[i].weight_version = c.version;
    out[i].slot = c.slot;
  }
  *n_out = k;
  return SGS_OK;
}

cudaEvent_t Engine::next_event() {
  if (ev_used_ == ev_pool_.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ev_pool_.push_back(e);
  }
  return ev_pool_[ev_used_++];
}

void Engine::ktic(KRec* r, int cls) {
  r->cls = -1;
  if (!timing_now_) return;
  r->cls = cls;
  if (rec_target_) {  // capturing: events owned by the graph
    cudaEventCreate(&r->a);
    cudaEventCreate(&r->b);
  } else {
    r->a = next_event();
    r->b = next_event();
  }
  // inside a capture the record must be an external event-record node to be replayed
  cudaEventRecordWithFlags(r->a, st_, rec_target_ ? cudaEventRecordExternal : cudaEventRecordDefault);
}

void Engine::ktoc(KRec* r, double bfix, double brow, double frow, int rows) {
  if (r->cls < 0) return;
  cudaEventRecordWithFlags(r->b, st_, rec_target_ ? cudaEventRecordExternal : cudaEventRecordDefault);
  r->bfix = bfix;
  r->brow = brow;
  r->frow = frow;
  r->rows = rec_target_ ? -1 : rows;
  (rec_target_ ? *rec_target_ : krec_).push_back(*r);
}

// after a stream synchronize: fold kernel timings into the stats
cudaError_t Engine::kflush(const std::vector<KRec>& recs, int rows) {
  for (const KRec& r : recs) {
    float ms = 0.f;
    cudaError_t e = cudaEventElapsedTime(&ms, r.a, r.b);
    if (e != cudaSuccess) return e;
    const int n = r.rows < 0 ? rows : r.rows;
    const double by = r.bfix < 0 ? cur_attn_bytes_ : r.bfix + r.brow * n;
    const double fl = r.bfix < 0 ? cur_attn_flops_ : r.frow * n;
    auto add = [&](int k) {
      kstat_ms[k] += ms;
      kstat_bytes[k] += by;
      kstat_flops[k] += fl;
      if (roof_bw_gbs > 0 && roof_tflops > 0)
        kstat_roof_ms[k] += std::max(by / (roof_bw_gbs * 1e6), fl / (roof_tflops * 1e9));
      kstat_n[k] += 1;
    };
    add(r.cls);
    if (cur_phase_) add(r.cls + kClasses * cur_phase_);
  }
  return cudaSuccess;
}

cudaError_t Engine::gemm(const void* W, const void* X, float* C, int N, int K, int T, bool accumulate,
                         const PreNorm* pn) {
  // SGS_F_DETERMINISTIC: no split-K (the fp32 red.add order is the only run-to-run variation, R21)
  const int splits = (e_.flags & SGS_F_DETERMINISTIC) ? 1 : gemm_auto_splits(N, K, T);
  cudaError_t e;
  KRec kr;
  ktic(&kr, gemm_cls_);
  if (splits > 1) {
    // qkv_ and gu_ are kept zeroed by their consumers (rope_append, silu_mul)
    if (!accumulate && C != qkv_ && C != gu_) {
      e = cudaMemsetAsync(C, 0, (size_t)T * N * 4, st_);
      if (e != cudaSuccess) return e;
    }
    e = gemm_bf16(W, X, C, N, K, T, N, 1, splits, st_, nullptr, pn, w_tiled_);
  } else {
    e = gemm_bf16(W, X, C, N, K, T, N, accumulate ? 2 : 0, 1, st_, nullptr, pn, w_tiled_);
  }
  // algorithmic bytes: weights + per row activations in + fp32 out (read-modify-write when accumulating)
  ktoc(&kr, 2.0 * N * K, 2.0 * K + (accumulate ? 8.0 : 4.0) * N, 2.0 * N * K, T);
  ++launches;
  return e;
}

// a13: greedy (parity mode, lowest index on ties) or top-p with Philox keyed by
// (sample_seed, sample id, token index); writes the next input token and the history
cudaError_t Engine::sample(const float* logits, int rows, const uint32_t* sid, const int32_t* slot,
                           const int32_t* tok_idx) {
  ++launches;
  if (e_.sampling == SGS_SAMPLE_TOP_P)
    return sample_top_p(logits, rows, m_.vocab, e_.temperature, e_.top_p, e_.sample_seed, sid, nullptr, slot, tok_idx,
                        last_tok_, hist_, max_gen_, st_);
  return argmax_rows(logits, rows, m_.vocab, nullptr, slot, tok_idx, last_tok_, hist_, max_gen_, st_);
}

// m = bf16(SiLU(x Wg^T) * (x Wu^T)): one GEMM with the SwiGLU epilogue when
// the gate/up GEMM needs no split-K (always at the model shapes: 2 f / 128 >=
// 148 tiles), else the fp32 GEMM + the silu_mul kernel.
cudaError_t Engine::gate_up(const void* W, int T, const PreNorm* pn) {
  const int d = m_.d_model, f = m_.d_ffn;
  // split-K (fp32 partials + a SwiGLU kernel) only when the unsplit GEMM has
  // fewer 128-row tiles than SMs; at >= 148 tiles (e.g. a TP = 2 shard of 7B)
  // the fused SwiGLU epilogue saves the extra kernel boundary
  const int tiles = (2 * f / 128) * ((T + 255) / 256);
  if (!(e_.flags & SGS_F_DETERMINISTIC) && tiles < 148 && gemm_auto_splits(2 * f, d, T) > 1) {
    cudaError_t e = gemm(W, x_, gu_, 2 * f, d, T, false, pn);
    if (e != cudaSuccess) return e;
    ++launches;
    return silu_mul(gu_, mm_, T, f, st_);
  }
  KRec kr;
  ktic(&kr, gemm_cls_);
  cudaError_t e = gemm_bf16(W, x_, reinterpret_cast<float*>(mm_), 2 * f, d, T, f, 3, 1, st_, nullptr, pn, w_tiled_);
  ktoc(&kr, 2.0 * 2 * f * d, 2.0 * d + 2.0 * f, 2.0 * 2 * f * d, T);
  ++launches;
  return e;
}

sgs_status Engine::run_iteration(const IterPlan& plan) {
  auto& S = sched.samples();
  const int n_adm = (int)plan.admitted.size();
  // decode rows: the running samples (ascending slot), then the group members
  // admitted without a prefill (their first token from position P-1)
  std::vector<int32_t> drows(plan.running);
  drows.insert(drows.end(), plan.admitted_decode.begin(), plan.admitted_decode.end());
  const int n_run = (int)drows.size();
  // the prompt tokens are needed only to stage this iteration's prefill; a
  // completed sample's id may be submitted again (R22)
  struct Release {
    std::vector<Sample>& S;
    const IterPlan& plan;
    std::unordered_set<uint64_t>& live;
    ~Release() {
      for (int32_t i : plan.admitted) std::vector<int32_t>().swap(S[i].prompt);
      for (int32_t i : plan.completed) live.erase(S[i].id);
    }
  } release{S, plan, live_ids_};
  if (null_) {
    for (int32_t i : plan.completed) {
      const Sample& s = S[i];
      Completion c{s.id, s.slot, s.admit_iter, s.finish_iter, version, std::vector<int32_t>(s.d, 0)};
      ready_.push_back(std::move(c));
    }
    return SGS_OK;
  }
  const int d = m_.d_model, hd = m_.head_dim, nq = m_.n_q_heads, nkv = m_.n_kv_heads, f = m_.d_ffn,
            V = m_.vocab;
  const int qkvN = (nq + 2 * nkv) * hd;
  (void)qkvN, (void)f, (void)d, (void)n_adm;
  // per-kernel CUDA events on 1 in kTimingStride iterations: events between
  // kernels serialise them (no PDL overlap), so the others run untouched
  {
    uint64_t z = (uint64_t)timing_iter_++ + 0x9E3779B97F4A7C15ull;  // splitmix64 of the counter
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    timing_now_ = (e_.flags & SGS_F_KERNEL_TIMING) && (z % kTimingStride == 0);
  }
  // staging buffers and events of this iteration (the other pair may still be in flight)
  cur_buf_ ^= 1;
  meta_host_ = meta_bufs_[cur_buf_], tok_host_ = tok_bufs_[cur_buf_];
  ev0_ = ev0s_[cur_buf_], ev1_ = ev1s_[cur_buf_];
  // ---------------- stage metadata (host, pinned) -> one H2D copy
  std::vector<int32_t> meta;
  meta.reserve(4096);
  auto put = [&](const int32_t* p, size_t n) {
    const size_t at = meta.size();
    meta.insert(meta.end(), p, p + n);
    return at;
  };
  // prefill chunks first (their metadata offsets then depend only on the
  // chunks, so a prefill graph can be replayed), block-table deltas after them
  struct Chunk {
    std::vector<int32_t> idx;
    int T = 0, nqb = 0, row_base = 0;
    size_t o_tok, o_pos, o_slot, o_offs, o_qb, o_last, o_pfslot, o_pftok;
  };
  std::vector<Chunk> chunks;
  {
    Chunk cur;
    for (int32_t i : plan.admitted) {
      if (S[i].group >= 0 && !S[i].group_first) continue;  // shared prefix: a decode row instead (R26)
      if (cur.T > 0 && cur.T + S[i].P > e_.max_prefill_tokens) {
        chunks.push_back(cur);
        cur = Chunk();
      }
      cur.idx.push_back(i);
      cur.T += S[i].P;
    }
    if (!cur.idx.empty()) chunks.push_back(cur);
  }
  int row_base = 0;
  for (auto& c : chunks) {
    std::vector<int32_t> tok, pos, slot, offs(1, 0), qb, last, pfs, pft, pfid;
    for (size_t k = 0; k < c.idx.size(); ++k) {
      const Sample& s = S[c.idx[k]];
      tok.insert(tok.end(), s.prompt.begin(), s.prompt.end());
      for (int j = 0; j < s.P; ++j) pos.push_back(j), slot.push_back(s.slot);
      offs.push_back(offs.back() + s.P);
      for (int b = 0; b < (s.P + qblk_ - 1) / qblk_; ++b) qb.push_back((int32_t)k), qb.push_back(b);
      last.push_back(offs.back() - 1);
      pfs.push_back(s.slot);
      pft.push_back(0);
      pfid.push_back((int32_t)(uint32_t)s.id), pfid.push_back((int32_t)(uint32_t)(s.id >> 32));
    }
    c.o_tok = put(tok.data(), tok.size());
    c.o_pos = put(pos.data(), pos.size());
    c.o_slot = put(slot.data(), slot.size());
    c.o_offs = put(offs.data(), offs.size());
    {
      // query blocks with more KV tiles first (causal: block b reads b + 1 tiles)
      std::vector<std::pair<int32_t, int32_t>> v;
      for (size_t x = 0; x + 1 < qb.size(); x += 2) v.push_back({qb[x + 1], qb[x]});
      std::stable_sort(v.begin(), v.end(), [](const std::pair<int32_t, int32_t>& a,
                                              const std::pair<int32_t, int32_t>& c) { return a.first > c.first; });
      for (size_t x = 0; x < v.size(); ++x) qb[2 * x] = v[x].second, qb[2 * x + 1] = v[x].first;
    }
    c.o_qb = put(qb.data(), qb.size());
    c.nqb = (int)qb.size() / 2;
    c.o_last = put(last.data(), last.size());
    c.o_pfslot = put(pfs.data(), pfs.size());
    c.o_pftok = put(pft.data(), pft.size());
    put(pfid.data(), pfid.size());  // sample ids (lo, hi), right after the token indices
    c.row_base = row_base;
    row_base += (int)c.idx.size();
  }
  std::vector<int32_t> deltas = plan.bt_deltas;
  for (int32_t i : plan.admitted_decode)  // the member's first decode row re-feeds the prompt's last token
    deltas.insert(deltas.end(), {S[i].slot, -1, S[i].prompt[S[i].P - 1]});
  const size_t o_bt = put(deltas.data(), deltas.size());
  const int n_bt = (int)deltas.size() / 3;
  const size_t o_cpa = put(plan.copies_after_prefill.data(), plan.copies_after_prefill.size());
  const size_t o_cpb = put(plan.copies_before_decode.data(), plan.copies_before_decode.size());
  // ---------------- decode rows (ascending slot) -> fixed region at the start of the metadata
  const int Bpad = (e_.max_batch + 15) / 16 * 16;
  const int Bk = (n_run + 15) / 16 * 16;  // CUDA-graph bucket; rows [n_run, Bk) are inert (slot -1)
  int32_t* D = reinterpret_cast<int32_t*>(meta_host_);
  int32_t *dslot = D + 4, *dpos = dslot + Bpad, *dctx = dpos + Bpad, *dtok = dctx + Bpad;
  uint32_t* dsid = reinterpret_cast<uint32_t*>(dtok + Bpad);  // sample id (lo, hi) per row, top-p key
  for (int r = 0; r < Bk; ++r) {
    if (r < n_run) {
      const Sample& s = S[drows[r]];
      const int j = s.produced - 1;  // tokens generated before this iteration (plan already counted this one)
      if (r >= (int)plan.running.size())  // shared-prefix member: position P-1 of its prompt, first token
        dslot[r] = s.slot, dpos[r] = s.P - 1, dctx[r] = s.P, dtok[r] = 0;
      else
        dslot[r] = s.slot, dpos[r] = s.P + j - 1, dctx[r] = s.P + j, dtok[r] = j;
      dsid[2 * r] = (uint32_t)s.id, dsid[2 * r + 1] = (uint32_t)(s.id >> 32);
    } else {
      dslot[r] = -1, dpos[r] = 0, dctx[r] = 1, dtok[r] = 0;
      dsid[2 * r] = 0, dsid[2 * r + 1] = 0;
    }
  }
  AttnPlan ap;
  attn_plan(dctx, dslot, n_run, nkv, e_.page_size, 0, &ap);
  if ((int)ap.items.size() > L_.max_items || ap.n_parts > L_.max_items) {
    err = "attention work list exceeds workspace";
    poisoned = true;
    return SGS_E_NOMEM;
  }
  D[0] = (int32_t)ap.items.size(), D[1] = (int32_t)ap.combs.size(), D[2] = n_run;
  // decode launch counter: PreNorm barrier parity (bit 0) and the TP exchange epochs
  D[3] = n_run > 0 ? (int32_t)(dec_launch_++ & 0x3fffffff) : 0;
  AttnComb* hcombs = reinterpret_cast<AttnComb*>(D + 4 + 6 * Bpad);
  AttnItem* hitems = reinterpret_cast<AttnItem*>(hcombs + L_.max_items);
  std::memcpy(hcombs, ap.combs.data(), ap.combs.size() * sizeof(AttnComb));
  std::memcpy(hitems, ap.items.data(), ap.items.size() * sizeof(AttnItem));
  const size_t dec_used = (uint8_t*)(hitems + ap.items.size()) - meta_host_;
  {
    double sum_ctx = 0;
    for (int r = 0; r < n_run; ++r) sum_ctx += dctx[r];
    // algorithmic bytes of one decode-attention launch: every cached K and V
    // element once + q in + o out; flops = 4 nq hd sum(ctx)
    cur_attn_bytes_ = sum_ctx * nkv * hd * 2 * 2 + (double)n_run * nq * hd * 2 * 2;
    cur_attn_flops_ = 4.0 * nq * hd * sum_ctx;
  }
  if ((int64_t)meta.size() * 4 > L_.meta_bytes - L_.meta_dec_bytes) {
    err = "iteration metadata exceeds the staging buffer";
    poisoned = true;
    return SGS_E_NOMEM;
  }
  std::memcpy(meta_host_ + L_.meta_dec_bytes, meta.data(), meta.size() * 4);
  const int32_t* MD = reinterpret_cast<const int32_t*>(meta_dev_ + L_.meta_dec_bytes);
  CK(cudaEventRecord(ev0_, st_), "event");
  if (n_run > 0) CK(cudaMemcpyAsync(meta_dev_, meta_host_, dec_used, cudaMemcpyHostToDevice, st_), "meta H2D");
  if (!meta.empty())
    CK(cudaMemcpyAsync(meta_dev_ + L_.meta_dec_bytes, meta_host_ + L_.meta_dec_bytes, meta.size() * 4,
                       cudaMemcpyHostToDevice, st_),
       "meta H2D");
  h2d_bytes += (int64_t)meta.size() * 4 + (n_run > 0 ? (int64_t)dec_used : 0);
  CK(apply_bt_deltas(bt_, L_.max_pages, MD + o_bt, n_bt, st_, last_tok_), "bt deltas");
  ++launches;
  const int64_t kv_layer_stride = n_pages_ * (L_.kv_page_bytes / m_.n_layers);
  auto copy_pages = [&](size_t o, size_t n_pairs) {
    ++launches;
    return copy_kv_pages(arena_ + L_.off_kv, kv_layer_stride, L_.kv_page_bytes / m_.n_layers, m_.n_layers, MD + o,
                         (int)n_pairs, st_);
  };

  // ---------------- prefill: on its own stream and scratch, concurrent with the decode graph
  // (disjoint rows, slots and pages); sequential in timed / graph-less iterations
  // (a group member decoding from a prefix prefilled in this same iteration
  // needs that prefill first: no concurrency then)
  const bool concurrent = !chunks.empty() && n_run > 0 && !(e_.flags & SGS_F_NO_GRAPHS) && !timing_now_ && tp_ == 1 &&
                          (plan.copies_after_prefill.empty() || plan.admitted_decode.empty());
  if (concurrent) {
    CK(cudaEventRecord(ev_meta_, st_), "event");
    CK(cudaStreamWaitEvent(st_pf_, ev_meta_, 0), "wait meta");
    std::swap(st_, st_pf_);
  }
  // SGS_F_SKIP_PREFILL (T(b) profiling only): the admitted prompts' prefill is
  // not computed; their pages keep stale KV and the first token is whatever
  // the token history holds -- decode iterations run unchanged
  if (e_.flags & SGS_F_SKIP_PREFILL) chunks.clear();
  for (auto& c : chunks) {
    {
      // causal self-attention of whole prompts: QK^T and PV over P(P+1)/2 pairs each
      double pairs = 0;
      for (int32_t i : c.idx) pairs += 0.5 * (double)S[i].P * (S[i].P + 1);
      cur_pf_attn_flops_ = 4.0 * nq * hd * pairs;
    }
    auto body = [&]() {
      return prefill_chunk(c.idx, c.row_base, MD + c.o_tok, MD + c.o_pos, MD + c.o_slot, MD + c.o_offs,
                           MD + c.o_qb, c.nqb, MD + c.o_last, MD + c.o_pfslot, MD + c.o_pftok, c.T);
    };
    if ((e_.flags & SGS_F_NO_GRAPHS) || timing_now_) {
      sgs_status s = body();
      if (s != SGS_OK) return s;
      continue;
    }
    std::vector<int64_t> key{c.row_base, (int64_t)c.o_tok, c.T, c.nqb};
    for (int32_t i : c.idx) key.push_back(S[i].P);
    if (pgraphs_.size() > 64 && !pgraphs_.count(key)) {  // bounded cache
      for (auto& kv : pgraphs_)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      pgraphs_.clear();
    }
    DecodeGraph& g = pgraphs_[key];
    if (!g.exec) {
      if (g.uses++ == 0) {  // first use eager
        sgs_status s = body();
        if (s != SGS_OK) return s;
        continue;
      }
      const int64_t l0 = launches;
      cudaGraph_t graph;
      CK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal), "begin capture");
      sgs_status s = body();
      cudaError_t ce = cudaStreamEndCapture(st_, &graph);
      if (s != SGS_OK) return s;
      CK(ce, "end capture");
      CK(cudaGraphInstantiate(&g.exec, graph, 0), "graph instantiate");
      cudaGraphDestroy(graph);
      g.kernels = launches - l0;
      launches = l0;
    }
    CK(cudaGraphLaunch(g.exec, st_), "graph launch");
    launches += g.kernels;
  }
  // a group's first member wrote the page holding position P-1 into its own
  // copy: the group's page gets it (the source of later members' copies)
  if (!plan.copies_after_prefill.empty()) CK(copy_pages(o_cpa, plan.copies_after_prefill.size() / 2), "kv copy");
  if (concurrent) {
    std::swap(st_, st_pf_);
    CK(cudaEventRecord(ev_pf_, st_pf_), "event");
  }
  if (!plan.copies_before_decode.empty()) CK(copy_pages(o_cpb, plan.copies_before_decode.size() / 2), "kv copy");
  // ---------------- decode (graph replay per bucket)
  if (n_run > 0) {
    sgs_status s = run_decode(n_run);
    if (s != SGS_OK) return s;
  }
  if (concurrent) CK(cudaStreamWaitEvent(st_, ev_pf_, 0), "join prefill");
  // ---------------- completions: D2H of their tokens
  int64_t off = 0;
  std::vector<int64_t> toff;
  for (int32_t i : plan.completed) {
    const Sample& s = S[i];
    if (off + s.d > tok_host_cap_) {
      err = "token staging overflow";
      poisoned = true;
      return SGS_E_NOMEM;
    }
    CK(cudaMemcpyAsync(tok_host_ + off, hist_ + (size_t)s.slot * max_gen_, (size_t)s.d * 4, cudaMemcpyDeviceToHost,
                       st_),
       "tokens D2H");
    toff.push_back(off);
    off += s.d;
    d2h_bytes += (int64_t)s.d * 4;
  }
  const int rows = row_base + n_run;
  if (e_.flags & SGS_F_KEEP_LOGITS) {
    kept_logits_.resize((size_t)rows * V);
    // prefill rows live after the Bpad decode rows of the logits buffer
    if (row_base)
      CK(cudaMemcpyAsync(kept_logits_.data(), logits_ + (size_t)Bpad * V, (size_t)row_base * V * 4,
                         cudaMemcpyDeviceToHost, st_),
         "logits D2H");
    if (n_run)
      CK(cudaMemcpyAsync(kept_logits_.data() + (size_t)row_base * V, logits_, (size_t)n_run * V * 4,
                         cudaMemcpyDeviceToHost, st_),
         "logits D2H");
    kept_ids_.clear();
    kept_tok_.clear();
    for (auto& c : chunks)
      for (int32_t i : c.idx) kept_ids_.push_back(S[i].id), kept_tok_.push_back(0);
    for (int32_t i : drows) kept_ids_.push_back(S[i].id), kept_tok_.push_back(S[i].produced - 1);
  }
  CK(cudaEventRecord(ev1_, st_), "event");
  Inflight fl;
  fl.buf = cur_buf_;
  fl.t = plan.t, fl.b = plan.b, fl.adm = n_adm, fl.sumctx = plan.sumctx, fl.n_run = n_run, fl.timing = timing_now_;
  for (auto& c : chunks) fl.pf_tok += c.T;
  for (int32_t i : plan.completed) {
    const Sample& s = S[i];
    fl.comps.push_back(Completion{s.id, s.slot, s.admit_iter, s.finish_iter, version, std::vector<int32_t>(s.d)});
  }
  fl.toff = std::move(toff);
  infl_.push_back(std::move(fl));
  // kernel-timing samples and logit capture need this iteration's results now
  if (timing_now_ || (e_.flags & SGS_F_KEEP_LOGITS)) return drain();
  return SGS_OK;
}

sgs_status Engine::finalize_front() {
  Inflight& f = infl_.front();
  CK(cudaEventSynchronize(ev1s_[f.buf]), "iteration sync");
  CK(cudaEventElapsedTime(&last_ms, ev0s_[f.buf], ev1s_[f.buf]), "elapsed");
  if (f.timing) {
    cur_phase_ = f.n_run >= 129 ? 1 : (f.n_run >= 1 && f.n_run <= 32 ? 2 : 0);
    CK(kflush(krec_, f.n_run), "kernel timing");
    krec_.clear();
    ev_used_ = 0;
    if (f.n_run > 0 && !(e_.flags & SGS_F_NO_GRAPHS)) {
      const DecodeGraph& g = graphs_[1][(f.n_run + 15) / 16];
      if (g.exec) CK(kflush(g.recs, f.n_run), "kernel timing");
    }
    kstat_ms[3] += last_ms;  // slot 3: device time of the sampled iterations (for the kernel shares)
    kstat_n[3] += 1;
    if (cur_phase_) kstat_ms[3 + kClasses * cur_phase_] += last_ms, kstat_n[3 + kClasses * cur_phase_] += 1;
  }
  iter_log.insert(iter_log.end(), {f.t, f.b, f.adm, f.pf_tok, f.sumctx, (int64_t)std::llround(last_ms * 1000.0)});
  const int32_t* tok = tok_bufs_[f.buf];
  for (size_t k = 0; k < f.comps.size(); ++k) {
    Completion& c = f.comps[k];
    std::copy(tok + f.toff[k], tok + f.toff[k] + c.tokens.size(), c.tokens.begin());
    ready_.push_back(std::move(c));
  }
  infl_.pop_front();
  return SGS_OK;
}

sgs_status Engine::drain() {
  while (!infl_.empty()) {
    sgs_status s = finalize_front();
    if (s != SGS_OK) return s;
  }
  return SGS_OK;
}

// The decode step for a bucket of Bk rows: every pointer is fixed (metadata
// region at meta_dev_, scratch buffers) and the attention work counts are
// read on the device, so the same launch sequence can be captured once per
// bucket and replayed.  Rows >= the real batch carry slot -1 and are inert.
sgs_status Engine::decode_body(int Bk) {
  const int d = m_.d_model, hd = m_.head_dim, nq = m_.n_q_heads, nkv = m_.n_kv_heads, f = m_.d_ffn,
            V = m_.vocab;
  const int qkvN = (nq + 2 * nkv) * hd;
  const int Bpad = (e_.max_batch + 15) / 16 * 16;
  const int32_t* MD = reinterpret_cast<const int32_t*>(meta_dev_);
  const int32_t* counts = MD;
  const int32_t* d_slot = MD + 4;
  const int32_t* d_pos = d_slot + Bpad;
  const int32_t* d_ctx = d_pos + Bpad;
  const int32_t* d_tok = d_ctx + Bpad;
  const uint32_t* d_sid = reinterpret_cast<const uint32_t*>(d_tok + Bpad);
  const AttnComb* d_combs = reinterpret_cast<const AttnComb*>(d_tok + 3 * Bpad);
  const AttnItem* d_items = reinterpret_cast<const AttnItem*>(d_combs + L_.max_items);
  float* part_o = reinterpret_cast<float*>(attn_ws_);
  float* part_ml = part_o + (size_t)L_.max_items * (nq / nkv) * hd;
  int* arrive = reinterpret_cast<int*>(part_ml + (size_t)L_.max_items * (nq / nkv) * 2);  // zeroed at init
  const int cap_items = std::min(L_.max_items, 2 * 148 + Bk * nkv + 64);
  const int cap_combs = Bk * nkv;
  // SGS_DEBUG_SKIP (timing ablation only; results are garbage): bit k skips
  // kernel class k of the decode program
  auto on = [&](int bit) { return !(skip_ & (1 << bit)); };
  // class-5 timing of the small kernels: algorithmic bytes per row
  auto other = [&](cudaError_t e, KRec* kr, double brow) {
    ktoc(kr, 0.0, brow, 0.0, Bk);
    return e;
  };
  gemm_cls_ = 1;
  KRec ko;
  ktic(&ko, 5);
  if (on(9)) CK(other(embed(embed_, nullptr, d_slot, last_tok_, h_, Bk, d, st_), &ko, 6.0 * d), "embed");
  ++launches;
  // RMSNorm fused into the QKV / gate-up / LM-head GEMMs (PreNorm: rows
  // normalised by the GEMM's own CTAs before a grid barrier); the barrier
  // parity is this decode launch's, read from the metadata (D[3])
  const bool fuse = fused_norm_ && on(0) && tp_ == 1;
  // TP over peer memory: each RMSNorm after the first is fused into the
  // exchange that produces its input (tp_comm.cu), and only shard 0 keeps
  // the residual (the exchange leaves h = 0 on the others)
  const bool p2p = tp_p2p_;
  const int nx = 2 * m_.n_layers + 1;  // exchanges per decode launch (epoch numbering)
  auto pnorm = [&](const void* w, int site) { return PreNorm{h_, w, nullptr, m_.rms_eps, norm_bar_, site, counts + 3}; };
  for (int l = 0; l < m_.n_layers; ++l) {
    const Layer& Ly = layers_[l];
    const PreNorm pn1 = pnorm(Ly.n1, 2 * l), pn2 = pnorm(Ly.n2, 2 * l + 1);
    if (!fuse) ktic(&ko, 5);
    if (on(0) && !fuse && !(p2p && l > 0))
      CK(other(rmsnorm(h_, Ly.n1, x_, nullptr, Bk, d, m_.rms_eps, st_), &ko, 6.0 * d), "rmsnorm1");
    if (on(1)) CK(gemm(Ly.wqkv, x_, qkv_, qkvN, d, Bk, false, fuse ? &pn1 : nullptr), "gemm qkv");
    ktic(&ko, 5);
    if (on(2))
      CK(other(rope_append(qkv_, Ly.bqkv, d_pos, d_slot, bt_, L_.max_pages, rope_, q_, Ly.kv, nullptr, nullptr, Bk,
                           nq, nkv, hd, e_.page_size, st_),
               &ko, 6.0 * qkvN),
         "rope_append");
    KRec kr;
    ktic(&kr, 0);
    if (on(3))
      CK(attn_decode(q_, Ly.kv, bt_, counts, d_items, cap_items, d_combs, cap_combs, nq, nkv, hd, e_.page_size,
                     L_.max_pages, ao_, 0, part_o, part_ml, arrive, st_),
         "attn_decode");
    ktoc(&kr, -1.0, 0.0, 0.0, 0);
    // TP: every shard adds its partial O projection; shard 0 keeps h, the others
    // start from 0, and the all-reduce (sum) leaves h + sum of partials on all
    if (tp_ > 1 && tp_rank_ != 0 && (!p2p || l == 0)) CK(cudaMemsetAsync(h_, 0, (size_t)Bk * d * 4, st_), "tp zero h");
    if (on(4)) CK(gemm(Ly.wo, ao_, h_, d, nq * hd, Bk, true), "gemm o");
    if (p2p) {  // exchange of the O partials + RMSNorm 2 in one kernel
      ktic(&ko, 5);
      CK(other(tp_allreduce_rmsnorm(h_, Ly.n2, x_, Bk, d, m_.rms_eps, tpp_, xch_rows_, counts + 3, 2 * l, nx, st_), &ko,
               (6.0 + 8.0 * (tp_ - 1)) * d),
         "tp exchange o + rmsnorm2");
    } else {
      if (tp_ > 1) CK(tp_allreduce_sum(h_, (size_t)Bk * d), "tp allreduce o");
      if (!fuse) ktic(&ko, 5);
      if (on(0) && !fuse) CK(other(rmsnorm(h_, Ly.n2, x_, nullptr, Bk, d, m_.rms_eps, st_), &ko, 6.0 * d), "rmsnorm2");
    }
    if (on(5)) CK(gate_up(Ly.wgu, Bk, fuse ? &pn2 : nullptr), "gemm gate_up + SwiGLU");
    if (tp_ > 1 && tp_rank_ != 0 && !p2p) CK(cudaMemsetAsync(h_, 0, (size_t)Bk * d * 4, st_), "tp zero h");
    if (on(6)) CK(gemm(Ly.wd, mm_, h_, d, f, Bk, true), "gemm down");
    if (p2p) {  // exchange of the down partials + the next layer's RMSNorm 1 (or the final norm)
      ktic(&ko, 5);
      CK(other(tp_allreduce_rmsnorm(h_, l + 1 < m_.n_layers ? layers_[l + 1].n1 : nf_, x_, Bk, d, m_.rms_eps, tpp_,
                                    xch_rows_, counts + 3, 2 * l + 1, nx, st_),
               &ko, (6.0 + 8.0 * (tp_ - 1)) * d),
         "tp exchange down + rmsnorm");
    } else if (tp_ > 1) {
      CK(tp_allreduce_sum(h_, (size_t)Bk * d), "tp allreduce down");
    }
    launches += fuse ? 2 : p2p ? (l == 0 ? 5 : 4) : 4;  // (rmsnorm x2 | exchanges,) RoPE, attention
  }
  const PreNorm pnf = pnorm(nf_, 2 * m_.n_layers);
  if (!fuse) ktic(&ko, 5);
  if (on(0) && !fuse && !p2p) CK(other(rmsnorm(h_, nf_, x_, nullptr, Bk, d, m_.rms_eps, st_), &ko, 6.0 * d), "rmsnorm f");
  if (e_.sampling == SGS_SAMPLE_GREEDY) {
    // LM head with greedy sampling fused into its epilogue (GEMM mode 4): no
    // fp32 logits round trip and no sampler launch; the logits are still
    // written for SGS_F_KEEP_LOGITS (same values, so the tests see the argmax
    // of exactly what was sampled)
    const bool keep = (e_.flags & SGS_F_KEEP_LOGITS) != 0;
    const int Bpad = (e_.max_batch + 15) / 16 * 16;
    ArgmaxArgs am{amax_keys_, reinterpret_cast<unsigned int*>(amax_keys_ + Bpad), d_slot, d_tok, last_tok_, hist_,
                  max_gen_, tp_rank_ * V, tp_ == 1};
    KRec kr;
    ktic(&kr, gemm_cls_);
    if (on(7))
      CK(gemm_bf16(lm_head_, x_, keep ? logits_ : nullptr, V, d, Bk, V, 4, 1, st_, &am, fuse ? &pnf : nullptr,
                   w_tiled_),
         "gemm lm_head");
    ktoc(&kr, 2.0 * V * d, 2.0 * d + (keep ? 4.0 * V : 0.0), 2.0 * V * d, Bk);
    launches += 1;
    if (p2p) {  // the shards' (max logit, lowest index) keys: exchange, max, tokens
      CK(tp_argmax_exchange(amax_keys_, Bk, d_slot, d_tok, last_tok_, hist_, max_gen_, tpp_, xch_rows_, d, counts + 3,
                            2 * m_.n_layers, nx, st_),
         "tp argmax exchange");
      ++launches;
    } else if (tp_ > 1) {  // the same over NCCL: all-reduce max, then the tokens
      CK(tp_allreduce_max_u64(amax_keys_, (size_t)Bk), "tp allreduce argmax");
      CK(argmax_keys_finalize(amax_keys_, Bk, d_slot, d_tok, last_tok_, hist_, max_gen_, st_), "argmax finalize");
      ++launches;
    }
  } else {
    if (on(7)) CK(gemm(lm_head_, x_, logits_, V, d, Bk, false, fuse ? &pnf : nullptr), "gemm lm_head");
    ktic(&ko, 5);
    if (on(8)) CK(other(sample(logits_, Bk, d_sid, d_slot, d_tok), &ko, 4.0 * V), "sampler");
  }
  if (!p2p) launches += 1;  // final rmsnorm (GEMM and sampler count themselves)
  return SGS_OK;
}

void Engine::swap_scratch() {
  std::swap(h_, dset_.h);
  std::swap(qkv_, dset_.qkv);
  std::swap(gu_, dset_.gu);
  std::swap(x_, dset_.x);
  std::swap(q_, dset_.q);
  std::swap(ao_, dset_.ao);
  std::swap(mm_, dset_.mm);
}

sgs_status Engine::run_decode(int b) {
  // the decode program always runs on the decode scratch set (graphs capture its pointers)
  swap_scratch();
  const sgs_status s = run_decode_body(b);
  swap_scratch();
  return s;
}

sgs_status Engine::run_decode_body(int b) {
  const int Bk = (b + 15) / 16 * 16;
  if (e_.flags & SGS_F_NO_GRAPHS) return decode_body(Bk);
  auto& gs = graphs_[timing_now_ ? 1 : 0];
  if (gs.empty()) gs.resize((e_.max_batch + 15) / 16 + 1);
  DecodeGraph& g = gs[Bk / 16];
  if (!g.exec) {
    if (g.uses++ == 0) return decode_body(Bk);  // first use eager: sets kernel attributes, warms caches
    const int64_t l0 = launches;
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal), "begin capture");
    rec_target_ = &g.recs;
    sgs_status s = decode_body(Bk);
    rec_target_ = nullptr;
    cudaError_t ce = cudaStreamEndCapture(st_, &graph);
    if (s != SGS_OK) return s;
    CK(ce, "end capture");
    CK(cudaGraphInstantiate(&g.exec, graph, 0), "graph instantiate");
    cudaGraphDestroy(graph);
    g.kernels = launches - l0;
    launches = l0;
  }
  CK(cudaGraphLaunch(g.exec, st_), "graph launch");
  launches += g.kernels;
  return SGS_OK;
}

sgs_status Engine::prefill_chunk(const std::vector<int32_t>& idx, int row_base, const int32_t* d_tokens,
                                 const int32_t* d_pos, const int32_t* d_slot, const int32_t* d_offs,
                                 const int32_t* d_qblocks, int n_qblocks, const int32_t* d_last_rows,
                                 const int32_t* d_pf_slot, const int32_t* d_pf_tok, int T, float* dump,
                                 int only_layer, const float* h_in) {
  const int d = m_.d_model, hd = m_.head_dim, nq = m_.n_q_heads, nkv = m_.n_kv_heads, f = m_.d_ffn,
            V = m_.vocab;
  const int qkvN = (nq + 2 * nkv) * hd;
  const int np = (int)idx.size();
  gemm_cls_ = 4;
  struct Restore {
    int& c;
    ~Restore() { c = 1; }
  } restore_cls{gemm_cls_};
  int n_dump = 0;
  auto save = [&]() -> cudaError_t {
    if (!dump || only_layer >= 0) return cudaSuccess;  // layer-local mode returns only the final h
    return cudaMemcpyAsync(dump + (size_t)(n_dump++) * T * d, h_, (size_t)T * d * 4, cudaMemcpyDeviceToHost, st_);
  };
  if (h_in) {  // layer-local parity: start from a given residual stream
    CK(cudaMemcpyAsync(h_, h_in, (size_t)T * d * 4, cudaMemcpyHostToDevice, st_), "h_in");
  } else {
    CK(embed(embed_, d_tokens, nullptr, nullptr, h_, T, d, st_), "embed");
    ++launches;
    CK(save(), "dump");
  }
  const int l_begin = only_layer >= 0 ? only_layer : 0;
  const int l_end = only_layer >= 0 ? only_layer + 1 : m_.n_layers;
  for (int l = l_begin; l < l_end; ++l) {
    const Layer& Ly = layers_[l];
    CK(rmsnorm(h_, Ly.n1, x_, nullptr, T, d, m_.rms_eps, st_), "rmsnorm1");
    CK(gemm(Ly.wqkv, x_, qkv_, qkvN, d, T, false), "gemm qkv");
    CK(rope_append(qkv_, Ly.bqkv, d_pos, d_slot, bt_, L_.max_pages, rope_, q_, Ly.kv, kc_, vc_, T, nq, nkv, hd,
                   e_.page_size, st_, qblk_ == 128),
       "rope_append");
    KRec kr;
    ktic(&kr, 2);
    if (qblk_ == 128)  // tcgen05/TMEM flash attention (hd 128)
      CK(attn_prefill_tc(q_, kc_, vc_, d_offs, d_qblocks, n_qblocks, L_.tmax, nq, nkv, ao_, st_), "attn_prefill_tc");
    else
      CK(attn_prefill(q_, kc_, vc_, d_offs, d_qblocks, n_qblocks, nq, nkv, hd, ao_, st_), "attn_prefill");
    // algorithmic bytes: q, k, v in and o out once per row (bf16); flops from the chunk's prompts
    ktoc(&kr, 0.0, 2.0 * hd * (2.0 * nq + 2.0 * nkv), cur_pf_attn_flops_ / std::max(T, 1), T);
    if (tp_ > 1 && tp_rank_ != 0) CK(cudaMemsetAsync(h_, 0, (size_t)T * d * 4, st_), "tp zero h");
    CK(gemm(Ly.wo, ao_, h_, d, nq * hd, T, true), "gemm o");
    if (tp_ > 1) CK(tp_allreduce_sum(h_, (size_t)T * d), "tp allreduce o");
    CK(save(), "dump");
    CK(rmsnorm(h_, Ly.n2, x_, nullptr, T, d, m_.rms_eps, st_), "rmsnorm2");
    CK(gate_up(Ly.wgu, T), "gemm gate_up + SwiGLU");
    if (tp_ > 1 && tp_rank_ != 0) CK(cudaMemsetAsync(h_, 0, (size_t)T * d * 4, st_), "tp zero h");
    CK(gemm(Ly.wd, mm_, h_, d, f, T, true), "gemm down");
    if (tp_ > 1) CK(tp_allreduce_sum(h_, (size_t)T * d), "tp allreduce down");
    CK(save(), "dump");
    launches += 4;  // rmsnorm x2, RoPE, attention; the GEMMs count themselves
  }
  if (only_layer >= 0) {
    if (dump) CK(cudaMemcpyAsync(dump, h_, (size_t)T * d * 4, cudaMemcpyDeviceToHost, st_), "h_out");
    return SGS_OK;
  }
  CK(rmsnorm(h_, nf_, x_, d_last_rows, np, d, m_.rms_eps, st_), "rmsnorm f");
  float* lg = logits_ + (size_t)((e_.max_batch + 15) / 16 * 16 + row_base) * V;
  if (tp_ > 1) {
    // the shards' LM-head halves: fused argmax keys, all-reduce max, tokens
    const bool keep = (e_.flags & SGS_F_KEEP_LOGITS) != 0;
    ArgmaxArgs am{amax_keys_pf_, nullptr, d_pf_slot, d_pf_tok, last_tok_, hist_, max_gen_, tp_rank_ * V, 0};
    CK(gemm_bf16(lm_head_, x_, keep ? lg : nullptr, V, d, np, V, 4, 1, st_, &am, nullptr, w_tiled_), "gemm lm_head");
    CK(tp_allreduce_max_u64(amax_keys_pf_, (size_t)np), "tp allreduce argmax");
    CK(argmax_keys_finalize(amax_keys_pf_, np, d_pf_slot, d_pf_tok, last_tok_, hist_, max_gen_, st_),
       "argmax finalize");
    launches += 3;
  } else {
    CK(gemm(lm_head_, x_, lg, V, d, np, false), "gemm lm_head");
    CK(sample(lg, np, reinterpret_cast<const uint32_t*>(d_pf_tok + np), d_pf_slot, d_pf_tok), "sampler");
  }
  launches += 1;  // final rmsnorm (GEMM and sampler count themselves)
  return SGS_OK;
}

// Standalone prefill forward of one prompt in slot 0 (idle handle only) with
// the residual stream dumped after the embedding and every residual add.
sgs_status Engine::debug_forward(const int32_t* tokens, int32_t T, float* dump, int layer, const float* h_in) {
  if (tp_ > 1) {
    err = "debug hooks are not available on tensor-parallel shards";
    return SGS_E_UNSUPPORTED;
  }
  if (layer == m_.n_layers && h_in && dump && !null_ && T > 0) return debug_head(h_in, T, dump);
  if (layer >= m_.n_layers || (layer >= 0 && !h_in) || (layer < 0 && !tokens)) {
    err = "debug_forward: bad layer / input";
    return SGS_E_INVAL;
  }
  std::vector<int32_t> zeros;
  if (!tokens) zeros.assign(T > 0 ? T : 0, 0), tokens = zeros.data();
  if (null_ || !sched.idle()) {
    err = "debug_forward needs a device handle with nothing in flight";
    return SGS_E_STATE;
  }
  {
    sgs_status ds = drain();
    if (ds != SGS_OK) return ds;
  }
  const int np = (T + e_.page_size - 1) / e_.page_size;
  if (T < 1 || T > e_.max_prefill_tokens || np > n_pages_ || np > L_.max_pages) {
    err = "debug_forward: prompt too long";
    return SGS_E_INVAL;
  }
  std::vector<int32_t> meta;
  for (int k = 0; k < np; ++k) meta.insert(meta.end(), {0, k, k});
  const size_t o_tok = meta.size();
  meta.insert(meta.end(), tokens, tokens + T);
  const size_t o_pos = meta.size();
  for (int j = 0; j < T; ++j) meta.push_back(j);
  const size_t o_slot = meta.size();
  for (int j = 0; j < T; ++j) meta.push_back(0);
  const size_t o_offs = meta.size();
  meta.push_back(0), meta.push_back(T);
  const size_t o_qb = meta.size();
  for (int b = 0; b < (T + qblk_ - 1) / qblk_; ++b) meta.push_back(0), meta.push_back(b);
  const size_t o_last = meta.size();
  meta.push_back(T - 1), meta.push_back(0), meta.push_back(0);  // last row, pf slot, pf tok
  meta.push_back(0), meta.push_back(0);                         // sample id (lo, hi)
  std::memcpy(meta_host_, meta.data(), meta.size() * 4);
  const int32_t* MD = reinterpret_cast<const int32_t*>(meta_dev_);
  CK(cudaMemcpyAsync(meta_dev_, meta_host_, meta.size() * 4, cudaMemcpyHostToDevice, st_), "meta");
  CK(apply_bt_deltas(bt_, L_.max_pages, MD, np, st_), "bt");
  std::vector<int32_t> idx(1, 0);
  cur_pf_attn_flops_ = 2.0 * m_.n_q_heads * m_.head_dim * (double)T * (T + 1);
  sgs_status s = prefill_chunk(idx, 0, MD + o_tok, MD + o_pos, MD + o_slot, MD + o_offs, MD + o_qb, (T + qblk_ - 1) / qblk_,
                               MD + o_last, MD + o_last + 1, MD + o_last + 2, T, dump, layer, h_in);
  if (s != SGS_OK) return s;
  CK(cudaStreamSynchronize(st_), "debug sync");
  return SGS_OK;
}

// Final RMSNorm + LM head of the CUDA path on a given fp32 residual stream
// (host [T x d]) -> fp32 logits (host [T x V]), in chunks of the logits buffer.
sgs_status Engine::debug_head(const float* h_in, int32_t T, float* logits) {
  if (!sched.idle()) {
    err = "debug_head needs an idle handle";
    return SGS_E_STATE;
  }
  {
    sgs_status ds = drain();
    if (ds != SGS_OK) return ds;
  }
  const int d = m_.d_model, V = m_.vocab;
  const int R = std::min(L_.tmax, (e_.max_batch + 15) / 16 * 16 + e_.max_batch);
  for (int r0 = 0; r0 < T; r0 += R) {
    const int n = std::min(R, T - r0);
    CK(cudaMemcpyAsync(h_, h_in + (size_t)r0 * d, (size_t)n * d * 4, cudaMemcpyHostToDevice, st_), "h_in");
    CK(rmsnorm(h_, nf_, x_, nullptr, n, d, m_.rms_eps, st_), "rmsnorm f");
    CK(gemm(lm_head_, x_, logits_, V, d, n, false), "gemm lm_head");
    CK(cudaMemcpyAsync(logits + (size_t)r0 * V, logits_, (size_t)n * V * 4, cudaMemcpyDeviceToHost, st_), "logits");
    CK(cudaStreamSynchronize(st_), "debug head sync");
  }
  return SGS_OK;
}

sgs_status Engine::last_logits(float* logits, uint64_t* ids, int32_t* tok_idx, int32_t cap, int32_t* rows) {
  const int n = (int)kept_ids_.size();
  *rows = n;
  if (!logits) return SGS_OK;
  const int k = std::min(n, cap);
  std::memcpy(logits, kept_logits_.data(), (size_t)k * m_.vocab * 4);
  for (int i = 0; i < k; ++i) ids[i] = kept_ids_[i], tok_idx[i] = kept_tok_[i];
  return SGS_OK;
}

// ------------------------------------------------------------------ NCCL (dlopen: the process's libnccl.so.2)
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
};

static NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.ok ? &api : nullptr;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
  api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
  api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
  api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  api.ok = api.GetUniqueId && api.CommInitRank && api.Broadcast && api.AllReduce && api.GroupStart && api.GroupEnd;
  return api.ok ? &api : nullptr;
}

sgs_status Engine::comm_init(const uint8_t id[128], int rank, int world) {
  if (null_) {
    err = "no device";
    return SGS_E_STATE;
  }
  NcclApi* api = nccl();
  if (!api) {
    err = "libnccl.so.2 not found";
    return SGS_E_NCCL;
  }
  ncclUniqueId uid;
  static_assert(sizeof(ncclUniqueId) == 128, "nccl unique id size");
  std::memcpy(&uid, id, 128);
  ncclComm_t comm;
  ncclResult_t r = api->CommInitRank(&comm, world, uid, rank);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + api->GetErrorString(r);
    return SGS_E_NCCL;
  }
  nccl_comm_ = comm;
  nccl_rank_ = rank;
  nccl_world_ = world;
  return SGS_OK;
}

// NEXT-2: the tensor-parallel communicator (shard tp_rank_ of tp_)
sgs_status Engine::tp_comm_init(const uint8_t id[128]) {
  if (tp_ <= 1) {
    err = "not a tensor-parallel handle (tp_size <= 1)";
    return SGS_E_STATE;
  }
  NcclApi* api = nccl();
  if (!api) {
    err = "libnccl.so.2 not found";
    return SGS_E_NCCL;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  ncclComm_t comm;
  ncclResult_t r = api->CommInitRank(&comm, tp_, uid, tp_rank_);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRank (tp): ") + api->GetErrorString(r);
    return SGS_E_NCCL;
  }
  tp_comm_ = comm;
  return tp_p2p_init();
}

// Decode-program exchange over NVLink peer memory (tp_comm.cu): every shard
// allocates its exchange buffer, the CUDA IPC handles are gathered over the
// new communicator (an 8-bit sum of zero-padded handles) and the peers'
// buffers opened in this process.  SGS_TP_NCCL_AR=1 keeps NCCL all-reduces.
sgs_status Engine::tp_p2p_init() {
  const char* env = std::getenv("SGS_TP_NCCL_AR");
  if ((env && env[0] == '1') || tp_ > TPX_MAX) return SGS_OK;
  xch_rows_ = (e_.max_batch + 15) / 16 * 16;
  const size_t bytes = tp_xch_bytes(tp_, xch_rows_, m_.d_model);
  cudaError_t e = cudaMalloc(&xch_, bytes);
  if (e == cudaSuccess) e = cudaMemset(xch_, 0, bytes);
  cudaIpcMemHandle_t mine;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&mine, xch_);
  uint8_t* gath = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&gath, (size_t)tp_ * sizeof(mine));
  if (e == cudaSuccess) e = cudaMemset(gath, 0, (size_t)tp_ * sizeof(mine));
  if (e == cudaSuccess) e = cudaMemcpy(gath + (size_t)tp_rank_ * sizeof(mine), &mine, sizeof(mine), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    err = std::string("tp exchange buffer: ") + cudaGetErrorString(e);
    if (gath) cudaFree(gath);
    return SGS_E_CUDA;
  }
  std::vector<cudaIpcMemHandle_t> all(tp_);
  const bool ok = nccl()->AllReduce(gath, gath, (size_t)tp_ * sizeof(mine), ncclUint8, ncclSum, (ncclComm_t)tp_comm_,
                                    st_) == ncclSuccess;
  e = ok ? cudaStreamSynchronize(st_) : cudaErrorUnknown;
  if (e == cudaSuccess) e = cudaMemcpy(all.data(), gath, (size_t)tp_ * sizeof(mine), cudaMemcpyDeviceToHost);
  cudaFree(gath);
  if (e != cudaSuccess) {
    err = "tp exchange: gathering the IPC handles failed";
    return SGS_E_NCCL;
  }
  tpp_.me = tp_rank_;
  tpp_.tp = tp_;
  for (int s = 0; s < tp_; ++s) {
    if (s == tp_rank_) {
      tpp_.base[s] = xch_;
      continue;
    }
    void* p = nullptr;
    e = cudaIpcOpenMemHandle(&p, all[s], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      err = std::string("tp exchange: cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
      return SGS_E_CUDA;
    }
    tpp_.base[s] = static_cast<uint8_t*>(p);
    xch_peer_.push_back(p);
  }
  // every shard has opened its peers' buffers before any exchange is launched
  uint8_t* one = nullptr;
  e = cudaMalloc(&one, 4);
  if (e == cudaSuccess) e = cudaMemset(one, 0, 4);
  const bool ok2 = e == cudaSuccess && nccl()->AllReduce(one, one, 1, ncclUint8, ncclSum, (ncclComm_t)tp_comm_, st_) ==
                                           ncclSuccess;
  e = ok2 ? cudaStreamSynchronize(st_) : cudaErrorUnknown;
  if (one) cudaFree(one);
  if (e != cudaSuccess) {
    err = "tp exchange: barrier failed";
    return SGS_E_NCCL;
  }
  tp_p2p_ = true;
  return SGS_OK;
}

cudaError_t Engine::tp_allreduce_sum(float* x, size_t n) {
  ++launches;
  return nccl()->AllReduce(x, x, n, ncclFloat32, ncclSum, (ncclComm_t)tp_comm_, st_) == ncclSuccess
             ? cudaSuccess
             : cudaErrorUnknown;
}

cudaError_t Engine::tp_allreduce_max_u64(unsigned long long* x, size_t n) {
  ++launches;
  return nccl()->AllReduce(x, x, n, ncclUint64, ncclMax, (ncclComm_t)tp_comm_, st_) == ncclSuccess
             ? cudaSuccess
             : cudaErrorUnknown;
}

sgs_status Engine::update_weights(const sgs_weights* src, int root) {
  if (tp_ > 1 && (src || nccl_world_ > 1)) {
    err = "weight sync is not available on tensor-parallel shards";
    return SGS_E_UNSUPPORTED;
  }
  if (poisoned) {
    err = "handle poisoned";
    return SGS_E_STATE;
  }
  if (sched.idle()) {
    sgs_status ds = drain();  // the last launched iteration finishes on the old weights
    if (ds != SGS_OK) return ds;
  }
  if (!sched.idle()) {
    err = "weight update with samples in flight";
    return SGS_E_STATE;
  }
  if (sync_pending_) {
    err = "an asynchronous weight update is in flight";
    return SGS_E_STATE;
  }
  const int me = nccl_world_ > 1 ? nccl_rank_ : 0;
  if (src && me != root) {
    err = "only the root passes the new weights";
    return SGS_E_INVAL;
  }
  if (null_) {
    ++version;
    return SGS_OK;
  }
  if (src) {
    sgs_status ls = load_weights(src, arena_, st_);
    if (ls != SGS_OK) return ls;
  }
  if (nccl_world_ > 1) {
    if (!nccl_comm_) {
      err = "sgs_comm_init not called";
      return SGS_E_STATE;
    }
    NcclApi* api = nccl();
    // the weights are one contiguous range at the arena start; broadcast in 256 MiB chunks
    const size_t total = (size_t)L_.weights_bytes;
    const size_t chunk = 256ull << 20;
    api->GroupStart();
    for (size_t o = 0; o < total; o += chunk) {
      const size_t n = std::min(chunk, total - o);
      ncclResult_t r = api->Broadcast(arena_ + o, arena_ + o, n, ncclUint8, root, (ncclComm_t)nccl_comm_, st_);
      if (r != ncclSuccess) {
        api->GroupEnd();
        err = std::string("ncclBroadcast: ") + api->GetErrorString(r);
        poisoned = true;
        return SGS_E_NCCL;
      }
    }
    ncclResult_t r = api->GroupEnd();
    if (r != ncclSuccess) {
      err = std::string("ncclGroupEnd: ") + api->GetErrorString(r);
      poisoned = true;
      return SGS_E_NCCL;
    }
    CK(cudaStreamSynchronize(st_), "broadcast sync");
  }
  ++version;
  return SGS_OK;
}

// ------------------------------------------------------------------ asynchronous weight sync (NEXT-1)
sgs_status Engine::shadow_weights(void** ptr, int64_t* bytes) {
  if (!null_ && !shadow_) {
    err = "engine created without SGS_F_SHADOW_WEIGHTS";
    return SGS_E_STATE;
  }
  *ptr = shadow_;
  *bytes = L_.weights_bytes;
  return SGS_OK;
}

sgs_status Engine::stage_weights_seed(uint64_t seed) {
  if (null_) return SGS_OK;
  if (!shadow_) {
    err = "engine created without SGS_F_SHADOW_WEIGHTS";
    return SGS_E_STATE;
  }
  if (sync_pending_) {
    err = "a weight update is in flight";
    return SGS_E_STATE;
  }
  // the previous commit may still be copying shadow -> active on st_
  CK(cudaStreamWaitEvent(st_side_, ev_commit_, 0), "wait commit");
  // the same tensors at the same offsets of the shadow buffer, on the side stream
  for (const auto& t : tensors_) {
    void* dst = shadow_ + (reinterpret_cast<uint8_t*>(t.ptr) - arena_);
    CK(hash_init(dst, seed, (uint64_t)t.id, t.n, t.is_norm, st_side_, t.cols, t.blk, t.stride, t.off, t.shard, t.tiled),
       "hash_init(shadow)");
  }
  return SGS_OK;
}

sgs_status Engine::stage_weights(const sgs_weights* src) {
  if (null_) return SGS_OK;
  if (!shadow_) {
    err = "engine created without SGS_F_SHADOW_WEIGHTS";
    return SGS_E_STATE;
  }
  if (sync_pending_) {
    err = "a weight update is in flight";
    return SGS_E_STATE;
  }
  CK(cudaStreamWaitEvent(st_side_, ev_commit_, 0), "wait commit");
  return load_weights(src, shadow_, st_side_);
}

sgs_status Engine::update_weights_begin(int root) {
  if (poisoned) {
    err = "handle poisoned";
    return SGS_E_STATE;
  }
  if (sync_pending_) {
    err = "a weight update is already in flight";
    return SGS_E_STATE;
  }
  if (null_) {
    sync_pending_ = true;
    return SGS_OK;
  }
  if (!shadow_) {
    err = "engine created without SGS_F_SHADOW_WEIGHTS";
    return SGS_E_STATE;
  }
  // the previous commit may still be copying shadow -> active on st_
  CK(cudaStreamWaitEvent(st_side_, ev_commit_, 0), "wait commit");
  if (nccl_world_ > 1) {
    if (!nccl_comm_) {
      err = "sgs_comm_init not called";
      return SGS_E_STATE;
    }
    NcclApi* api = nccl();
    const size_t total = (size_t)L_.weights_bytes;
    const size_t chunk = 256ull << 20;
    api->GroupStart();
    for (size_t o = 0; o < total; o += chunk) {
      const size_t n = std::min(chunk, total - o);
      ncclResult_t r = api->Broadcast(shadow_ + o, shadow_ + o, n, ncclUint8, root, (ncclComm_t)nccl_comm_, st_side_);
      if (r != ncclSuccess) {
        api->GroupEnd();
        err = std::string("ncclBroadcast: ") + api->GetErrorString(r);
        poisoned = true;
        return SGS_E_NCCL;
      }
    }
    ncclResult_t r = api->GroupEnd();
    if (r != ncclSuccess) {
      err = std::string("ncclGroupEnd: ") + api->GetErrorString(r);
      poisoned = true;
      return SGS_E_NCCL;
    }
  }
  CK(cudaEventRecord(ev_sync_, st_side_), "record sync");
  sync_pending_ = true;
  return SGS_OK;
}

sgs_status Engine::update_weights_ready(int32_t* ready) {
  if (!sync_pending_) {
    err = "no weight update in flight";
    return SGS_E_STATE;
  }
  if (null_) {
    *ready = 1;
    return SGS_OK;
  }
  const cudaError_t q = cudaEventQuery(ev_sync_);
  if (q != cudaSuccess && q != cudaErrorNotReady) return cuda_fail(q, "query sync");
  *ready = q == cudaSuccess ? 1 : 0;
  return SGS_OK;
}

sgs_status Engine::update_weights_commit() {
  if (!sync_pending_) {
    err = "no weight update in flight";
    return SGS_E_STATE;
  }
  if (sched.idle()) {
    sgs_status ds = drain();
    if (ds != SGS_OK) return ds;
  }
  if (!sched.idle()) {
    err = "weight commit with samples in flight (the swap happens at an RL-batch boundary)";
    return SGS_E_STATE;
  }
  if (!null_) {
    CK(cudaStreamWaitEvent(st_, ev_sync_, 0), "wait sync");
    CK(cudaMemcpyAsync(arena_, shadow_, (size_t)L_.weights_bytes, cudaMemcpyDeviceToDevice, st_), "swap weights");
    CK(cudaEventRecord(ev_commit_, st_), "record commit");
  }
  ++version;
  sync_pending_ = false;
  return SGS_OK;
}

}  // namespace sgs

// ------------------------------------------------------------------ sgs_rope_table / sgs_comm_unique_id
extern "C" sgs_status sgs_rope_table(float* out, int32_t max_pos, int32_t hd, double theta) {
  if (!out || max_pos <= 0 || hd <= 0 || hd % 2) return SGS_E_INVAL;
  const int half = hd / 2;
  for (int p = 0; p < max_pos; ++p)
    for (int i = 0; i < half; ++i) {
      const double a = (double)p * std::pow(theta, -2.0 * i / (double)hd);
      out[((size_t)p * half + i) * 2] = (float)std::cos(a);
      out[((size_t)p * half + i) * 2 + 1] = (float)std::sin(a);
    }
  return SGS_OK;
}

extern "C" sgs_status sgs_comm_unique_id(uint8_t out[128]) {
  sgs::NcclApi* api = sgs::nccl();
  if (!api) return SGS_E_NCCL;
  ncclUniqueId uid;
  if (api->GetUniqueId(&uid) != ncclSuccess) return SGS_E_NCCL;
  std::memcpy(out, &uid, 128);
  return SGS_OK;
}
