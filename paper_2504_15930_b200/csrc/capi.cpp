// extern "C" implementation of include/sgs.h.
#include <cuda_runtime.h>
#include <execinfo.h>
#include <signal.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sgs.h"
#include "engine/engine.hpp"
#include "host/sched.hpp"
#include "kernels/kernels.h"

struct sgs_handle {
  sgs::Engine eng;
};

static thread_local std::string g_init_err;

// SGS_DEBUG_SIGNALS=1: a fatal signal inside the library prints the native
// backtrace (libsgs.so offsets, resolve with addr2line) before the default action
static void sgs_fatal_signal(int sig) {
  void* bt[64];
  const int n = backtrace(bt, 64);
  backtrace_symbols_fd(bt, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
static struct SgsSignalHooks {
  SgsSignalHooks() {
    const char* e = std::getenv("SGS_DEBUG_SIGNALS");
    if (e && e[0] == '1')
      for (int s : {SIGFPE, SIGSEGV, SIGBUS, SIGABRT}) signal(s, sgs_fatal_signal);
  }
} g_signal_hooks;

extern "C" {

sgs_status sgs_arena_bytes(const sgs_model_cfg* m, const sgs_engine_cfg* e, int64_t n_pages, int64_t* fixed_bytes,
                           int64_t* kv_page_bytes) {
  if (!m || !e || n_pages < 0) return SGS_E_INVAL;
  sgs::ArenaLayout L0, L;
  sgs::Engine::layout(*m, *e, 0, &L0);
  sgs::Engine::layout(*m, *e, n_pages, &L);
  if (fixed_bytes) *fixed_bytes = L0.total + 4096;
  if (kv_page_bytes) *kv_page_bytes = L.kv_page_bytes;
  return SGS_OK;
}

sgs_status sgs_weight_tensors(const sgs_model_cfg* m, int64_t* ids, int64_t* rows, int64_t* cols, int32_t cap,
                              int32_t* n) {
  if (!m || !n || cap < 0 || m->n_layers < 0) return SGS_E_INVAL;
  const int64_t d = m->d_model, hd = m->head_dim, nq = m->n_q_heads, nkv = m->n_kv_heads, f = m->d_ffn,
                V = m->vocab;
  std::vector<std::array<int64_t, 3>> t{{0, V, d}, {1, V, d}, {2, d, 1}};
  const int64_t shapes[12][2] = {{nq * hd, d}, {nkv * hd, d}, {nkv * hd, d}, {nq * hd, 1}, {nkv * hd, 1},
                                 {nkv * hd, 1}, {d, nq * hd},  {f, d},       {f, d},       {d, f},
                                 {d, 1},        {d, 1}};
  for (int64_t l = 0; l < m->n_layers; ++l)
    for (int k = 0; k < 12; ++k) t.push_back({16 + 16 * l + k, shapes[k][0], shapes[k][1]});
  *n = (int32_t)t.size();
  for (int32_t i = 0; i < std::min<int32_t>(cap, *n); ++i) {
    if (ids) ids[i] = t[i][0];
    if (rows) rows[i] = t[i][1];
    if (cols) cols[i] = t[i][2];
  }
  return SGS_OK;
}

sgs_status sgs_init(const sgs_model_cfg* m, const sgs_engine_cfg* e, const sgs_weights* weights, sgs_handle** out) {
  if (!m || !e || !out) return SGS_E_INVAL;
  auto* h = new sgs_handle();
  sgs_status s = h->eng.init(*m, *e, weights);
  if (s != SGS_OK) {
    g_init_err = h->eng.err;
    delete h;
    *out = nullptr;
    return s;
  }
  *out = h;
  return SGS_OK;
}

void sgs_destroy(sgs_handle* h) { delete h; }

const char* sgs_last_error(const sgs_handle* h) { return h ? h->eng.err.c_str() : g_init_err.c_str(); }

sgs_status sgs_submit(sgs_handle* h, const sgs_prompt* prompts, int32_t n, const int32_t* hint,
                      const int32_t* forced_len, int32_t* n_mine) {
  if (!h) return SGS_E_INVAL;
  return h->eng.submit(prompts, n, hint, forced_len, n_mine);
}

sgs_status sgs_step(sgs_handle* h, sgs_completion* out, int32_t cap, int32_t* n_out) {
  if (!h || !n_out || cap < 0 || (cap > 0 && !out)) return SGS_E_INVAL;
  return h->eng.step(out, cap, n_out);
}

sgs_status sgs_pending(const sgs_handle* h, int64_t* queued, int64_t* active) {
  if (!h) return SGS_E_INVAL;
  if (queued) *queued = h->eng.sched.queued();
  // samples whose iteration is launched but not yet waited for count as active
  if (active) *active = h->eng.sched.active() + h->eng.inflight_samples();
  return SGS_OK;
}

sgs_status sgs_host_state(const sgs_handle* h, int64_t* records, int64_t* queue_entries, int64_t* live_ids) {
  if (!h) return SGS_E_INVAL;
  if (records) *records = (int64_t)h->eng.sched.records();
  if (queue_entries) *queue_entries = h->eng.sched.queue_entries();
  if (live_ids) *live_ids = h->eng.live_ids();
  return SGS_OK;
}

sgs_status sgs_comm_init(sgs_handle* h, const uint8_t id[128], int32_t rank, int32_t world) {
  if (!h || !id || world < 1 || rank < 0 || rank >= world) return SGS_E_INVAL;
  return h->eng.comm_init(id, rank, world);
}

sgs_status sgs_tp_comm_init(sgs_handle* h, const uint8_t id[128]) {
  if (!h || !id) return SGS_E_INVAL;
  return h->eng.tp_comm_init(id);
}

sgs_status sgs_update_weights(sgs_handle* h, const sgs_weights* src, int32_t root) {
  if (!h) return SGS_E_INVAL;
  return h->eng.update_weights(src, root);
}

sgs_status sgs_stage_weights(sgs_handle* h, const sgs_weights* src) {
  if (!h || !src) return SGS_E_INVAL;
  return h->eng.stage_weights(src);
}

sgs_status sgs_shadow_weights(sgs_handle* h, void** ptr, int64_t* bytes) {
  if (!h || !ptr || !bytes) return SGS_E_INVAL;
  return h->eng.shadow_weights(ptr, bytes);
}

sgs_status sgs_stage_weights_seed(sgs_handle* h, uint64_t seed) {
  if (!h) return SGS_E_INVAL;
  return h->eng.stage_weights_seed(seed);
}

sgs_status sgs_update_weights_begin(sgs_handle* h, int32_t root) {
  if (!h) return SGS_E_INVAL;
  return h->eng.update_weights_begin(root);
}

sgs_status sgs_update_weights_ready(sgs_handle* h, int32_t* ready) {
  if (!h || !ready) return SGS_E_INVAL;
  return h->eng.update_weights_ready(ready);
}

sgs_status sgs_update_weights_commit(sgs_handle* h) {
  if (!h) return SGS_E_INVAL;
  return h->eng.update_weights_commit();
}

sgs_status sgs_load_weights_seed(sgs_handle* h, uint64_t seed) {
  if (!h) return SGS_E_INVAL;
  return h->eng.load_weights_seed(seed);
}

sgs_status sgs_weight_checksum(sgs_handle* h, int64_t tensor_id, uint64_t* out) {
  if (!h || !out) return SGS_E_INVAL;
  return h->eng.checksum(tensor_id, out);
}

sgs_status sgs_weight_version(const sgs_handle* h, int32_t* out) {
  if (!h || !out) return SGS_E_INVAL;
  *out = h->eng.version;
  return SGS_OK;
}

sgs_status sgs_trace(const sgs_handle* h, int32_t which, int64_t* buf, int64_t cap, int64_t* n) {
  if (!h || !n) return SGS_E_INVAL;
  std::vector<int64_t> tmp;
  const std::vector<int64_t>* src;
  if (which == 0) {
    src = &h->eng.sched.trace_iters;
  } else {
    h->eng.sched.sample_trace(&tmp);
    src = &tmp;
  }
  *n = (int64_t)src->size();
  if (buf) std::memcpy(buf, src->data(), sizeof(int64_t) * (size_t)std::min<int64_t>(cap, *n));
  return SGS_OK;
}

sgs_status sgs_trace_clear(sgs_handle* h) {
  if (!h) return SGS_E_INVAL;
  h->eng.sched.trace_iters.clear();
  return SGS_OK;
}

sgs_status sgs_last_logits(sgs_handle* h, float* logits, uint64_t* ids, int32_t* tok_idx, int32_t cap,
                           int32_t* rows) {
  if (!h || !rows) return SGS_E_INVAL;
  return h->eng.last_logits(logits, ids, tok_idx, cap, rows);
}

sgs_status sgs_debug_forward(sgs_handle* h, const int32_t* tokens, int32_t T, float* dump) {
  if (!h || !tokens || !dump) return SGS_E_INVAL;
  return h->eng.debug_forward(tokens, T, dump);
}

sgs_status sgs_debug_layer(sgs_handle* h, int32_t layer, const float* h_in, int32_t T, float* h_out) {
  if (!h || !h_in || !h_out || layer < 0 || layer > h->eng.n_layers()) return SGS_E_INVAL;
  return h->eng.debug_forward(nullptr, T, h_out, layer, h_in);
}

sgs_status sgs_last_iter_ms(sgs_handle* h, float* ms) {
  if (!h || !ms) return SGS_E_INVAL;
  *ms = h->eng.last_ms;
  return SGS_OK;
}

sgs_status sgs_kernel_stats(sgs_handle* h, int32_t cls, double* ms, double* bytes, double* flops, int64_t* launches,
                            int32_t reset) {
  if (!h || cls < 0 || cls >= sgs::Engine::kClasses * sgs::Engine::kPhases) return SGS_E_INVAL;
  auto& E = h->eng;
  if (ms) *ms = E.kstat_ms[cls];
  if (bytes) *bytes = E.kstat_bytes[cls];
  if (flops) *flops = E.kstat_flops[cls];
  if (launches) *launches = E.kstat_n[cls];
  if (reset) E.kstat_ms[cls] = E.kstat_bytes[cls] = E.kstat_flops[cls] = E.kstat_roof_ms[cls] = 0, E.kstat_n[cls] = 0;
  return SGS_OK;
}

sgs_status sgs_set_roofline(sgs_handle* h, double bw_gbs, double tflops) {
  if (!h || bw_gbs <= 0 || tflops <= 0) return SGS_E_INVAL;
  h->eng.roof_bw_gbs = bw_gbs;
  h->eng.roof_tflops = tflops;
  return SGS_OK;
}

sgs_status sgs_kernel_roofline_ms(const sgs_handle* h, int32_t cls, double* ms) {
  if (!h || !ms || cls < 0 || cls >= sgs::Engine::kClasses * sgs::Engine::kPhases) return SGS_E_INVAL;
  *ms = h->eng.kstat_roof_ms[cls];
  return SGS_OK;
}

sgs_status sgs_iter_log(const sgs_handle* h, int64_t* buf, int64_t cap, int64_t* n) {
  if (!h || !n) return SGS_E_INVAL;
  const auto& v = h->eng.iter_log;
  *n = (int64_t)v.size();
  if (buf) std::memcpy(buf, v.data(), sizeof(int64_t) * (size_t)std::min<int64_t>(cap, *n));
  return SGS_OK;
}

sgs_status sgs_io_bytes(const sgs_handle* h, int64_t* h2d, int64_t* d2h) {
  if (!h) return SGS_E_INVAL;
  if (h2d) *h2d = h->eng.h2d_bytes;
  if (d2h) *d2h = h->eng.d2h_bytes;
  return SGS_OK;
}

sgs_status sgs_kernel_launches(const sgs_handle* h, int64_t* n) {
  if (!h || !n) return SGS_E_INVAL;
  *n = h->eng.launches;
  return SGS_OK;
}

sgs_status sgs_fit_profile(int32_t n, const double* b, const double* T_ns, double out[5], sgs_tb_profile* prof) {
  if (n <= 0 || !b || !T_ns || !out || !prof) return SGS_E_INVAL;
  int64_t bs = 0, p[4];
  if (!sgs::fit_tb(n, b, T_ns, out, &bs, p)) return SGS_E_INVAL;
  prof->t0_ns = p[0], prof->k0_ps = p[1], prof->b_star = p[2], prof->k1_ps = p[3];
  return SGS_OK;
}

sgs_status sgs_dispatch_plan(const sgs_engine_cfg* e, int32_t n, const uint64_t* ids, const int32_t* prompt_len,
                             const int32_t* hint, int64_t pool_pages, int32_t* instance, int32_t* n_l) {
  if (!e || n < 0 || (n > 0 && (!ids || !prompt_len || !hint || !instance)) || e->n_instances < 1 ||
      pool_pages < 1)
    return SGS_E_INVAL;
  sgs::DispatchCfg dc{e->n_instances, e->max_batch, e->page_size, pool_pages, e->profile.t0_ns, e->profile.k0_ps,
                      e->profile.b_star, e->profile.k1_ps, e->alpha_pct, e->score, e->tail_ceil, e->dispatch,
                      e->sample_seed};
  const int nl = sgs::dispatch_alg2(dc, n, ids, prompt_len, hint, instance);
  if (n_l) *n_l = nl;
  return SGS_OK;
}

sgs_status sgs_elastic_plan(const sgs_engine_cfg* e, int32_t n, const uint64_t* ids, const int32_t* prompt_len,
                            const int32_t* hint, int64_t pool_pages, int64_t delta_ps, int64_t t_gen_ps[2],
                            int64_t* delta_prime_ps, int32_t* scale_out) {
  if (!e || n < 0 || (n > 0 && (!ids || !prompt_len || !hint)) || e->n_instances < 1 || pool_pages < 1 ||
      e->max_batch < 1 || e->page_size < 1)
    return SGS_E_INVAL;
  sgs::DispatchCfg dc{e->n_instances, e->max_batch, e->page_size, pool_pages, e->profile.t0_ns, e->profile.k0_ps,
                      e->profile.b_star, e->profile.k1_ps, e->alpha_pct, e->score, e->tail_ceil, e->dispatch,
                      e->sample_seed};
  __int128 t[2];
  t[0] = sgs::predicted_generation_ps(dc, n, ids, prompt_len, hint);
  dc.N += 1;
  t[1] = sgs::predicted_generation_ps(dc, n, ids, prompt_len, hint);
  const __int128 dp = t[0] - t[1];
  if (t_gen_ps) t_gen_ps[0] = (int64_t)t[0], t_gen_ps[1] = (int64_t)t[1];
  if (delta_prime_ps) *delta_prime_ps = (int64_t)dp;
  if (scale_out) *scale_out = dp > 0 && (__int128)delta_ps >= dp ? 1 : 0;
  return SGS_OK;
}

sgs_status sgs_tp_tail_plan(const sgs_engine_cfg* e, int64_t pool_pages, int32_t tp_size, int32_t tp_max_batch,
                            int64_t tp_pool_pages, const sgs_tb_profile* tp_profile, int64_t kv_ps, int64_t tp_kv_ps,
                            int64_t pf_ps, int64_t tp_pf_ps, int32_t n, const uint64_t* ids,
                            const int32_t* prompt_len, const int32_t* hint, int32_t* n_tail, int64_t t_ps[3]) {
  if (!e || !tp_profile || n < 0 || (n > 0 && (!ids || !prompt_len || !hint)) || e->n_instances < 1 ||
      pool_pages < 1 || e->max_batch < 1 || e->page_size < 1 || tp_size < 1 || tp_max_batch < 1 || tp_pool_pages < 1 ||
      kv_ps < 0 || tp_kv_ps < 0 || pf_ps < 0 || tp_pf_ps < 0)
    return SGS_E_INVAL;
  sgs::DispatchCfg dp{e->n_instances, e->max_batch, e->page_size, pool_pages, e->profile.t0_ns, e->profile.k0_ps,
                      e->profile.b_star, e->profile.k1_ps, e->alpha_pct, e->score, e->tail_ceil, e->dispatch,
                      e->sample_seed};
  sgs::DispatchCfg tp{1, tp_max_batch, e->page_size, tp_pool_pages, tp_profile->t0_ns, tp_profile->k0_ps,
                      tp_profile->b_star, tp_profile->k1_ps, e->alpha_pct, e->score, e->tail_ceil, e->dispatch,
                      e->sample_seed};
  dp.kv_ps = kv_ps, dp.pf_ps = pf_ps;
  tp.kv_ps = tp_kv_ps, tp.pf_ps = tp_pf_ps;
  const sgs::TailPlan p = sgs::tp_tail_plan(dp, tp, tp_size, n, ids, prompt_len, hint);
  if (n_tail) *n_tail = p.n_tail;
  if (t_ps) t_ps[0] = (int64_t)p.t_tp, t_ps[1] = (int64_t)p.t_dp, t_ps[2] = (int64_t)p.t_all;
  return SGS_OK;
}

sgs_status sgs_set_instances(sgs_handle* h, int32_t n_instances, int32_t instance_rank) {
  if (!h || n_instances < 1 || instance_rank < 0 || instance_rank >= n_instances) return SGS_E_INVAL;
  return h->eng.set_instances(n_instances, instance_rank);
}

// ------------------------------------------------------------------ kernel-level entry points
static sgs_status cuda_status(cudaError_t e) { return e == cudaSuccess ? SGS_OK : SGS_E_CUDA; }

int64_t sgs_attn_workspace_bytes(int32_t b, int32_t nq, int32_t nkv, int32_t hd, int32_t max_pages_per_seq) {
  const int64_t items = (int64_t)b * nkv * max_pages_per_seq + 64;
  return sgs::attn_workspace_bytes((int)items, (int)items, nq / nkv, hd);
}

sgs_status sgs_op_decode_attention(const void* q, const void* kv, const int32_t* block_table, const int32_t* ctx,
                                   int32_t b, int32_t nq, int32_t nkv, int32_t hd, int32_t page,
                                   int32_t max_pages_per_seq, int32_t max_ctx_hint, void* out, int32_t out_fp32,
                                   void* workspace, int64_t workspace_bytes, int32_t split_pages, void* stream) {
  (void)max_ctx_hint;
  if (b <= 0) return SGS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  std::vector<int32_t> hctx(b);
  if (cudaMemcpyAsync(hctx.data(), ctx, (size_t)b * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return SGS_E_CUDA;
  for (int i = 0; i < b; ++i)
    if (hctx[i] < 1 || (hctx[i] + page - 1) / page > max_pages_per_seq) return SGS_E_INVAL;
  sgs::AttnPlan plan;
  sgs::attn_plan(hctx.data(), nullptr, b, nkv, page, split_pages, &plan);
  const int g = nq / nkv;
  const int64_t need = sgs::attn_workspace_bytes((int)plan.items.size(), plan.n_parts, g, hd);
  if (need > workspace_bytes) return SGS_E_NOMEM;
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  auto* d_items = reinterpret_cast<sgs::AttnItem*>(ws);
  auto* d_combs = reinterpret_cast<sgs::AttnComb*>(ws + plan.items.size() * sizeof(sgs::AttnItem));
  size_t off = plan.items.size() * sizeof(sgs::AttnItem) + plan.combs.size() * sizeof(sgs::AttnComb);
  off = (off + 255) / 256 * 256;
  float* part_o = reinterpret_cast<float*>(ws + off);
  float* part_ml = part_o + (size_t)std::max(plan.n_parts, 1) * g * hd;
  if (cudaMemcpyAsync(d_items, plan.items.data(), plan.items.size() * sizeof(sgs::AttnItem), cudaMemcpyHostToDevice,
                      st) != cudaSuccess)
    return SGS_E_CUDA;
  if (!plan.combs.empty() &&
      cudaMemcpyAsync(d_combs, plan.combs.data(), plan.combs.size() * sizeof(sgs::AttnComb), cudaMemcpyHostToDevice,
                      st) != cudaSuccess)
    return SGS_E_CUDA;
  int* arrive = reinterpret_cast<int*>(part_ml + (size_t)std::max(plan.n_parts, 1) * g * 2);
  if (!plan.combs.empty() && cudaMemsetAsync(arrive, 0, plan.combs.size() * sizeof(int), st) != cudaSuccess)
    return SGS_E_CUDA;
  cudaError_t e = sgs::attn_decode(q, kv, block_table, nullptr, d_items, (int)plan.items.size(), d_combs,
                                   (int)plan.combs.size(), nq, nkv, hd, page, max_pages_per_seq, out, out_fp32,
                                   part_o, part_ml, arrive, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // host plan vectors die here
  return cuda_status(e);
}

sgs_status sgs_op_decode_attention_timed(const void* q, const void* kv, const int32_t* block_table,
                                         const int32_t* ctx, int32_t b, int32_t nq, int32_t nkv, int32_t hd,
                                         int32_t page, int32_t max_pages_per_seq, void* out, void* workspace,
                                         int64_t workspace_bytes, int32_t reps, void* l2_flush,
                                         int64_t l2_flush_bytes, float* ms, void* stream) {
  if (b <= 0 || reps <= 0 || !ms) return SGS_E_INVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  std::vector<int32_t> hctx(b);
  if (cudaMemcpyAsync(hctx.data(), ctx, (size_t)b * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return SGS_E_CUDA;
  for (int i = 0; i < b; ++i)
    if (hctx[i] < 1 || (hctx[i] + page - 1) / page > max_pages_per_seq) return SGS_E_INVAL;
  sgs::AttnPlan plan;
  sgs::attn_plan(hctx.data(), nullptr, b, nkv, page, 0, &plan);
  const int g = nq / nkv;
  if (sgs::attn_workspace_bytes((int)plan.items.size(), plan.n_parts, g, hd) > workspace_bytes) return SGS_E_NOMEM;
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  auto* d_items = reinterpret_cast<sgs::AttnItem*>(ws);
  auto* d_combs = reinterpret_cast<sgs::AttnComb*>(ws + plan.items.size() * sizeof(sgs::AttnItem));
  size_t off = plan.items.size() * sizeof(sgs::AttnItem) + plan.combs.size() * sizeof(sgs::AttnComb);
  off = (off + 255) / 256 * 256;
  float* part_o = reinterpret_cast<float*>(ws + off);
  float* part_ml = part_o + (size_t)std::max(plan.n_parts, 1) * g * hd;
  int* arrive = reinterpret_cast<int*>(part_ml + (size_t)std::max(plan.n_parts, 1) * g * 2);
  cudaError_t e = cudaMemcpyAsync(d_items, plan.items.data(), plan.items.size() * sizeof(sgs::AttnItem),
                                  cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && !plan.combs.empty())
    e = cudaMemcpyAsync(d_combs, plan.combs.data(), plan.combs.size() * sizeof(sgs::AttnComb),
                        cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && !plan.combs.empty()) e = cudaMemsetAsync(arrive, 0, plan.combs.size() * sizeof(int), st);
  auto launch = [&]() {
    return sgs::attn_decode(q, kv, block_table, nullptr, d_items, (int)plan.items.size(), d_combs,
                            (int)plan.combs.size(), nq, nkv, hd, page, max_pages_per_seq, out, 0, part_o, part_ml,
                            arrive, st);
  };
  if (e == cudaSuccess) e = launch();  // warm-up
  std::vector<cudaEvent_t> ev(2 * (size_t)reps, nullptr);
  for (auto& x : ev)
    if (e == cudaSuccess) e = cudaEventCreate(&x);
  for (int r = 0; r < reps && e == cudaSuccess; ++r) {
    if (l2_flush && l2_flush_bytes > 0) e = cudaMemsetAsync(l2_flush, r & 0xff, (size_t)l2_flush_bytes, st);
    if (e == cudaSuccess) e = cudaEventRecord(ev[2 * r], st);
    if (e == cudaSuccess) e = launch();
    if (e == cudaSuccess) e = cudaEventRecord(ev[2 * r + 1], st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  float tot = 0.f;
  for (int r = 0; r < reps && e == cudaSuccess; ++r) {
    float t = 0.f;
    e = cudaEventElapsedTime(&t, ev[2 * r], ev[2 * r + 1]);
    tot += t;
  }
  for (auto& x : ev)
    if (x) cudaEventDestroy(x);
  *ms = tot / reps;
  return cuda_status(e);
}

sgs_status sgs_op_gemm(const void* W, const void* X, void* C, int32_t N, int32_t K, int32_t T, int32_t ldc,
                       int32_t mode, int32_t splits, void* stream) {
  if (!W || !X || !C || N <= 0 || K <= 0 || T < 0 || mode < 0 || mode > 3) return SGS_E_INVAL;
  if (mode == 3 && (splits > 1 || ldc * 2 != N)) return SGS_E_INVAL;
  if (N % 128 || K % 64) return SGS_E_UNSUPPORTED;
  return cuda_status(sgs::gemm_bf16(W, X, reinterpret_cast<float*>(C), N, K, T, ldc, mode, splits,
                                    reinterpret_cast<cudaStream_t>(stream)));
}

sgs_status sgs_op_rmsnorm(const float* x, const void* w, void* y, int32_t T, int32_t d, float eps, void* stream) {
  if (!x || !w || !y || T < 0 || d <= 0) return SGS_E_INVAL;
  return cuda_status(sgs::rmsnorm(x, w, y, nullptr, T, d, eps, reinterpret_cast<cudaStream_t>(stream)));
}

sgs_status sgs_op_rope_append(const float* qkv, const void* bias, const int32_t* pos, const int32_t* slot,
                              const int32_t* block_table, int32_t max_pages_per_seq, const float* cos_sin,
                              void* q_out, void* kv, int32_t T, int32_t nq, int32_t nkv, int32_t hd, int32_t page,
                              void* stream) {
  if (!qkv || !pos || !cos_sin || !q_out || T < 0) return SGS_E_INVAL;
  return cuda_status(sgs::rope_append(qkv, bias, pos, slot, block_table, max_pages_per_seq, cos_sin, q_out, kv,
                                      nullptr, nullptr, T, nq, nkv, hd, page, reinterpret_cast<cudaStream_t>(stream)));
}

int64_t sgs_prefill_workspace_bytes(int32_t T, int32_t n_prompts, int32_t nkv, int32_t hd) {
  // (prompt, query block) pairs: sum ceil(len/64) <= T/64 + n_prompts; plus
  // the fp16 copy of v for the tcgen05 kernel (hd 128)
  const int64_t blocks = 8 * ((int64_t)(T > 0 ? T : 0) / 64 + (n_prompts > 0 ? n_prompts : 0) + 1);
  return (blocks + 255) / 256 * 256 + (hd == 128 ? (int64_t)(T > 0 ? T : 0) * nkv * hd * 2 : 0);
}

sgs_status sgs_op_prefill_attention(const void* q, const void* k, const void* v, const int32_t* offs,
                                    int32_t n_prompts, int32_t nq, int32_t nkv, int32_t hd, void* out,
                                    void* workspace, int64_t workspace_bytes, void* stream) {
  if (!q || !k || !v || !offs || !out || n_prompts < 0 || nq <= 0 || nkv <= 0 || nq % nkv) return SGS_E_INVAL;
  if (n_prompts == 0) return SGS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  std::vector<int32_t> ho(n_prompts + 1);
  if (cudaMemcpyAsync(ho.data(), offs, ho.size() * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return SGS_E_CUDA;
  const int T = ho[n_prompts];
  const bool tc = hd == 128 && !(std::getenv("SGS_PREFILL_LEGACY") && std::atoi(std::getenv("SGS_PREFILL_LEGACY")));
  const int blk = tc ? 128 : 64;
  std::vector<int32_t> qb;
  for (int p = 0; p < n_prompts; ++p)
    for (int b = 0; b < (ho[p + 1] - ho[p] + blk - 1) / blk; ++b) qb.push_back(p), qb.push_back(b);
  if (qb.empty()) return SGS_OK;
  if (!workspace || sgs_prefill_workspace_bytes(T, n_prompts, nkv, hd) > workspace_bytes) return SGS_E_NOMEM;
  int32_t* d_qb = reinterpret_cast<int32_t*>(workspace);
  cudaError_t e = cudaMemcpyAsync(d_qb, qb.data(), qb.size() * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && tc) {
    // the kernel's P.V operand: fp16(bf16 v) (exact), in the workspace
    const int64_t blocks = 8 * ((int64_t)T / 64 + n_prompts + 1);
    void* vh = reinterpret_cast<uint8_t*>(workspace) + (blocks + 255) / 256 * 256;
    e = sgs::bf16_to_f16(v, vh, (int64_t)T * nkv * hd, st);
    if (e == cudaSuccess)
      e = sgs::attn_prefill_tc(q, k, vh, offs, d_qb, (int)qb.size() / 2, T, nq, nkv, out, st);
  } else if (e == cudaSuccess) {
    e = sgs::attn_prefill(q, k, v, offs, d_qb, (int)qb.size() / 2, nq, nkv, hd, out, st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the host block list dies here
  return cuda_status(e);
}

sgs_status sgs_op_silu_mul(const float* gu, void* m, int32_t T, int32_t f, void* stream) {
  if (!gu || !m || T < 0 || f <= 0 || f % 2) return SGS_E_INVAL;
  return cuda_status(sgs::silu_mul(gu, m, T, f, reinterpret_cast<cudaStream_t>(stream)));
}

sgs_status sgs_op_sample_top_p(const float* logits, int32_t rows, int32_t V, float temperature, float top_p,
                               uint64_t seed, const uint64_t* sample_ids, const int32_t* steps, int32_t* ids,
                               void* stream) {
  if (!logits || !ids || !sample_ids || !steps || rows < 0 || V <= 0 || !(top_p > 0.f)) return SGS_E_INVAL;
  return cuda_status(sgs::sample_top_p(logits, rows, V, temperature, top_p, seed,
                                       reinterpret_cast<const uint32_t*>(sample_ids), ids, nullptr, steps, nullptr,
                                       nullptr, 0, reinterpret_cast<cudaStream_t>(stream)));
}

sgs_status sgs_op_argmax(const float* logits, int32_t rows, int32_t V, int32_t* ids, void* stream) {
  if (!logits || !ids || rows < 0 || V <= 0) return SGS_E_INVAL;
  return cuda_status(sgs::argmax_rows(logits, rows, V, ids, nullptr, nullptr, nullptr, nullptr, 0,
                                      reinterpret_cast<cudaStream_t>(stream)));
}

}  // extern "C"
