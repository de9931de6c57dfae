// ORACLE — test infrastructure only (see oracle.hpp).  extern "C" surface for
// ctypes (oracle/__init__.py).  Results that are variable-length come back as
// an int64 blob: call once with out == NULL to get the length, then again.
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracle.hpp"

using namespace oracle;

static std::string g_err;
static std::vector<int64_t> g_blob_iters, g_blob_samples;

static void split128(__int128 v, int64_t* out2) {
  out2[0] = (int64_t)(v >> 64);
  out2[1] = (int64_t)(uint64_t)v;
}

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

float oracle_bf16_round(float x) { return bf16_round(x); }

// Returns number of iterations (>=0) or -1 on error.  Blobs retrievable via
// oracle_sched_blob.  time_ps128 receives {hi, lo} of sum_t T(b_t).
int64_t oracle_sched_sim(int32_t n, const int64_t* ids, const int32_t* P, const int32_t* d,
                         const int32_t* hint, const int32_t* batch, const int64_t* arrival_after, int32_t B,
                         int32_t page, int64_t pool_pages, const int64_t* profile4, int64_t* time_ps128,
                         const int64_t* group) {
  try {
    std::vector<SimSample> s(n);
    for (int i = 0; i < n; ++i)
      s[i] = SimSample{ids[i], P[i], d[i], hint[i], batch ? batch[i] : 0, arrival_after ? arrival_after[i] : 0,
                       group ? group[i] : -1};
    Profile prof{};
    if (profile4) prof = Profile{profile4[0], profile4[1], profile4[2], profile4[3]};
    SimResult r = sched_sim(s, B, page, pool_pages, profile4 ? &prof : nullptr);
    g_blob_iters = std::move(r.iters);
    g_blob_samples = std::move(r.samples);
    if (time_ps128) split128(r.time_ps, time_ps128);
    return r.n_iters;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// which: 0 = iteration records, 1 = per-sample records
int64_t oracle_sched_blob(int32_t which, int64_t* out) {
  auto& b = which == 0 ? g_blob_iters : g_blob_samples;
  if (out) std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
  return (int64_t)b.size();
}

// Alg. 2.  out_instance[n]; info[8] = {n_l, n_tail, L_alpha, L_r, score_hi, score_lo, 0, 0};
// scores128[2*(N-1)] optional.
int32_t oracle_dispatch(int32_t n, const int64_t* ids, const int32_t* P, const int32_t* hint, int32_t N, int32_t B,
                        int32_t page, int64_t pool_pages, const int64_t* profile4, int32_t alpha_pct,
                        int32_t score_max, int32_t tail_ceil, int32_t* out_instance, int64_t* info,
                        int64_t* scores128) {
  DispatchIn in;
  in.id.assign(ids, ids + n);
  in.P.assign(P, P + n);
  in.hint.assign(hint, hint + n);
  in.N = N, in.B = B, in.page = page, in.pool_pages = pool_pages;
  in.prof = Profile{profile4[0], profile4[1], profile4[2], profile4[3]};
  in.alpha_pct = alpha_pct, in.score_max = score_max, in.tail_ceil = tail_ceil;
  DispatchOut o = dispatch(in);
  for (int i = 0; i < n; ++i) out_instance[i] = o.instance[i];
  info[0] = o.n_l, info[1] = o.n_tail, info[2] = o.L_alpha, info[3] = o.L_r;
  split128(o.score, info + 4);
  info[6] = (int64_t)o.scores.size(), info[7] = 0;
  if (scores128)
    for (size_t i = 0; i < o.scores.size(); ++i) split128(o.scores[i], scores128 + 2 * i);
  return 0;
}

// NEXT-4: out128 = {t_gen(N) hi, lo, t_gen(N+1) hi, lo, delta' hi, lo}, returns the decision
int32_t oracle_elastic_plan(int32_t n, const int64_t* ids, const int32_t* P, const int32_t* hint, int32_t N, int32_t B,
                            int32_t page, int64_t pool_pages, const int64_t* profile4, int32_t alpha_pct,
                            int32_t score_max, int32_t tail_ceil, int64_t delta_ps, int64_t* out128) {
  DispatchIn in;
  in.id.assign(ids, ids + n);
  in.P.assign(P, P + n);
  in.hint.assign(hint, hint + n);
  in.N = N, in.B = B, in.page = page, in.pool_pages = pool_pages;
  in.prof = Profile{profile4[0], profile4[1], profile4[2], profile4[3]};
  in.alpha_pct = alpha_pct, in.score_max = score_max, in.tail_ceil = tail_ceil;
  const ElasticOut o = elastic_plan(in, (__int128)delta_ps);
  split128(o.t_gen_ps[0], out128);
  split128(o.t_gen_ps[1], out128 + 2);
  split128(o.delta_prime_ps, out128 + 4);
  return o.scale_out;
}

// NEXT-2: out128 = {t_tp hi, lo, t_dp hi, lo, t_all hi, lo}; returns n_tail
int32_t oracle_tp_tail_plan(int32_t n, const int64_t* ids, const int32_t* P, const int32_t* hint, int32_t N, int32_t B,
                            int32_t page, int64_t pool_pages, const int64_t* profile4, int32_t alpha_pct,
                            int32_t score_max, int32_t tail_ceil, int32_t policy, int32_t tp_size, int32_t tp_B,
                            int64_t tp_pool_pages, const int64_t* tp_profile4, int64_t kv_ps, int64_t tp_kv_ps,
                            int64_t pf_ps, int64_t tp_pf_ps, int64_t* out128) {
  DispatchIn in;
  in.id.assign(ids, ids + n);
  in.P.assign(P, P + n);
  in.hint.assign(hint, hint + n);
  in.N = N, in.B = B, in.page = page, in.pool_pages = pool_pages;
  in.prof = Profile{profile4[0], profile4[1], profile4[2], profile4[3], kv_ps, pf_ps};
  in.alpha_pct = alpha_pct, in.score_max = score_max, in.tail_ceil = tail_ceil;
  const TailPlanOut o = tp_tail_plan(in, policy, tp_size, tp_B, tp_pool_pages,
                                     Profile{tp_profile4[0], tp_profile4[1], tp_profile4[2], tp_profile4[3], tp_kv_ps,
                                             tp_pf_ps});
  split128(o.t_tp, out128);
  split128(o.t_dp, out128 + 2);
  split128(o.t_all, out128 + 4);
  return o.n_tail;
}

int64_t oracle_nearest_rank(int32_t n, const int64_t* v, int32_t q_pct) {
  return nearest_rank(std::vector<int64_t>(v, v + n), q_pct);
}

void oracle_T_ps(const int64_t* profile4, int64_t b, int64_t* out128) {
  Profile p{profile4[0], profile4[1], profile4[2], profile4[3]};
  split128(T_ps(p, b), out128);
}

// fit: out_d[5] = {t0, k0, k1, t1, sse}; out_i[5] = {ok, b_star, t0_ns, k0_ps, k1_ps}
void oracle_tb_fit(int32_t n, const double* b, const double* T_ns, double* out_d, int64_t* out_i) {
  Fit f = tb_fit(std::vector<double>(b, b + n), std::vector<double>(T_ns, T_ns + n));
  out_d[0] = f.t0, out_d[1] = f.k0, out_d[2] = f.k1, out_d[3] = f.t1, out_d[4] = f.sse;
  out_i[0] = f.ok, out_i[1] = f.b_star, out_i[2] = f.prof.t0_ns, out_i[3] = f.prof.k0_ps, out_i[4] = f.prof.k1_ps;
}

// out4 = {gain_hi, gain_lo, x, y}
void oracle_tb_min_merge_gain(const int64_t* profile4, int64_t bmax, int64_t* out4) {
  Profile p{profile4[0], profile4[1], profile4[2], profile4[3]};
  int64_t x = 0, y = 0;
  split128(tb_min_merge_gain(p, bmax, &x, &y), out4);
  out4[2] = x, out4[3] = y;
}

// out6 = {lf_time hi, lo, opt_time hi, lo, lf_iters, opt_iters_min}
void oracle_brute_force(int32_t M, const int32_t* d, int32_t B, const int64_t* profile4, int64_t* out6) {
  Profile p{profile4[0], profile4[1], profile4[2], profile4[3]};
  BruteOut o = brute_force(std::vector<int32_t>(d, d + M), B, p);
  split128(o.lf_time, out6);
  split128(o.opt_time, out6 + 2);
  out6[4] = o.lf_iters, out6[5] = o.opt_iters_min;
}

void oracle_run_order(int32_t M, const int32_t* d, const int32_t* order, int32_t B, const int64_t* profile4,
                      int64_t* out3) {
  Profile p{profile4[0], profile4[1], profile4[2], profile4[3]};
  __int128 t;
  int64_t it;
  run_order(std::vector<int32_t>(d, d + M), std::vector<int>(order, order + M), B, p, &t, &it);
  split128(t, out3);
  out3[2] = it;
}

void oracle_attention(int32_t nq, int32_t nkv, int32_t hd, int32_t ctx, const float* q, const float* K,
                      const float* V, double* out) {
  attention_fp64(nq, nkv, hd, ctx, q, K, V, out);
}

void oracle_gen_tensor(uint64_t seed, uint64_t tensor_id, int64_t n, int32_t is_norm, float* out) {
  gen_tensor(seed, tensor_id, n, is_norm, out);
}

uint64_t oracle_tensor_checksum(uint64_t seed, uint64_t tensor_id, int64_t n, int32_t is_norm) {
  return tensor_checksum(seed, tensor_id, n, is_norm);
}

uint64_t oracle_weight_hash(uint64_t seed, uint64_t tensor_id, uint64_t i) { return weight_hash(seed, tensor_id, i); }

// cfg_i = {n_layers, d, nq, nkv, hd, ffn, vocab}; cfg_d = {eps, theta}
int32_t oracle_decoder_forward(const int32_t* cfg_i, const double* cfg_d, uint64_t seed, const int32_t* tokens,
                               int32_t T, int32_t first_row, double* logits) {
  try {
    ModelCfg c{cfg_i[0], cfg_i[1], cfg_i[2], cfg_i[3], cfg_i[4], cfg_i[5], cfg_i[6], cfg_d[0], cfg_d[1]};
    decoder_forward(c, seed, tokens, T, first_row, logits);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// residual stream after the embedding and after every residual add: dump [(2L+1) x T x d]
int32_t oracle_decoder_dump(const int32_t* cfg_i, const double* cfg_d, uint64_t seed, const int32_t* tokens,
                            int32_t T, double* dump) {
  try {
    ModelCfg c{cfg_i[0], cfg_i[1], cfg_i[2], cfg_i[3], cfg_i[4], cfg_i[5], cfg_i[6], cfg_d[0], cfg_d[1]};
    std::vector<double> logits((size_t)c.vocab);
    decoder_forward(c, seed, tokens, T, T - 1, logits.data(), dump);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void oracle_weight_cache(int32_t on) { weight_cache(on); }

int32_t oracle_decoder_head(const int32_t* cfg_i, const double* cfg_d, uint64_t seed, const double* h_in, int32_t T,
                            double* logits) {
  ModelCfg c{cfg_i[0], cfg_i[1], cfg_i[2], cfg_i[3], cfg_i[4], cfg_i[5], cfg_i[6], cfg_d[0], cfg_d[1]};
  decoder_head(c, seed, h_in, T, logits);
  return 0;
}

int32_t oracle_decoder_layer(const int32_t* cfg_i, const double* cfg_d, uint64_t seed, int32_t layer,
                             const double* h_in, int32_t T, double* h_out) {
  ModelCfg c{cfg_i[0], cfg_i[1], cfg_i[2], cfg_i[3], cfg_i[4], cfg_i[5], cfg_i[6], cfg_d[0], cfg_d[1]};
  decoder_layer(c, seed, layer, h_in, T, h_out);
  return 0;
}

// y = bf16(x / sqrt(mean(x^2) + eps) * w), rows of x [T x d]
void oracle_rmsnorm(const double* x, const float* w, int32_t T, int32_t d, double eps, double* y) {
  std::vector<double> h(x, x + (size_t)T * d), out;
  rmsnorm_bf16(h, T, d, std::vector<float>(w, w + d), eps, out);
  std::memcpy(y, out.data(), sizeof(double) * (size_t)T * d);
}

// NeoX rotate-half RoPE of one head vector (in place, fp64)
void oracle_rope(double* v, int32_t hd, int32_t pos, double theta) { rope(v, hd, pos, theta); }

int32_t oracle_argmax(const float* x, int64_t n) { return argmax_lowest(x, n); }

void oracle_philox(const uint32_t* ctr4, const uint32_t* key2, uint32_t* out4) { philox4x32_10(ctr4, key2, out4); }

int32_t oracle_sample_top_p(const float* logits, int64_t V, float temperature, float top_p, uint64_t seed,
                            uint64_t sample_id, uint64_t step) {
  return sample_top_p(logits, V, temperature, top_p, seed, sample_id, step);
}

}  // extern "C"
