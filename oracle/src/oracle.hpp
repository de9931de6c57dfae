// ORACLE — test infrastructure only.  Plain, slow, obviously-correct CPU code
// that restates what StreamRL's generation stage computes (PAPER.md =
// /root/reference/PAPER.md, cited as P:<line>).  Only tests/, the smoke()
// check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
// leg may load this library.  It shares no code with paper_2504_15930_b200/.
//
// Pins (what each function is checked against) are listed in DESIGN.md §4 and
// in tests/test_oracle_*.py.  Functions with no independent pin say
// "parity unpinned" in their comment.
#pragma once
#include <cstdint>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------------------
// C3: piecewise-linear iteration-time model T(b) (appendix).
// Integer profile: T(b) [ps] = t0_ns*1000 + k0_ps*b            for b <  b*
//                            = t0_ns*1000 + k0_ps*b* + k1_ps*(b-b*)  for b >= b*
// (the second line is k1*b + t1 with t1 derived from continuity).
// ---------------------------------------------------------------------------
struct Profile {
  int64_t t0_ns, k0_ps, b_star, k1_ps;
  int64_t kv_ps = 0;  // R27 predictions: ps per cached context token per iteration (0: T(b) alone)
  int64_t pf_ps = 0;  // R27 predictions: ps per prompt token prefilled in the iteration
};
__int128 T_ps(const Profile& p, int64_t b);

// ---------------------------------------------------------------------------
// C2: per-instance continuous-batching longest-first simulator.
// ---------------------------------------------------------------------------
struct SimSample {
  int64_t id;
  int32_t P, d, hint;
  int32_t batch;          // FIFO batch index (one sgs_submit call)
  int64_t arrival_after;  // queued after this many executed iterations
  int64_t group = -1;     // NEXT-3 prefix sharing: samples of one group share their (identical) prompt
};
struct SimResult {
  std::vector<int64_t> iters;    // per iteration: t,b,sumctx,nadm,ncomp,nalloc,nfree, ids..., pages...
  std::vector<int64_t> samples;  // per sample (ascending id): id,slot,admit,finish,npages,pages...
  int64_t n_iters = 0;
  __int128 time_ps = 0;          // sum_t T(b_t) under the profile
};
SimResult sched_sim(const std::vector<SimSample>& s, int B, int page, int64_t pool_pages,
                    const Profile* prof);

// ---------------------------------------------------------------------------
// C5: Alg. 2 skewness-aware dispatching with Eq. 2.
// ---------------------------------------------------------------------------
struct DispatchIn {
  std::vector<int64_t> id;
  std::vector<int32_t> P, hint;
  int N, B, page;
  int64_t pool_pages;
  Profile prof;
  int alpha_pct;   // 20
  int score_max;   // 0: literal sum, 1: max
  int tail_ceil;   // 0: floor(alpha*n), 1: ceil
};
struct DispatchOut {
  int n_l = 0, n_tail = 0;
  int64_t L_alpha = 0, L_r = 0;
  __int128 score = 0;
  std::vector<int32_t> instance;   // per input sample (input order)
  std::vector<__int128> scores;    // score per N_l = 1..N-1 (empty when degenerate)
};
DispatchOut dispatch(const DispatchIn& in);

// NEXT-4: predicted generation time on N and N + 1 instances and
// the scale-out decision delta >= delta' (elastic.cpp).
struct ElasticOut {
  __int128 t_gen_ps[2] = {0, 0};
  __int128 delta_prime_ps = 0;
  int scale_out = 0;
};
__int128 predicted_generation_ps(const DispatchIn& in);
ElasticOut elastic_plan(const DispatchIn& in, __int128 delta_ps);
// NEXT-2 two-dimensional dispatch (R27); policy of the DP side: 0 Alg. 2, 1 round robin
struct TailPlanOut {
  int n_tail = 0;
  __int128 t_tp = 0, t_dp = 0, t_all = 0;
};
TailPlanOut tp_tail_plan(const DispatchIn& dp, int dp_policy, int tp_size, int tp_B, int64_t tp_pool_pages,
                         const Profile& tp_prof);
int64_t nearest_rank(std::vector<int64_t> v, int q_pct);

// ---------------------------------------------------------------------------
// C3 fit: hinge least squares over measured (b, T) points.
// ---------------------------------------------------------------------------
struct Fit {
  double t0, k0, k1, t1, sse;
  int64_t b_star;
  Profile prof;  // rounded integer profile
  int ok;
};
Fit tb_fit(const std::vector<double>& b, const std::vector<double>& T_ns);
// min over x,y>=1, x+y<=bmax of T(x)+T(y)-T(x+y) in ps (Lemma).
__int128 tb_min_merge_gain(const Profile& p, int64_t bmax, int64_t* ax, int64_t* ay);

// ---------------------------------------------------------------------------
// C4: longest-first vs brute force over all admission orders (M <= 8).
// ---------------------------------------------------------------------------
struct BruteOut {
  __int128 lf_time, opt_time;
  int64_t lf_iters, opt_iters_min;  // iterations of LF, minimum over all orders
};
BruteOut brute_force(const std::vector<int32_t>& d, int B, const Profile& p);
// work-conserving continuous batching for a given admission order
void run_order(const std::vector<int32_t>& d, const std::vector<int>& order, int B, const Profile& p,
               __int128* time, int64_t* iters);

// ---------------------------------------------------------------------------
// C6/C7/C8/K11: decoder, attention, sampler, weight generator.
// ---------------------------------------------------------------------------
struct ModelCfg {
  int n_layers, d, nq, nkv, hd, ffn, vocab;
  double eps, theta;
};
float bf16_round(float x);                                    // IEEE RNE to bf16, returned as float
uint64_t weight_hash(uint64_t seed, uint64_t tensor_id, uint64_t i);
float weight_value(uint64_t seed, uint64_t tensor_id, uint64_t i, int is_norm);
void gen_tensor(uint64_t seed, uint64_t tensor_id, int64_t n, int is_norm, float* out);
uint64_t tensor_checksum(uint64_t seed, uint64_t tensor_id, int64_t n, int is_norm);

void attention_fp64(int nq, int nkv, int hd, int ctx, const float* q, const float* K, const float* V,
                    double* out);

void rmsnorm_bf16(const std::vector<double>& h, int T, int d, const std::vector<float>& w, double eps,
                  std::vector<double>& x);
void rope(double* v, int hd, int pos, double theta);
void decoder_forward(const ModelCfg& c, uint64_t seed, const int32_t* tokens, int T, int first_row,
                     double* logits /* [(T-first_row) x vocab] */, double* dump = nullptr);

// one layer (layer-local parity): h_out = layer(h_in), positions 0..T-1
void decoder_layer(const ModelCfg& c, uint64_t seed, int layer, const double* h_in, int T, double* h_out);
void weight_cache(int on);
void decoder_head(const ModelCfg& c, uint64_t seed, const double* h_in, int T, double* logits);
int32_t argmax_lowest(const float* x, int64_t n);
void philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
int32_t sample_top_p(const float* logits, int64_t V, float temperature, float top_p, uint64_t seed,
                     uint64_t sample_id, uint64_t step);

}  // namespace oracle
