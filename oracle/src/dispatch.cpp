// ORACLE — test infrastructure only (see oracle.hpp).
//
// C5: Alg. 2 "Skewness-aware Dispatching Algorithm" (§5.3) with the
// per-instance latency of Eq. 2:
//     Latency = PTL(BS) * L_avg * ceil(M / BS),
// BS limited by KV memory.  Readings (R6-R10):
//   * sort by estimated length descending, ties by id ascending,
//   * P_alpha = the first floor(alpha% * |P|) samples (ceil is a flag),
//   * L_alpha = P90, L_r = P50 of D = this batch's hints, nearest rank,
//   * total latency = literal sum of the two groups or max (flag),
//   * argmin over N_l = 1..N-1, ties -> smaller N_l,
//   * "evenly distributed within their respective instances" =
//     round-robin in sorted order.
// All arithmetic is integer (picoseconds, 128-bit) so both sides agree bit for bit.
#include <algorithm>
#include <numeric>

#include "oracle.hpp"

namespace oracle {

int64_t nearest_rank(std::vector<int64_t> v, int q_pct) {
  // ceil(q * n)-th smallest value (1-based); nearest-rank percentile.
  std::sort(v.begin(), v.end());
  int64_t n = (int64_t)v.size();
  int64_t rank = (q_pct * n + 99) / 100;
  if (rank < 1) rank = 1;
  return v[rank - 1];
}

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Eq. 2 for a group of `count` samples spread over `n_inst` instances.
static __int128 group_latency(int64_t count, int64_t L, int n_inst, const DispatchIn& in,
                              int64_t mean_prompt) {
  if (count == 0) return 0;
  int64_t M = cdiv(count, n_inst);
  int64_t per_sample_pages = cdiv(mean_prompt + L - 1, in.page);
  int64_t mem_bs = in.pool_pages / per_sample_pages;
  int64_t BS = std::min<int64_t>(M, std::min<int64_t>(in.B, mem_bs));
  if (BS < 1) BS = 1;
  return T_ps(in.prof, BS) * (__int128)L * (__int128)cdiv(M, BS);
}

DispatchOut dispatch(const DispatchIn& in) {
  DispatchOut out;
  const int n = (int)in.id.size();
  out.instance.assign(n, 0);
  if (n == 0) return out;
  // Sort(P, L, descending)
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int a, int b) {
    if (in.hint[a] != in.hint[b]) return in.hint[a] > in.hint[b];
    return in.id[a] < in.id[b];
  });
  int64_t n_tail = in.tail_ceil ? ((int64_t)in.alpha_pct * n + 99) / 100 : ((int64_t)in.alpha_pct * n) / 100;
  if (n_tail > n) n_tail = n;
  out.n_tail = (int)n_tail;
  std::vector<int64_t> D(in.hint.begin(), in.hint.end());
  out.L_alpha = nearest_rank(D, 90);
  out.L_r = nearest_rank(D, 50);
  int64_t sumP = 0;
  for (int i = 0; i < n; ++i) sumP += in.P[i];
  int64_t mean_prompt = cdiv(sumP, n);
  const int N = in.N;
  int64_t n_reg = n - n_tail;
  int n_l;
  if (N == 1 || n_tail == 0 || n_reg == 0) {
    // degenerate: a single group over all instances
    n_l = (n_reg == 0 && N > 1) ? N : 0;
    if (N == 1) n_l = 0;
    out.score = n_l == 0 ? group_latency(n, out.L_r, N, in, mean_prompt)
                         : group_latency(n, out.L_alpha, N, in, mean_prompt);
  } else {
    // for N_l, N_r such that N_l + N_r = N
    __int128 best = 0;
    n_l = -1;
    for (int nl = 1; nl <= N - 1; ++nl) {
      __int128 la = group_latency(n_tail, out.L_alpha, nl, in, mean_prompt);
      __int128 lr = group_latency(n_reg, out.L_r, N - nl, in, mean_prompt);
      __int128 tot = in.score_max ? std::max(la, lr) : la + lr;
      out.scores.push_back(tot);
      if (n_l < 0 || tot < best) {  // strict: ties keep the smaller N_l
        best = tot;
        n_l = nl;
      }
    }
    out.score = best;
  }
  out.n_l = n_l;
  // evenly distribute within each group, round-robin in sorted order
  int tail_groups = n_l, reg_groups = N - n_l;
  for (int j = 0; j < n; ++j) {
    int i = ord[j];
    bool tail = j < n_tail && n_l > 0;
    if (n_l == 0) tail = false;
    if (reg_groups == 0) tail = true;
    if (tail)
      out.instance[i] = j % tail_groups;
    else {
      int jr = n_l == 0 ? j : j - (int)n_tail;
      out.instance[i] = n_l + jr % reg_groups;
    }
  }
  return out;
}

}  // namespace oracle
