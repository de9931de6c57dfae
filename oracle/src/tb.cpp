// ORACLE — test infrastructure only (see oracle.hpp).
//
// C3: the iteration-time model of the appendix,
//     T(b) = k0 b + t0 (1 <= b < b*),  k1 b + t1 (b >= b*),
//     0 < k0 < k1, t0, t1 > 0, continuity k0 b* + t0 = k1 b* + t1,
// "profiled in advance".  The fit is ordinary least squares on the
// hinge basis [1, b, max(0, b - b*)] for every candidate b* among the measured
// batch sizes; the candidate with the least SSE wins, ties -> smaller b*
// (R11).  The lemma T(x+y) < T(x) + T(y) is checked
// exhaustively on the integer profile by tb_min_merge_gain.
//
// C4: longest-first versus brute force over all admission orders.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <set>

#include "oracle.hpp"

namespace oracle {

// Solve the 3x3 normal equations (X^T X) beta = X^T y by Gaussian elimination
// with partial pivoting, in double precision.
static bool solve3(double A[3][3], double y[3], double x[3]) {
  int p[3] = {0, 1, 2};
  for (int c = 0; c < 3; ++c) {
    int best = c;
    for (int r = c + 1; r < 3; ++r)
      if (std::fabs(A[r][c]) > std::fabs(A[best][c])) best = r;
    if (std::fabs(A[best][c]) < 1e-300) return false;
    for (int k = 0; k < 3; ++k) std::swap(A[c][k], A[best][k]);
    std::swap(y[c], y[best]);
    std::swap(p[c], p[best]);
    for (int r = c + 1; r < 3; ++r) {
      double f = A[r][c] / A[c][c];
      for (int k = c; k < 3; ++k) A[r][k] -= f * A[c][k];
      y[r] -= f * y[c];
    }
  }
  for (int r = 2; r >= 0; --r) {
    double s = y[r];
    for (int k = r + 1; k < 3; ++k) s -= A[r][k] * x[k];
    x[r] = s / A[r][r];
  }
  return true;
}

Fit tb_fit(const std::vector<double>& b, const std::vector<double>& T) {
  Fit best{};
  best.ok = 0;
  std::set<double> distinct(b.begin(), b.end());
  const size_t n = b.size();
  for (double bs : distinct) {
    // identifiable: >= 2 distinct b <= b*, >= 1 distinct b > b*
    int left = 0, right = 0;
    for (double v : distinct) (v <= bs ? left : right)++;
    if (left < 2 || right < 1) continue;
    double A[3][3] = {{0}}, y[3] = {0};
    for (size_t i = 0; i < n; ++i) {
      double row[3] = {1.0, b[i], std::max(0.0, b[i] - bs)};
      for (int r = 0; r < 3; ++r) {
        y[r] += row[r] * T[i];
        for (int c = 0; c < 3; ++c) A[r][c] += row[r] * row[c];
      }
    }
    double beta[3];
    if (!solve3(A, y, beta)) continue;
    double sse = 0;
    for (size_t i = 0; i < n; ++i) {
      double e = T[i] - (beta[0] + beta[1] * b[i] + beta[2] * std::max(0.0, b[i] - bs));
      sse += e * e;
    }
    if (!best.ok || sse < best.sse) {
      best.ok = 1;
      best.sse = sse;
      best.t0 = beta[0];
      best.k0 = beta[1];
      best.k1 = beta[1] + beta[2];
      best.b_star = (int64_t)bs;
      best.t1 = beta[0] + (beta[1] - best.k1) * bs;  // continuity
    }
  }
  if (best.ok) {
    best.prof.t0_ns = std::llround(best.t0);
    best.prof.k0_ps = std::llround(best.k0 * 1000.0);
    best.prof.k1_ps = std::llround(best.k1 * 1000.0);
    best.prof.b_star = best.b_star;
  }
  return best;
}

__int128 tb_min_merge_gain(const Profile& p, int64_t bmax, int64_t* ax, int64_t* ay) {
  // D(x,y) = T(x) + T(y) - T(x+y), exhaustively over 1 <= x <= y, x + y <= bmax.
  __int128 best = 0;
  bool first = true;
  for (int64_t x = 1; x <= bmax; ++x)
    for (int64_t y = x; x + y <= bmax; ++y) {
      __int128 D = T_ps(p, x) + T_ps(p, y) - T_ps(p, x + y);
      if (first || D < best) {
        best = D;
        first = false;
        if (ax) *ax = x;
        if (ay) *ay = y;
      }
    }
  return best;
}

void run_order(const std::vector<int32_t>& d, const std::vector<int>& order, int B, const Profile& p,
               __int128* time, int64_t* iters) {
  // Work-conserving continuous batching (P:9): whenever a slot is free
  // and samples remain, the next sample in `order` enters immediately.
  std::vector<int> rem;  // remaining iterations of the running samples
  size_t next = 0;
  __int128 tt = 0;
  int64_t it = 0;
  while (next < order.size() || !rem.empty()) {
    while ((int)rem.size() < B && next < order.size()) rem.push_back(d[order[next++]]);
    tt += T_ps(p, (int64_t)rem.size());
    ++it;
    std::vector<int> keep;
    for (int r : rem)
      if (r - 1 > 0) keep.push_back(r - 1);
    rem.swap(keep);
  }
  *time = tt;
  *iters = it;
}

BruteOut brute_force(const std::vector<int32_t>& d, int B, const Profile& p) {
  const int M = (int)d.size();
  std::vector<int> lf(M);
  std::iota(lf.begin(), lf.end(), 0);
  // longest first: d descending, ties by index (= id) ascending
  std::stable_sort(lf.begin(), lf.end(), [&](int a, int b) { return d[a] > d[b]; });
  BruteOut o{};
  run_order(d, lf, B, p, &o.lf_time, &o.lf_iters);
  std::vector<int> perm(M);
  std::iota(perm.begin(), perm.end(), 0);
  bool first = true;
  do {
    __int128 tt;
    int64_t it;
    run_order(d, perm, B, p, &tt, &it);
    if (first || tt < o.opt_time) o.opt_time = tt;
    if (first || it < o.opt_iters_min) o.opt_iters_min = it;
    first = false;
  } while (std::next_permutation(perm.begin(), perm.end()));
  return o;
}

}  // namespace oracle
