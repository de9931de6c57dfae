// ORACLE — test infrastructure only (see oracle.hpp).
//
// NEXT-4: dynamic adjustment of the generation stage's DP size (§4.2
// "Dynamic adjustment"): "StreamRL estimates the reduction in
// generation time, delta', achievable by adding one data parallel (DP) unit to
// SGS.  delta' is calculated using the aforementioned profiler and the current
// RL workload.  When delta >= delta', adjustment is triggered by adding one
// more DP unit", with delta the measured gap between generation and training
// time.  Reading (R25): the generation time of a batch on
// N instances is the makespan of Alg. 2's dispatch (C5) with every instance
// running the longest-first continuous-batching schedule (C2) on the ranker's
// hints as output lengths, timed with the fitted T(b) profile (C3):
//     T_gen(N) = max_i sum_t T(b_t^(i)),   delta' = T_gen(N) - T_gen(N + 1).
#include <algorithm>

#include "oracle.hpp"

namespace oracle {

__int128 predicted_generation_ps(const DispatchIn& in) {
  const DispatchOut d = dispatch(in);
  __int128 makespan = 0;
  for (int inst = 0; inst < in.N; ++inst) {
    std::vector<SimSample> mine;
    for (size_t i = 0; i < in.id.size(); ++i)
      if (d.instance[i] == inst)
        mine.push_back(SimSample{in.id[i], in.P[i], in.hint[i], in.hint[i], 0, 0});  // d = hint (predicted)
    if (mine.empty()) continue;
    const SimResult r = sched_sim(mine, in.B, in.page, in.pool_pages, &in.prof);
    makespan = std::max(makespan, r.time_ps);
  }
  return makespan;
}

ElasticOut elastic_plan(const DispatchIn& in, __int128 delta_ps) {
  ElasticOut o;
  DispatchIn a = in, b = in;
  b.N = in.N + 1;
  o.t_gen_ps[0] = predicted_generation_ps(a);
  o.t_gen_ps[1] = predicted_generation_ps(b);
  o.delta_prime_ps = o.t_gen_ps[0] - o.t_gen_ps[1];
  o.scale_out = o.delta_prime_ps > 0 && delta_ps >= o.delta_prime_ps;
  return o;
}

// NEXT-2, tensor parallelism for the long tail (§3 P:390-393 "tensor
// parallelism ... to reduce the per-sample latency"; §5 P:856-861 long-tail
// samples on dedicated instances), reading R27 (the paper gives no rule for
// the split): sort the samples by hint descending (ties: id ascending), send
// the first k to one TP instance and the rest to the DP instances; each side's
// time is the R25 prediction (longest-first schedule on the hints, T(b) of
// its own profile).  k = the smallest k with T_tp(k) >= T_dp(k), found by
// bisection on [0, n], replaced by k - 1 when max(T_tp, T_dp) is not larger
// there.  T_all: every sample on N + tp_size DP instances.

// R25's prediction with the DP side's policy (1 = round robin over the
// (hint desc, id asc) order, as in Alg. 2's "otherwise" branch P:979-981)
static __int128 predicted_policy(const DispatchIn& in, int policy) {
  if (policy == 0 || in.N == 1) return predicted_generation_ps(in);
  const size_t n = in.id.size();
  std::vector<size_t> order(n);
  for (size_t i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    return in.hint[a] != in.hint[b] ? in.hint[a] > in.hint[b] : in.id[a] < in.id[b];
  });
  __int128 makespan = 0;
  for (int inst = 0; inst < in.N; ++inst) {
    std::vector<SimSample> mine;
    for (size_t j = inst; j < n; j += in.N) {
      const size_t i = order[j];
      mine.push_back(SimSample{in.id[i], in.P[i], in.hint[i], in.hint[i], 0, 0});
    }
    if (mine.empty()) continue;
    makespan = std::max(makespan, sched_sim(mine, in.B, in.page, in.pool_pages, &in.prof).time_ps);
  }
  return makespan;
}

TailPlanOut tp_tail_plan(const DispatchIn& dp, int dp_policy, int tp_size, int tp_B, int64_t tp_pool_pages,
                         const Profile& tp_prof) {
  const int n = (int)dp.id.size();
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return dp.hint[a] != dp.hint[b] ? dp.hint[a] > dp.hint[b] : dp.id[a] < dp.id[b];
  });
  // T_tp(k) and T_dp(k) for the split at k
  auto side = [&](int k, __int128* t_tp, __int128* t_dp) {
    DispatchIn tp = dp, rest = dp;
    tp.id.clear(), tp.P.clear(), tp.hint.clear();
    rest.id.clear(), rest.P.clear(), rest.hint.clear();
    for (int j = 0; j < n; ++j) {
      DispatchIn& to = j < k ? tp : rest;
      to.id.push_back(dp.id[order[j]]);
      to.P.push_back(dp.P[order[j]]);
      to.hint.push_back(dp.hint[order[j]]);
    }
    tp.N = 1, tp.B = tp_B, tp.pool_pages = tp_pool_pages, tp.prof = tp_prof;
    *t_tp = k > 0 ? predicted_generation_ps(tp) : 0;
    *t_dp = k < n ? predicted_policy(rest, dp_policy) : 0;
  };
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    __int128 a, b;
    side(mid, &a, &b);
    if (a >= b)
      hi = mid;
    else
      lo = mid + 1;
  }
  TailPlanOut o;
  side(lo, &o.t_tp, &o.t_dp);
  o.n_tail = lo;
  if (lo > 0) {
    __int128 a, b;
    side(lo - 1, &a, &b);
    if (std::max(a, b) <= std::max(o.t_tp, o.t_dp)) o.n_tail = lo - 1, o.t_tp = a, o.t_dp = b;
  }
  DispatchIn all = dp;
  all.N = dp.N + tp_size;
  o.t_all = n > 0 ? predicted_policy(all, dp_policy) : 0;
  return o;
}

}  // namespace oracle
