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

}  // namespace oracle
