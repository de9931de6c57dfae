// Host control plane: page allocator, longest-first scheduler, Alg. 2, T(b) fit.
//
// Scheduler semantics (P = PAPER.md):
//  * order: RL batches FIFO; within a batch by ranker hint descending, id
//    ascending — "samples are assigned to the batch in descending order of
//    their estimated output lengths. Once a sample is completed, the sample
//    with the longest remaining output length is added";
//  * refill: free slots (lowest index first) are filled from the queue head
//    while active < B and the head's page reservation ceil((P+d-1)/page)
//    fits the pool (BS "constrained by the GPU memory capacity");
//    strict order, no backfill;
//  * every active sample produces one token per iteration (prefill counts as
//    the first) and completes after exactly d tokens (forced lengths,
//    P:1105-1110); completions stream out in ascending id.
#include "sched.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>

namespace sgs {

// ------------------------------------------------------------------ PageAllocator
void PageAllocator::reset(int64_t n) {
  n_ = n;
  n_free_ = n;
  words_.assign((size_t)((n + 63) / 64), ~0ull);
  if (n % 64) words_.back() = (1ull << (n % 64)) - 1;
  if (n == 0) words_.clear();
  summary_.assign((words_.size() + 63) / 64, 0ull);
  for (size_t w = 0; w < words_.size(); ++w)
    if (words_[w]) summary_[w / 64] |= 1ull << (w % 64);
}

int64_t PageAllocator::alloc() {
  for (size_t s = 0; s < summary_.size(); ++s) {
    if (!summary_[s]) continue;
    const size_t w = s * 64 + (size_t)__builtin_ctzll(summary_[s]);
    const int bit = __builtin_ctzll(words_[w]);
    words_[w] &= words_[w] - 1;
    if (!words_[w]) summary_[s] &= ~(1ull << (w % 64));
    --n_free_;
    return (int64_t)w * 64 + bit;
  }
  return -1;
}

void PageAllocator::free(int64_t p) {
  const size_t w = (size_t)(p / 64);
  words_[w] |= 1ull << (p % 64);
  summary_[w / 64] |= 1ull << (w % 64);
  ++n_free_;
}

// ------------------------------------------------------------------ Scheduler
void Scheduler::init(int max_batch, int page, int64_t n_pages) {
  B_ = max_batch;
  page_ = page;
  pages_.reset(n_pages);
  slot_of_.assign(max_batch, -1);
}

// pages a sample owns: all of its block table, except the leading
// floor((P-1)/page) prompt pages a prefix group shares (R26)
static inline int64_t shared_pages(const Sample& s, int page) { return s.group >= 0 ? (int64_t)(s.P - 1) / page : 0; }
static inline int64_t reservation(const Sample& s, int page) {
  return ((int64_t)s.P + s.d - 1 + page - 1) / page - shared_pages(s, page);
}

void Scheduler::submit(std::vector<Sample>&& batch) {
  // drop the consumed queue prefix once it dominates the queue
  if (qhead_ >= 1024 && 2 * qhead_ >= queue_.size()) {
    queue_.erase(queue_.begin(), queue_.begin() + (std::ptrdiff_t)qhead_);
    qhead_ = 0;
  }
  std::vector<int32_t> idx;
  idx.reserve(batch.size());
  for (auto& s : batch) {
    if (s.group >= 0) ++groups_[s.group].remain;
    if (!tracing && !free_idx_.empty()) {
      idx.push_back(free_idx_.back());
      free_idx_.pop_back();
      samples_[idx.back()] = std::move(s);
    } else {
      idx.push_back((int32_t)samples_.size());
      samples_.push_back(std::move(s));
    }
  }
  std::sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
    const Sample &x = samples_[a], &y = samples_[b];
    if (x.hint != y.hint) return x.hint > y.hint;
    return x.id < y.id;
  });
  queue_.insert(queue_.end(), idx.begin(), idx.end());
}

bool Scheduler::plan(IterPlan* p) {
  p->admitted.clear();
  p->running.clear();
  p->completed.clear();
  p->bt_deltas.clear();
  p->alloc_log.clear();
  p->free_log.clear();
  p->admitted_decode.clear();
  p->copies_after_prefill.clear();
  p->copies_before_decode.clear();
  if (idle()) return false;
  // records of the samples completed by the previous plan are free from now on
  if (!tracing) {
    free_idx_.insert(free_idx_.end(), retire_.begin(), retire_.end());
    retire_.clear();
  }
  p->t = t_;
  // running samples are those active before admission
  for (int s = 0; s < B_; ++s)
    if (slot_of_[s] >= 0) p->running.push_back(slot_of_[s]);
  // refill, strict longest-first
  while (active_ < B_ && qhead_ < queue_.size()) {
    const int32_t i = queue_[qhead_];
    Sample& s = samples_[i];
    const bool first = s.group >= 0 && groups_[s.group].pages.empty();
    const int64_t R = reservation(s, page_) + (first ? ((int64_t)s.P + page_ - 1) / page_ : 0);
    if (reserved_ + R > pages_.capacity()) break;
    int slot = 0;
    while (slot_of_[slot] >= 0) ++slot;
    slot_of_[slot] = i;
    s.slot = slot;
    s.admit_iter = t_;
    reserved_ += R;
    ++active_;
    ++qhead_;
    p->admitted.push_back(i);
    auto alloc = [&]() {
      const int64_t pg = pages_.alloc();
      if (pg < 0) throw std::runtime_error("page pool exhausted (reservation invariant broken)");
      p->alloc_log.push_back((int32_t)pg);
      return (int32_t)pg;
    };
    if (s.group >= 0) {
      Group& g = groups_[s.group];
      if (first)
        for (int k = 0; k < (s.P + page_ - 1) / page_; ++k) g.pages.push_back(alloc());
      const int n_sh = (int)shared_pages(s, page_);
      for (int k = 0; k < n_sh; ++k) {
        s.pages.push_back(g.pages[k]);
        p->bt_deltas.insert(p->bt_deltas.end(), {slot, k, g.pages[k]});
      }
      const int32_t own = alloc();  // private copy of the page holding position P-1
      s.pages.push_back(own);
      p->bt_deltas.insert(p->bt_deltas.end(), {slot, n_sh, own});
      s.group_first = first;
      if (first) {
        p->copies_after_prefill.insert(p->copies_after_prefill.end(), {own, g.pages[n_sh]});
      } else {
        p->copies_before_decode.insert(p->copies_before_decode.end(), {g.pages[n_sh], own});
        p->admitted_decode.push_back(i);
      }
    } else {
      const int np = (s.P + page_ - 1) / page_;
      for (int k = 0; k < np; ++k) {
        const int32_t pg = alloc();
        s.pages.push_back(pg);
        p->bt_deltas.insert(p->bt_deltas.end(), {slot, k, pg});
      }
    }
  }
  if (active_ == 0) throw std::runtime_error("queue head can never fit the page pool");
  // running samples feed token j at position P + j - 1 (ascending slot)
  int64_t sumctx = 0;
  for (int32_t i : p->running) {
    Sample& s = samples_[i];
    const int64_t pos = (int64_t)s.P + s.produced - 1;
    if (pos == (int64_t)s.pages.size() * page_) {
      const int64_t pg = pages_.alloc();
      if (pg < 0) throw std::runtime_error("page pool exhausted (reservation invariant broken)");
      p->bt_deltas.insert(p->bt_deltas.end(), {s.slot, (int32_t)s.pages.size(), (int32_t)pg});
      s.pages.push_back((int32_t)pg);
      p->alloc_log.push_back((int32_t)pg);
    }
    sumctx += pos + 1;
  }
  for (int32_t i : p->admitted) sumctx += samples_[i].P;
  p->sumctx = sumctx;
  p->b = active_;
  // every active sample produces one token; completions ascending id
  for (int s = 0; s < B_; ++s) {
    const int32_t i = slot_of_[s];
    if (i < 0) continue;
    Sample& x = samples_[i];
    if (++x.produced == x.d) p->completed.push_back(i);
  }
  std::sort(p->completed.begin(), p->completed.end(),
            [&](int32_t a, int32_t b) { return samples_[a].id < samples_[b].id; });
  for (int32_t i : p->completed) {
    Sample& s = samples_[i];
    s.finish_iter = t_;
    for (size_t k = (size_t)shared_pages(s, page_); k < s.pages.size(); ++k) {  // its own pages
      pages_.free(s.pages[k]);
      p->free_log.push_back(s.pages[k]);
    }
    slot_of_[s.slot] = -1;
    reserved_ -= reservation(s, page_);
    if (s.group >= 0) {
      auto g = groups_.find(s.group);
      if (--g->second.remain == 0) {  // the group's last member: its prompt pages go back
        for (int32_t pg : g->second.pages) {
          pages_.free(pg);
          p->free_log.push_back(pg);
        }
        reserved_ -= ((int64_t)s.P + page_ - 1) / page_;
        groups_.erase(g);
      }
    }
    --active_;
    if (!tracing) retire_.push_back(i);
  }
  if (tracing) {
    auto& o = trace_iters;
    o.push_back(t_);
    o.push_back(p->b);
    o.push_back(p->sumctx);
    o.push_back((int64_t)p->admitted.size());
    o.push_back((int64_t)p->completed.size());
    o.push_back((int64_t)p->alloc_log.size());
    o.push_back((int64_t)p->free_log.size());
    for (int32_t i : p->admitted) o.push_back((int64_t)samples_[i].id);
    for (int32_t i : p->completed) o.push_back((int64_t)samples_[i].id);
    for (int32_t pg : p->alloc_log) o.push_back(pg);
    for (int32_t pg : p->free_log) o.push_back(pg);
  }
  ++t_;
  return true;
}

void Scheduler::sample_trace(std::vector<int64_t>* out) const {
  std::vector<int32_t> idx;
  for (int32_t i = 0; i < (int32_t)samples_.size(); ++i)
    if (samples_[i].admit_iter >= 0) idx.push_back(i);
  std::sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return samples_[a].id < samples_[b].id; });
  for (int32_t i : idx) {
    const Sample& s = samples_[i];
    out->push_back((int64_t)s.id);
    out->push_back(s.slot);
    out->push_back(s.admit_iter);
    out->push_back(s.finish_iter);
    out->push_back((int64_t)s.pages.size());
    for (int32_t pg : s.pages) out->push_back(pg);
  }
}

// ------------------------------------------------------------------ Alg. 2
// T(b) in picoseconds from the integer profile (appendix, continuity P:49).
static __int128 tb_ps(const DispatchCfg& c, int64_t b) {
  const __int128 base = (__int128)c.t0_ns * 1000;
  if (b < c.b_star) return base + (__int128)c.k0_ps * b;
  return base + (__int128)c.k0_ps * c.b_star + (__int128)c.k1_ps * (b - c.b_star);
}

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Eq. 2: PTL(BS) * L * ceil(M / BS), BS memory-capped.
static __int128 eq2(const DispatchCfg& c, int64_t members, int64_t L, int64_t instances, int64_t pbar) {
  if (members <= 0) return 0;
  const int64_t M = cdiv(members, instances);
  const int64_t by_mem = c.pool_pages / cdiv(pbar + L - 1, c.page);
  int64_t bs = std::min<int64_t>({M, (int64_t)c.B, by_mem});
  if (bs < 1) bs = 1;
  return tb_ps(c, bs) * L * cdiv(M, bs);
}

// nearest-rank percentile (ceil(q n)-th order statistic)
static int64_t pct(std::vector<int64_t> v, int q) {
  const int64_t n = (int64_t)v.size();
  int64_t k = cdiv((int64_t)q * n, 100);
  if (k < 1) k = 1;
  std::nth_element(v.begin(), v.begin() + (k - 1), v.end());
  return v[k - 1];
}

int dispatch_alg2(const DispatchCfg& c, int n, const uint64_t* ids, const int32_t* P, const int32_t* hint,
                  int32_t* instance) {
  if (n <= 0) return 0;
  std::vector<int32_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  if (c.policy == 2) {
    // "prompts are typically assigned randomly": seeded permutation, round robin
    uint64_t s = c.seed ? c.seed : 1;
    for (int i = n - 1; i > 0; --i) {
      s ^= s << 13, s ^= s >> 7, s ^= s << 17;
      std::swap(order[i], order[(int)(s % (uint64_t)(i + 1))]);
    }
    for (int j = 0; j < n; ++j) instance[order[j]] = j % c.N;
    return 0;
  }
  // Sort(P, L, descending), ties by id
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    if (hint[a] != hint[b]) return hint[a] > hint[b];
    return ids[a] < ids[b];
  });
  if (c.policy == 1 || c.N == 1) {
    for (int j = 0; j < n; ++j) instance[order[j]] = j % c.N;
    return 0;
  }
  int64_t n_tail = c.tail_ceil ? cdiv((int64_t)c.alpha_pct * n, 100) : ((int64_t)c.alpha_pct * n) / 100;
  n_tail = std::min<int64_t>(n_tail, n);
  const int64_t n_reg = n - n_tail;
  std::vector<int64_t> D(hint, hint + n);
  const int64_t L_alpha = pct(D, 90), L_r = pct(D, 50);
  int64_t sumP = 0;
  for (int i = 0; i < n; ++i) sumP += P[i];
  const int64_t pbar = cdiv(sumP, n);
  int n_l;
  if (n_tail == 0) {
    n_l = 0;
  } else if (n_reg == 0) {
    n_l = c.N;
  } else {
    __int128 best = 0;
    n_l = -1;
    for (int nl = 1; nl < c.N; ++nl) {
      const __int128 a = eq2(c, n_tail, L_alpha, nl, pbar);
      const __int128 r = eq2(c, n_reg, L_r, c.N - nl, pbar);
      const __int128 tot = c.score_max ? (a > r ? a : r) : a + r;
      if (n_l < 0 || tot < best) best = tot, n_l = nl;
    }
  }
  for (int j = 0; j < n; ++j) {
    const int32_t i = order[j];
    if (n_l == c.N || (n_l > 0 && j < n_tail))
      instance[i] = j % n_l;
    else {
      const int64_t jr = n_l == 0 ? j : j - n_tail;
      instance[i] = n_l + (int32_t)(jr % (c.N - n_l));
    }
  }
  return n_l;
}

// ------------------------------------------------------------------ elastic DP (NEXT-4)
__int128 predicted_generation_ps(const DispatchCfg& c, int n, const uint64_t* ids, const int32_t* P,
                                 const int32_t* hint) {
  std::vector<int32_t> inst(n, 0);
  dispatch_alg2(c, n, ids, P, hint, inst.data());
  __int128 makespan = 0;
  for (int k = 0; k < c.N; ++k) {
    std::vector<Sample> mine;
    for (int i = 0; i < n; ++i) {
      if (inst[i] != k) continue;
      Sample s;
      s.id = ids[i], s.P = P[i], s.d = hint[i], s.hint = hint[i], s.batch = 0;  // the hint as the length
      mine.push_back(std::move(s));
    }
    if (mine.empty()) continue;
    Scheduler sch;
    sch.init(c.B, c.page, c.pool_pages);
    sch.submit(std::move(mine));
    IterPlan plan;
    __int128 t = 0;
    while (sch.plan(&plan)) {  // b = samples that ran in the iteration, sumctx = their cached tokens
      int64_t pf = 0;          // prompt tokens prefilled in it
      for (int32_t i : plan.admitted) {
        const Sample& a = sch.samples()[i];
        if (a.group < 0 || a.group_first) pf += a.P;  // later group members share the prefill (R26)
      }
      t += tb_ps(c, plan.b) + (__int128)c.kv_ps * plan.sumctx + (__int128)c.pf_ps * pf;
    }
    makespan = std::max(makespan, t);
  }
  return makespan;
}

// ------------------------------------------------------------------ NEXT-2 two-dimensional dispatch
TailPlan tp_tail_plan(const DispatchCfg& c_dp, const DispatchCfg& c_tp, int tp_size, int n, const uint64_t* ids,
                      const int32_t* P, const int32_t* hint) {
  std::vector<int32_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    if (hint[a] != hint[b]) return hint[a] > hint[b];
    return ids[a] < ids[b];
  });
  std::vector<uint64_t> sid(n);
  std::vector<int32_t> sP(n), sh(n);
  for (int j = 0; j < n; ++j) sid[j] = ids[order[j]], sP[j] = P[order[j]], sh[j] = hint[order[j]];
  DispatchCfg tp1 = c_tp;
  tp1.N = 1;
  // predicted times of the split at k (the sorted prefix [0, k) to the TP instance)
  auto times = [&](int k, __int128* t_tp, __int128* t_dp) {
    *t_tp = k > 0 ? predicted_generation_ps(tp1, k, sid.data(), sP.data(), sh.data()) : 0;
    *t_dp = k < n ? predicted_generation_ps(c_dp, n - k, sid.data() + k, sP.data() + k, sh.data() + k) : 0;
  };
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    __int128 a, b;
    times(mid, &a, &b);
    if (a >= b)
      hi = mid;
    else
      lo = mid + 1;
  }
  TailPlan out;
  __int128 a, b;
  times(lo, &a, &b);
  out.n_tail = lo, out.t_tp = a, out.t_dp = b;
  if (lo > 0) {
    __int128 a2, b2;
    times(lo - 1, &a2, &b2);
    if (std::max(a2, b2) <= std::max(a, b)) out.n_tail = lo - 1, out.t_tp = a2, out.t_dp = b2;
  }
  DispatchCfg all = c_dp;
  all.N = c_dp.N + tp_size;
  out.t_all = n > 0 ? predicted_generation_ps(all, n, ids, P, hint) : 0;
  return out;
}

// ------------------------------------------------------------------ T(b) fit
// Least squares on the hinge basis [1, b, (b - b*)+] for every measured b* with
// >= 2 distinct points at or below and >= 1 above; minimum SSE wins, ties ->
// smaller b*.  3x3 normal equations solved by Cramer's rule.
static double det3(const double m[3][3]) {
  return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
         m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

bool fit_tb(int n, const double* b, const double* T, double out[5], int64_t* b_star, int64_t prof[4]) {
  std::vector<double> xs(b, b + n);
  std::sort(xs.begin(), xs.end());
  xs.erase(std::unique(xs.begin(), xs.end()), xs.end());
  bool have = false;
  double best_sse = 0, bt0 = 0, bk0 = 0, bdk = 0, bbs = 0;
  for (size_t ci = 0; ci < xs.size(); ++ci) {
    const double bs = xs[ci];
    const size_t left = ci + 1, right = xs.size() - ci - 1;
    if (left < 2 || right < 1) continue;
    double G[3][3] = {{0}}, r[3] = {0};
    for (int i = 0; i < n; ++i) {
      const double f[3] = {1.0, b[i], b[i] > bs ? b[i] - bs : 0.0};
      for (int a = 0; a < 3; ++a) {
        r[a] += f[a] * T[i];
        for (int c = 0; c < 3; ++c) G[a][c] += f[a] * f[c];
      }
    }
    const double D = det3(G);
    if (std::fabs(D) < 1e-300) continue;
    double beta[3];
    for (int k = 0; k < 3; ++k) {
      double Mk[3][3];
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) Mk[a][c] = c == k ? r[a] : G[a][c];
      beta[k] = det3(Mk) / D;
    }
    double sse = 0;
    for (int i = 0; i < n; ++i) {
      const double e = T[i] - beta[0] - beta[1] * b[i] - beta[2] * (b[i] > bs ? b[i] - bs : 0.0);
      sse += e * e;
    }
    if (!have || sse < best_sse) {
      have = true;
      best_sse = sse, bt0 = beta[0], bk0 = beta[1], bdk = beta[2], bbs = bs;
    }
  }
  if (!have) return false;
  const double k1 = bk0 + bdk;
  out[0] = bt0, out[1] = bk0, out[2] = k1, out[3] = bt0 + (bk0 - k1) * bbs, out[4] = best_sse;
  *b_star = (int64_t)bbs;
  prof[0] = std::llround(bt0), prof[1] = std::llround(bk0 * 1000.0), prof[2] = (int64_t)bbs,
  prof[3] = std::llround(k1 * 1000.0);
  return true;
}

}  // namespace sgs
