// ORACLE — test infrastructure only (see oracle.hpp).
//
// C2: the per-instance scheduler of the Stream Generation Service, simulated
// iteration by iteration.
//
//  * Longest-first order: "samples are assigned to the batch in descending
//    order of their estimated output lengths. Once a sample is completed, the
//    sample with the longest remaining output length is added to the batch"
//    (§5.3 Scheduling Order; also appendix steps 1-3).
//    Estimated length = the ranker hint; ties -> lower id (R2).
//  * Continuous batching under cap B (P:9); a sample occupies its
//    slot for exactly d iterations, prefill not differentiated.
//  * Memory cap: admission reserves ceil((P+d-1)/page) pages
//    (R3); strict order, no backfill.
//  * Paged KV: prompt pages at admission, one page on each
//    boundary crossing, lowest free index first (R4).
//  * Prefix sharing (NEXT-3; "prefix sharing to save key-value cache usage",
//    P:1005-1007), reading R26: the samples of a group (one prompt, several
//    samples -- GRPO) share the prompt's pages before the one holding its last
//    token.  The group's ceil(P/page) prompt pages are allocated (and
//    reserved) when its first member is admitted and freed (and released)
//    when its last member completes; a member's block table is the group's
//    floor((P-1)/page) leading pages followed by private pages: a copy of the
//    page holding position P-1 and its generation pages, so it reserves
//    ceil((P+d-1)/page) - floor((P-1)/page).
#include <algorithm>
#include <map>
#include <set>
#include <stdexcept>

#include "oracle.hpp"

namespace oracle {

__int128 T_ps(const Profile& p, int64_t b) {
  // Appendix equation; t1 from continuity k0 b* + t0 = k1 b* + t1.
  __int128 left = (__int128)p.t0_ns * 1000 + (__int128)p.k0_ps * b;
  if (b < p.b_star) return left;
  __int128 at_star = (__int128)p.t0_ns * 1000 + (__int128)p.k0_ps * p.b_star;
  return at_star + (__int128)p.k1_ps * (b - p.b_star);
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

SimResult sched_sim(const std::vector<SimSample>& s, int B, int page, int64_t pool_pages,
                    const Profile* prof) {
  SimResult r;
  const int n = (int)s.size();
  // queue order: batch FIFO, then hint descending, then id ascending
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    if (s[a].batch != s[b].batch) return s[a].batch < s[b].batch;
    if (s[a].hint != s[b].hint) return s[a].hint > s[b].hint;
    return s[a].id < s[b].id;
  });

  std::set<int64_t> free_pages;
  for (int64_t p = 0; p < pool_pages; ++p) free_pages.insert(p);
  // prefix groups: pages, members not yet completed
  std::map<int64_t, std::vector<int64_t>> gpages;
  std::map<int64_t, int> gremain;
  for (int i = 0; i < n; ++i)
    if (s[i].group >= 0) ++gremain[s[i].group];
  auto shared_pages = [&](int i) { return s[i].group >= 0 ? (int64_t)(s[i].P - 1) / page : 0; };
  auto own_reservation = [&](int i) { return ceil_div((int64_t)s[i].P + s[i].d - 1, page) - shared_pages(i); };
  std::vector<int> slot_of(B, -1);              // slot -> sample index
  std::vector<int> produced(n, 0), slot(n, -1);
  std::vector<int64_t> admit(n, -1), finish(n, -1);
  std::vector<std::vector<int64_t>> pages(n);
  int64_t reserved = 0;
  int active = 0;
  size_t qhead = 0;  // next position in `order`
  int done = 0;
  int64_t t = 0;

  auto alloc_page = [&](int i, std::vector<int64_t>& log) {
    if (free_pages.empty()) throw std::runtime_error("oracle: page pool exhausted");
    int64_t p = *free_pages.begin();
    free_pages.erase(free_pages.begin());
    pages[i].push_back(p);
    log.push_back(p);
  };

  int64_t horizon = 0;  // samples with arrival_after <= horizon are queued
  while (done < n) {
    // A sample is queued once `arrival_after` iterations have executed.  An
    // idle instance executes no iteration, so the next batch then arrives at
    // the next executed iteration (idle step calls do not count, R5).
    horizon = std::max(horizon, t);
    if (active == 0 && qhead < (size_t)n && s[order[qhead]].arrival_after > horizon)
      horizon = s[order[qhead]].arrival_after;
    std::vector<int64_t> adm, comp, alloc_log, free_log;
    int64_t pf_tokens = 0;  // prompt tokens prefilled this iteration (R27 predictions)
    std::vector<bool> is_new(n, false);
    // (ii) admission, strict longest-first, lowest free slot
    while (active < B && qhead < (size_t)n) {
      int h = order[qhead];
      if (s[h].arrival_after > horizon) break;
      const bool first = s[h].group >= 0 && gpages[s[h].group].empty();
      int64_t R = own_reservation(h) + (first ? ceil_div(s[h].P, page) : 0);
      if (reserved + R > pool_pages) break;
      int sl = 0;
      while (slot_of[sl] != -1) ++sl;
      slot_of[sl] = h;
      slot[h] = sl;
      reserved += R;
      admit[h] = t;
      is_new[h] = true;
      ++active;
      ++qhead;
      adm.push_back(s[h].id);
      if (first || s[h].group < 0) pf_tokens += s[h].P;
      if (s[h].group >= 0) {
        auto& gp = gpages[s[h].group];
        if (first) {  // the group's prompt pages
          for (int64_t k = 0; k < ceil_div(s[h].P, page); ++k) {
            if (free_pages.empty()) throw std::runtime_error("oracle: page pool exhausted");
            gp.push_back(*free_pages.begin());
            alloc_log.push_back(*free_pages.begin());
            free_pages.erase(free_pages.begin());
          }
        }
        for (int64_t k = 0; k < shared_pages(h); ++k) pages[h].push_back(gp[k]);  // shared leading pages
        alloc_page(h, alloc_log);  // private copy of the page holding position P-1
      } else {
        int64_t np = ceil_div(s[h].P, page);
        for (int64_t k = 0; k < np; ++k) alloc_page(h, alloc_log);
      }
    }
    if (active == 0) throw std::runtime_error("oracle: head sample does not fit the pool");
    // (iii) running samples feed token j at pos P+j-1, ascending slot order
    int64_t sumctx = 0;
    for (int sl = 0; sl < B; ++sl) {
      int i = slot_of[sl];
      if (i < 0) continue;
      if (is_new[i]) {
        sumctx += s[i].P;
        continue;
      }
      int64_t pos = (int64_t)s[i].P + produced[i] - 1;
      if (pos == (int64_t)pages[i].size() * page) alloc_page(i, alloc_log);
      sumctx += pos + 1;
    }
    // (iv) every active sample produces one token
    std::vector<int> fin;
    for (int sl = 0; sl < B; ++sl) {
      int i = slot_of[sl];
      if (i < 0) continue;
      produced[i] += 1;
      if (produced[i] == s[i].d) fin.push_back(i);
    }
    // (v) completions, ascending id; pages return to the pool
    std::sort(fin.begin(), fin.end(), [&](int a, int b) { return s[a].id < s[b].id; });
    for (int i : fin) {
      comp.push_back(s[i].id);
      finish[i] = t;
      for (size_t k = (size_t)shared_pages(i); k < pages[i].size(); ++k) {  // private pages
        free_pages.insert(pages[i][k]);
        free_log.push_back(pages[i][k]);
      }
      reserved -= own_reservation(i);
      if (s[i].group >= 0 && --gremain[s[i].group] == 0) {  // the group's last member: its prompt pages
        for (int64_t p : gpages[s[i].group]) {
          free_pages.insert(p);
          free_log.push_back(p);
        }
        reserved -= ceil_div(s[i].P, page);
        gpages.erase(s[i].group);
      }
      slot_of[slot[i]] = -1;
      --active;
      ++done;
    }
    if (prof)
      r.time_ps += T_ps(*prof, active + (int64_t)fin.size()) + (__int128)prof->kv_ps * sumctx +
                   (__int128)prof->pf_ps * pf_tokens;
    auto& o = r.iters;
    o.push_back(t);
    o.push_back(active + (int64_t)fin.size());
    o.push_back(sumctx);
    o.push_back((int64_t)adm.size());
    o.push_back((int64_t)comp.size());
    o.push_back((int64_t)alloc_log.size());
    o.push_back((int64_t)free_log.size());
    o.insert(o.end(), adm.begin(), adm.end());
    o.insert(o.end(), comp.begin(), comp.end());
    o.insert(o.end(), alloc_log.begin(), alloc_log.end());
    o.insert(o.end(), free_log.begin(), free_log.end());
    ++t;
  }
  r.n_iters = t;
  std::vector<int> by_id(n);
  for (int i = 0; i < n; ++i) by_id[i] = i;
  std::sort(by_id.begin(), by_id.end(), [&](int a, int b) { return s[a].id < s[b].id; });
  for (int i : by_id) {
    r.samples.push_back(s[i].id);
    r.samples.push_back(slot[i]);
    r.samples.push_back(admit[i]);
    r.samples.push_back(finish[i]);
    r.samples.push_back((int64_t)pages[i].size());
    r.samples.insert(r.samples.end(), pages[i].begin(), pages[i].end());
  }
  return r;
}

}  // namespace oracle
