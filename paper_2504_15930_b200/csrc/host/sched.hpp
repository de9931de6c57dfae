// Host-side control plane of one generation instance: paged-KV page
// allocator, longest-first continuous-batching scheduler, Alg. 2 dispatcher
// and the T(b) fit.  Pure C++ (no CUDA); the engine consumes IterPlan.
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

namespace sgs {

// ------------------------------------------------------------------ pages
// Lowest-free-index page allocator over a two-level bitmap (R4).
class PageAllocator {
 public:
  void reset(int64_t n_pages);
  int64_t alloc();  // -1 when empty
  void free(int64_t p);
  int64_t n_free() const { return n_free_; }
  int64_t capacity() const { return n_; }

 private:
  int64_t n_ = 0, n_free_ = 0;
  std::vector<uint64_t> words_;    // bit = 1: page free
  std::vector<uint64_t> summary_;  // bit = 1: word has a free page
};

// ------------------------------------------------------------------ samples
struct Sample {
  uint64_t id;
  int32_t P, d, hint;
  int32_t batch;
  std::vector<int32_t> prompt;  // prompt tokens; released once the prefill metadata is staged
  int64_t group = -1;           // NEXT-3 prefix-sharing group (identical prompts of one batch), -1: none
  bool group_first = false;     // the group's first admitted member (runs the group's prefill)
  // runtime
  int32_t slot = -1;
  int32_t produced = 0;
  int64_t admit_iter = -1, finish_iter = -1;
  std::vector<int32_t> pages;
};

struct IterPlan {
  int64_t t = 0;
  std::vector<int32_t> admitted;         // sample indices, admission order
  std::vector<int32_t> running;          // sample indices decoding this iteration, ascending slot
  std::vector<int32_t> completed;        // sample indices, ascending id
  std::vector<int32_t> bt_deltas;        // (slot, page_idx, page) triples in allocation order
  std::vector<int32_t> alloc_log, free_log;
  // prefix sharing (R26): admitted non-first group members, which produce their
  // first token as a decode row at position P-1 (their prompt KV is shared);
  // page copies (src, dst): a first member's private copy of the page holding
  // P-1 -> the group's page after the prefill, the group's page -> a later
  // member's private copy before the decode program
  std::vector<int32_t> admitted_decode;
  std::vector<int32_t> copies_after_prefill, copies_before_decode;
  int64_t sumctx = 0;
  int32_t b = 0;
};

class Scheduler {
 public:
  void init(int max_batch, int page, int64_t n_pages);
  // Append one RL batch (already restricted to this instance).
  void submit(std::vector<Sample>&& batch);
  bool idle() const { return active_ == 0 && qhead_ == queue_.size(); }
  // Build the next iteration; returns false when idle (no iteration counted).
  bool plan(IterPlan* p);
  int64_t iterations() const { return t_; }
  int64_t queued() const { return (int64_t)(queue_.size() - qhead_); }
  int32_t active() const { return active_; }
  std::vector<Sample>& samples() { return samples_; }
  const std::vector<Sample>& samples() const { return samples_; }
  int page() const { return page_; }
  int64_t pool_pages() const { return pages_.capacity(); }
  // trace (DESIGN.md §5 format).  Without tracing the host state is bounded
  // by the samples in flight: completed sample records are recycled (one
  // iteration after their completion, so the engine can still read them while
  // it stages that iteration) and the consumed queue prefix is dropped.
  std::vector<int64_t> trace_iters;
  bool tracing = false;
  void sample_trace(std::vector<int64_t>* out) const;
  size_t records() const { return samples_.size(); }
  int64_t queue_entries() const { return (int64_t)queue_.size(); }

 private:
  int B_ = 0, page_ = 16;
  PageAllocator pages_;
  std::vector<Sample> samples_;   // all samples ever submitted (index = handle-local)
  std::vector<int32_t> queue_;    // sample indices in admission order (FIFO by batch, LF within)
  size_t qhead_ = 0;
  std::vector<int32_t> slot_of_;  // slot -> sample index or -1
  std::vector<int32_t> free_idx_, retire_;  // recyclable sample records (tracing off)
  struct Group {
    std::vector<int32_t> pages;  // the prompt's ceil(P/page) pages (allocated at the first admission)
    int remain = 0;              // members not yet completed
  };
  std::unordered_map<int64_t, Group> groups_;
  int64_t reserved_ = 0;
  int32_t active_ = 0;
  int64_t t_ = 0;
};

// ------------------------------------------------------------------ dispatch (Alg. 2)
struct DispatchCfg {
  int N, B, page;
  int64_t pool_pages;
  int64_t t0_ns, k0_ps, b_star, k1_ps;
  int alpha_pct, score_max, tail_ceil, policy;  // policy: 0 skew, 1 round robin, 2 random
  uint64_t seed;
  // predictions only (R27): ps per cached context token per iteration added to
  // T(b) (the KV stream of the decode attention); 0 = the paper's T(b) alone
  int64_t kv_ps = 0;
  int64_t pf_ps = 0;  // predictions only: ps per prompt token prefilled in the iteration
};
// instance[i] for each sample i; returns N_l.
int dispatch_alg2(const DispatchCfg& c, int n, const uint64_t* ids, const int32_t* P, const int32_t* hint,
                  int32_t* instance);

// ------------------------------------------------------------------ elastic DP (NEXT-4)
// Predicted generation time (ps) of a batch on c.N instances: Alg. 2, then
// each instance's longest-first schedule on the hints as lengths (the same
// Scheduler the engine runs), summing T(b_t) of the integer profile; the
// makespan over instances (R25).
__int128 predicted_generation_ps(const DispatchCfg& c, int n, const uint64_t* ids, const int32_t* P,
                                 const int32_t* hint);

// ------------------------------------------------------------------ NEXT-2 two-dimensional dispatch
// The longest k samples (hint descending, id ascending -- the long tail the
// ranker identifies) go to one tensor-parallel instance, the rest to the DP
// instances with c_dp's policy (R27):
//   T_tp(k) = predicted_generation_ps(c_tp [N = 1], top k),  T_dp(k) = that of c_dp, the rest,
// k = the smallest k with T_tp(k) >= T_dp(k) (binary search over [0, n]) or
// k - 1, whichever has the smaller max(T_tp, T_dp) (ties: the smaller k);
// t_all = all samples on c_dp.N + tp_size DP instances.  Returns k.
struct TailPlan {
  int n_tail = 0;
  __int128 t_tp = 0, t_dp = 0, t_all = 0;
};
TailPlan tp_tail_plan(const DispatchCfg& c_dp, const DispatchCfg& c_tp, int tp_size, int n, const uint64_t* ids,
                      const int32_t* P, const int32_t* hint);

// ------------------------------------------------------------------ T(b) fit
bool fit_tb(int n, const double* b, const double* T_ns, double out[5], int64_t* b_star, int64_t prof[4]);

}  // namespace sgs
