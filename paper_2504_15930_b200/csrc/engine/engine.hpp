// One generation instance: device arena (weights | KV pool | scratch), the
// host scheduler, and the per-iteration device program (prefill of admitted
// prompts + one decode step of the running samples).
#pragma once
#include <cuda_runtime.h>

#include <deque>
#include <map>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../../include/sgs.h"
#include "../host/sched.hpp"
#include "../kernels/kernels.h"

namespace sgs {

struct TensorRef {
  int64_t id;
  void* ptr;
  int64_t n;
  int is_norm;
  int64_t cols = 1;  // row-block placement (interleaved gate/up): blk rows every stride rows at off
  int blk = 0, stride = 0, off = 0;
  ShardMap shard{};  // tensor-parallel window of the full tensor (NEXT-2)
  int tiled = 0;     // GEMM weight in the tiled layout (kernels.h weight placement)
};

struct ArenaLayout {
  int64_t weights_bytes = 0, kv_bytes = 0, scratch_bytes = 0, total = 0, kv_page_bytes = 0;
  // offsets (bytes from arena start)
  int64_t off_kv = 0, off_h = 0, off_x = 0, off_qkv = 0, off_q = 0, off_kc = 0, off_vc = 0, off_ao = 0,
          off_gu = 0, off_mm = 0, off_logits = 0, off_rope = 0, off_bt = 0, off_last = 0, off_hist = 0,
          off_meta = 0, off_attn = 0, off_cksum = 0, off_shadow = -1, off_amax = 0, off_nbar = 0;
  // decode scratch (Bpad rows), separate from the prefill scratch so the two run concurrently
  int64_t off_dh = 0, off_dx = 0, off_dqkv = 0, off_dq = 0, off_dao = 0, off_dgu = 0, off_dmm = 0;
  int64_t meta_bytes = 0, attn_bytes = 0, meta_dec_bytes = 0;
  int tmax = 0, max_pages = 0, max_items = 0;
};

struct Completion {
  uint64_t id;
  int32_t slot;
  int64_t admit_iter, finish_iter;
  int32_t version;
  std::vector<int32_t> tokens;
};

class Engine {
 public:
  ~Engine();
  sgs_status init(const sgs_model_cfg& m, const sgs_engine_cfg& e, const sgs_weights* w);
  sgs_status submit(const sgs_prompt* prompts, int32_t n, const int32_t* hint, const int32_t* forced,
                    int32_t* n_mine);
  sgs_status step(sgs_completion* out, int32_t cap, int32_t* n_out);
  sgs_status load_weights_seed(uint64_t seed);
  sgs_status set_instances(int32_t n_instances, int32_t instance_rank);
  sgs_status checksum(int64_t tensor_id, uint64_t* out);
  sgs_status comm_init(const uint8_t id[128], int rank, int world);
  sgs_status tp_comm_init(const uint8_t id[128]);
  sgs_status update_weights(const sgs_weights* src, int root);
  sgs_status load_weights(const sgs_weights* w, uint8_t* base, cudaStream_t st);
  sgs_status stage_weights(const sgs_weights* src);
  // asynchronous weight sync (SGS_F_SHADOW_WEIGHTS): shadow buffer, side stream
  sgs_status shadow_weights(void** ptr, int64_t* bytes);
  sgs_status stage_weights_seed(uint64_t seed);
  sgs_status update_weights_begin(int root);
  sgs_status update_weights_ready(int32_t* ready);
  sgs_status update_weights_commit();
  sgs_status debug_head(const float* h_in, int32_t T, float* logits);
  sgs_status last_logits(float* logits, uint64_t* ids, int32_t* tok_idx, int32_t cap, int32_t* rows);
  sgs_status debug_forward(const int32_t* tokens, int32_t T, float* dump, int layer = -1,
                           const float* h_in = nullptr);

  static sgs_status layout(const sgs_model_cfg& m, const sgs_engine_cfg& e, int64_t n_pages, ArenaLayout* L);

  std::string err;
  bool poisoned = false;
  Scheduler sched;
  float last_ms = 0.f;
  // kernel-class timing (SGS_F_KERNEL_TIMING) and I/O accounting
  // classes: 0 decode attention, 1 decode GEMMs, 2 prefill attention, 3 device
  // time of the sampled iterations, 4 prefill GEMMs, 5 other decode kernels
  // (RMSNorm, RoPE + KV append, embedding, sampler)
  // (index cls + kClasses * phase; phase 0 every sampled iteration, 1 those
  // with >= 129 decode rows, 2 those with 1..32)
  static constexpr int kClasses = 6, kPhases = 3;
  double kstat_ms[kClasses * kPhases] = {0}, kstat_bytes[kClasses * kPhases] = {0},
         kstat_flops[kClasses * kPhases] = {0};
  int64_t kstat_n[kClasses * kPhases] = {0};
  int64_t h2d_bytes = 0, d2h_bytes = 0;
  // per-iteration log (T(b) profiling, a16): t, b, admitted, prefill tokens, sum ctx, device us
  std::vector<int64_t> iter_log;
  // roofline time of the timed launches: sum_k max(bytes_k / BW, flops_k / F) (sgs_set_roofline)
  double roof_bw_gbs = 0, roof_tflops = 0, kstat_roof_ms[kClasses * kPhases] = {0};
  int cur_phase_ = 0;
  int64_t launches = 0;
  int32_t version = 0;

 private:
  sgs_status cuda_fail(cudaError_t e, const char* what);
  sgs_status run_iteration(const IterPlan& plan);
  sgs_status prefill_chunk(const std::vector<int32_t>& idx, int row_base, const int32_t* d_tokens,
                           const int32_t* d_pos, const int32_t* d_slot, const int32_t* d_offs,
                           const int32_t* d_qblocks, int n_qblocks, const int32_t* d_last_rows,
                           const int32_t* d_pf_slot, const int32_t* d_pf_tok, int T, float* dump = nullptr,
                           int only_layer = -1, const float* h_in = nullptr);
  cudaError_t gemm(const void* W, const void* X, float* C, int N, int K, int T, bool accumulate,
                   const PreNorm* pn = nullptr);
  cudaError_t gate_up(const void* W, int T, const PreNorm* pn = nullptr);
  cudaError_t sample(const float* logits, int rows, const uint32_t* sid, const int32_t* slot, const int32_t* tok_idx);
  void build_tensor_table();
  // kernel-class timing record: bytes = bfix + brow * rows (bfix < 0: the
  // iteration's decode-attention bytes/flops), flops = frow * rows
  struct KRec {
    int cls;
    cudaEvent_t a, b;
    double bfix, brow, frow;
    int rows;  // -1: the decode rows of the flush (graph records)
  };
  std::vector<cudaEvent_t> ev_pool_;
  size_t ev_used_ = 0;
  std::vector<KRec> krec_;
  cudaEvent_t next_event();
  void ktic(KRec* r, int cls);
  void ktoc(KRec* r, double bfix, double brow, double frow, int rows);
  cudaError_t kflush(const std::vector<KRec>& recs, int rows);
  // decode iteration as a CUDA graph per 16-row bucket (fixed pointers, device-side work counts)
  struct DecodeGraph {
    cudaGraphExec_t exec = nullptr;
    int uses = 0;
    int64_t kernels = 0;
    std::vector<KRec> recs;
  };
  std::vector<DecodeGraph> graphs_[2];  // [timed]: variant with event-record nodes
  // prefill chunks as CUDA graphs keyed by their metadata shape (row base,
  // offset, prompt lengths): refills of equal-length prompts replay one graph
  // instead of ~8 eager launches per layer (untimed iterations only)
  std::map<std::vector<int64_t>, DecodeGraph> pgraphs_;
  bool timing_now_ = false;             // this iteration is a timing sample
  int skip_ = 0;                        // SGS_DEBUG_SKIP ablation mask (decode program)
  int64_t timing_iter_ = 0;
  // about 1 in 64 iterations carries the per-kernel events, chosen by a hash of
  // the iteration counter (a fixed stride would alias with the schedule: every
  // config-2 batch has a multiple of 32 iterations, so t = 0 would always be sampled)
  static constexpr int kTimingStride = 64;
  int gemm_cls_ = 1;  // 1 while the decode program is issued, 4 in prefill chunks
  std::vector<KRec>* rec_target_ = nullptr;  // non-null while capturing
  double cur_attn_bytes_ = 0, cur_attn_flops_ = 0;
  double cur_pf_attn_flops_ = 0;  // causal attention flops of the prefill chunk being issued
  sgs_status decode_body(int Bk);
  sgs_status run_decode(int b);
  sgs_status run_decode_body(int b);

  sgs_model_cfg m_{};
  sgs_engine_cfg e_{};
  bool null_ = true;
  cudaStream_t st_ = nullptr;
  ArenaLayout L_{};
  uint8_t* arena_ = nullptr;
  int64_t n_pages_ = 0;
  int max_gen_ = 0;
  // weights
  struct Layer {
    void *wqkv, *bqkv, *wo, *wgu, *wd, *n1, *n2;
    void* kv;
  };
  std::vector<Layer> layers_;
  void *embed_ = nullptr, *lm_head_ = nullptr, *nf_ = nullptr;
  std::vector<TensorRef> tensors_;
  // scratch
  float *h_ = nullptr, *qkv_ = nullptr, *gu_ = nullptr, *logits_ = nullptr, *rope_ = nullptr;
  // the decode scratch set, swapped into h_/x_/qkv_/q_/ao_/gu_/mm_ while the decode program is built
  struct ScratchSet {
    float *h, *qkv, *gu;
    void *x, *q, *ao, *mm;
  } dset_{};
  void swap_scratch();
  cudaStream_t st_pf_ = nullptr;                     // prefill chunks, concurrent with the decode graph
  cudaEvent_t ev_meta_ = nullptr, ev_pf_ = nullptr;  // metadata ready / prefill done
  void *x_ = nullptr, *q_ = nullptr, *kc_ = nullptr, *vc_ = nullptr, *ao_ = nullptr, *mm_ = nullptr;
  int32_t *bt_ = nullptr, *last_tok_ = nullptr, *hist_ = nullptr;
  uint8_t* meta_dev_ = nullptr;
  uint8_t* meta_host_ = nullptr;  // pinned (the current one of meta_bufs_)
  uint8_t* attn_ws_ = nullptr;
  unsigned long long* cksum_dev_ = nullptr;
  unsigned long long* amax_keys_ = nullptr;  // fused greedy sampling (GEMM mode 4): [Bpad] keys + counter
  unsigned int* norm_bar_ = nullptr;          // PreNorm grid barriers: 2 per site (2 per layer + final)
  bool fused_norm_ = false;                   // RMSNorm fused into the decode GEMMs (SGS_FUSED_NORM=1)
  int64_t dec_launch_ = 0;                    // decode-program launches (PreNorm barrier parity)
  int qblk_ = 64;                             // prefill attention query block (128: tcgen05 kernel)
  int w_tiled_ = 0;                           // GEMM weights tiled [N/128][K/64][128][64] (SGS_WEIGHT_LAYOUT)
  // NEXT-2 tensor parallelism: m_ holds this shard's dims (q/kv heads, FFN, vocab
  // rows divided by tp_); the embedding table is the full vocabulary
  int tp_ = 1, tp_rank_ = 0;
  int64_t vocab_full_ = 0;
  void* tp_comm_ = nullptr;
  unsigned long long* amax_keys_pf_ = nullptr;  // prefill rows' argmax keys (TP)
  cudaError_t tp_allreduce_sum(float* x, size_t n);
  cudaError_t tp_allreduce_max_u64(unsigned long long* x, size_t n);
  // decode-program exchange over NVLink peer memory (tp_comm.cu; NCCL when off)
  sgs_status tp_p2p_init();
  bool tp_p2p_ = false;
  uint8_t* xch_ = nullptr;
  std::vector<void*> xch_peer_;
  TpPeers tpp_{};
  int xch_rows_ = 0;
  int32_t* tok_host_ = nullptr;  // pinned, completed tokens (the current one of tok_bufs_)
  int64_t tok_host_cap_ = 0;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  // Host/device pipelining: iteration i+1 is planned and launched before
  // iteration i is waited for, so the GPU never idles on host work; each
  // in-flight iteration owns one of two pinned staging/token buffers and event
  // pairs.  Off with SGS_F_KEEP_LOGITS and on kernel-timing samples.
  struct Inflight {
    int buf = 0;
    int64_t t = 0, b = 0, adm = 0, pf_tok = 0, sumctx = 0;
    int n_run = 0;
    bool timing = false;
    std::vector<Completion> comps;  // tokens filled when finalized
    std::vector<int64_t> toff;
  };
  std::deque<Inflight> infl_;
  uint8_t* meta_bufs_[2] = {nullptr, nullptr};
  int32_t* tok_bufs_[2] = {nullptr, nullptr};
  cudaEvent_t ev0s_[2] = {nullptr, nullptr}, ev1s_[2] = {nullptr, nullptr};
  int cur_buf_ = 0;
  sgs_status finalize_front();
 public:
  sgs_status drain();  // finalize every in-flight iteration (before weight updates, debug calls, ...)
  int n_layers() const { return m_.n_layers; }
  int64_t live_ids() const { return (int64_t)live_ids_.size(); }
  int64_t inflight_samples() const {
    int64_t n = 0;
    for (const auto& f : infl_) n += (int64_t)f.comps.size();
    return n;
  }
 private:
  uint8_t* shadow_ = nullptr;           // second weight buffer (SGS_F_SHADOW_WEIGHTS)
  cudaStream_t st_side_ = nullptr;      // weight staging + broadcast, concurrent with generation
  cudaEvent_t ev_sync_ = nullptr;       // end of the in-flight broadcast on st_side_
  cudaEvent_t ev_commit_ = nullptr;     // end of the last commit's shadow -> active copy (on st_)
  bool sync_pending_ = false;
  // prompts (host)
  std::unordered_set<uint64_t> live_ids_;  // ids queued or active (R22)
  int batch_counter_ = 0;
  std::deque<Completion> ready_;
  std::vector<Completion> handed_;  // storage for the completions returned by the last step
  // logits kept for tests
  std::vector<float> kept_logits_;
  std::vector<uint64_t> kept_ids_;
  std::vector<int32_t> kept_tok_;
  // nccl
  void* nccl_comm_ = nullptr;
  int nccl_rank_ = -1, nccl_world_ = 0;
};

}  // namespace sgs
