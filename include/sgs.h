/*
 * sgs.h — C-ABI of the B200-native Stream Generation Service hot path
 * (StreamRL, arXiv 2504.15930; PAPER.md = the paper's text, cited P:<line>).
 *
 * SGS exposes update(weights) and generate(prompts) (§3) and
 * returns each completed sample "in a stream fashion".
 * Prompts arrive with ranker-estimated output lengths;
 * output lengths are forced for evaluation.
 *
 * Conventions (all entry points):
 *  - Every call returns an sgs_status; the message is in sgs_last_error().
 *  - Inputs are caller-owned and copied before return.  Pointers documented
 *    "device" are CUDA device pointers on the handle's device; "host" pointers
 *    are ordinary (or pinned) host memory.
 *  - A handle is single-threaded.  One handle = one generation instance =
 *    one GPU (data-parallel instances are "entirely independent").
 *  - After a CUDA or NCCL error the handle is poisoned: later calls return
 *    SGS_E_STATE.
 *  - Device memory comes from the caller (PyTorch) as one arena; the library
 *    never calls cudaMalloc after sgs_init.
 *  - device < 0 selects "null-device" mode: the host scheduler, allocator and
 *    dispatcher run and trace exactly as on the GPU, no kernel is launched and
 *    every generated token is 0 (CPU parity of the schedule).
 */
#ifndef SGS_H_
#define SGS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sgs_handle sgs_handle;

typedef enum {
  SGS_OK = 0,
  SGS_E_INVAL = -1,       /* bad argument; the call had no effect */
  SGS_E_NOMEM = -2,       /* arena too small */
  SGS_E_STATE = -3,       /* wrong state (poisoned handle, update while busy, no comm) */
  SGS_E_CAPACITY = -4,    /* a sample can never fit (pages > pool or P+d-1 > max_ctx) */
  SGS_E_CUDA = -5,
  SGS_E_NCCL = -6,
  SGS_E_UNSUPPORTED = -7  /* shape not supported by the sm_100a kernels */
} sgs_status;

/* Model shape (Table 2; fields the paper omits follow Qwen2.5). */
typedef struct {
  int32_t n_layers, d_model, n_q_heads, n_kv_heads, head_dim, d_ffn, vocab;
  float rms_eps;      /* 1e-6 */
  double rope_theta;  /* 1e6, NeoX rotate-half */
} sgs_model_cfg;

/* Integer T(b) profile (appendix): T(b)[ps] = t0_ns*1000 + k0_ps*b
 * for b < b_star, continued with slope k1_ps above (t1 from continuity P:49). */
typedef struct {
  int64_t t0_ns, k0_ps, b_star, k1_ps;
} sgs_tb_profile;

enum { SGS_DISPATCH_SKEW = 0, SGS_DISPATCH_ROUND_ROBIN = 1, SGS_DISPATCH_RANDOM = 2 };
enum { SGS_SCORE_SUM = 0, SGS_SCORE_MAX = 1 };
enum { SGS_SAMPLE_GREEDY = 0, SGS_SAMPLE_TOP_P = 1 };
enum {
  SGS_F_KEEP_LOGITS = 1,     /* keep fp32 logits of the last iteration (teacher-forcing tests) */
  SGS_F_NO_GRAPHS = 2,       /* launch the decode iteration eagerly (no CUDA graphs) */
  SGS_F_KERNEL_TIMING = 4,   /* CUDA-event timing per kernel class (sgs_kernel_stats) */
  SGS_F_SHADOW_WEIGHTS = 8,  /* reserve a second weight buffer for the asynchronous weight sync */
  SGS_F_TRACE = 16,          /* keep the schedule trace (sgs_trace) and every sample record; off by
                                default: without it the host state is bounded by the samples in flight */
  SGS_F_DETERMINISTIC = 32,  /* no split-K in the GEMMs: bitwise run-to-run reproducible results
                                (split-K's fp32 red.add order is the only variation, R21) */
  SGS_F_SKIP_PREFILL = 64,   /* T(b) profiling only (config 5): admitted prompts are not prefilled (stale
                                KV, garbage tokens); decode iterations and their timing are unchanged */
  SGS_F_PREFIX_SHARING = 128 /* NEXT-3 (R26): samples of one sgs_submit batch with
                                identical prompts (GRPO groups) share the prompt's KV pages; the group's
                                first admitted member runs the prefill, later members start with one decode
                                row at position P-1 over the shared pages */
};

typedef struct {
  int32_t max_batch;         /* B, the per-instance batch cap */
  int32_t page_size;         /* KV page in tokens (16) */
  int32_t max_ctx;           /* longest prompt + output - 1 a sample may reach */
  int32_t max_prefill_tokens;/* prefill chunk, tokens (0 -> 16384) */
  int64_t n_pages;           /* KV pool pages; 0 -> as many as fit in the arena */
  void* arena;               /* device memory from the caller (ignored in null-device mode) */
  int64_t arena_bytes;
  void* stream;              /* cudaStream_t the library launches on (NULL = legacy default) */
  int32_t device;            /* CUDA device ordinal; < 0 -> null-device mode */
  int32_t n_instances;       /* N data-parallel instances (one per GPU / rank) */
  int32_t instance_rank;     /* this handle's instance in [0, N) */
  int32_t dispatch;          /* SGS_DISPATCH_* (Alg. 2 by default) */
  int32_t alpha_pct;         /* long-tail threshold alpha in percent (20) */
  int32_t score;             /* SGS_SCORE_SUM (literal P:935) or SGS_SCORE_MAX */
  int32_t tail_ceil;         /* 0: floor(alpha*n), 1: ceil */
  sgs_tb_profile profile;    /* T(b) used by Eq. 2 */
  int32_t sampling;          /* SGS_SAMPLE_* */
  float temperature, top_p;
  uint64_t sample_seed;      /* Philox key for top-p */
  uint64_t weight_seed;      /* hash-init seed when sgs_init gets no weights */
  int32_t flags;             /* SGS_F_* */
  /* NEXT-2 tensor parallelism: this handle is shard
   * tp_rank of a tp_size-GPU instance (0 or 1 = no TP).  q/kv heads, FFN
   * columns and vocabulary rows are split tp_size ways (they must divide);
   * the O / down projections and the LM head's argmax are combined across
   * shards: in the decode program by exchange kernels over NVLink peer
   * memory (each fused with the RMSNorm that consumes the sum), in prefill
   * (and with SGS_TP_NCCL_AR=1 everywhere) by NCCL all-reduces.  Every shard
   * runs the same scheduler on the same submissions.  TP shards generate
   * their weights from weight_seed (sgs_init's weights must be NULL), decode
   * greedily, and have no debug hooks or weight sync. */
  int32_t tp_size, tp_rank;
} sgs_engine_cfg;

/* One prompt (host memory, copied by sgs_submit). */
typedef struct {
  uint64_t id;               /* unique within the handle's lifetime */
  const int32_t* tokens;     /* host, len token ids in [0, vocab) */
  int32_t len;               /* prompt length P >= 1 */
} sgs_prompt;

/* One completed sample, emitted in ascending id within an iteration. */
typedef struct {
  uint64_t id;
  int32_t instance;
  int32_t n_tokens;          /* = forced length d */
  const int32_t* tokens;     /* host, library-owned, valid until the next sgs_step */
  int64_t admit_iter, finish_iter;  /* per-instance iteration counter */
  int32_t weight_version;
  int32_t slot;
} sgs_completion;

/* Bytes the caller must provide as the arena for a given configuration
 * (weights + KV pool of n_pages + scratch).  kv_page_bytes = bytes of one page
 * over all layers, so callers can size n_pages from free memory. */
sgs_status sgs_arena_bytes(const sgs_model_cfg* m, const sgs_engine_cfg* e, int64_t n_pages,
                           int64_t* fixed_bytes, int64_t* kv_page_bytes);

/* Weights in the canonical tensor order: index 0 embed [V, d],
 * 1 lm_head [V, d], 2 final norm [d]; then per layer l, at 3 + 12 l:
 * +0 Wq [nq hd, d], +1 Wk [nkv hd, d], +2 Wv [nkv hd, d], +3 bq [nq hd],
 * +4 bk [nkv hd], +5 bv [nkv hd], +6 Wo [d, nq hd], +7 Wgate [f, d],
 * +8 Wup [f, d], +9 Wdown [d, f], +10 attention norm [d], +11 MLP norm [d].
 * Every tensor is bf16, row-major in that logical shape (a PyTorch
 * Linear.weight is [out, in]).  ptrs[i] may be host or device memory (CUDA
 * unified addressing decides the copy direction); the library copies the
 * values into its own layout (gate/up interleaved in 64-row blocks; with
 * SGS_WEIGHT_LAYOUT=tiles every GEMM weight matrix stored as contiguous
 * [128 rows x 64 cols] blocks) before the call returns, so the
 * caller keeps ownership (pageable host memory is page-locked for the copy
 * and released).  sgs_weight_tensors lists the order, logical ids and
 * shapes. */
typedef struct {
  const void* const* ptrs;   /* n pointers, canonical order */
  int32_t n;                 /* 3 + 12 * n_layers */
} sgs_weights;

/* Canonical weight order of a model: for i < *n (<= cap): ids[i] = the
 * logical tensor id (0, 1, 2, 16 + 16 l + k: the ids sgs_weight_checksum
 * takes), rows[i] x cols[i] = its shape (cols = 1 for vectors).  Any output
 * pointer may be NULL. */
sgs_status sgs_weight_tensors(const sgs_model_cfg* m, int64_t* ids, int64_t* rows, int64_t* cols, int32_t cap,
                              int32_t* n);

/* Create an instance.  weights == NULL: hash-initialise every tensor on the
 * device from e->weight_seed; otherwise copy the caller's
 * weights (SGS_E_INVAL if weights->n or a pointer is wrong).  Null-device
 * mode ignores arena and weights.  Shapes the sm_100a kernels cannot run
 * (page != 16, head_dim not in {32, 64, 128}, GQA group nq/nkv > 8, model
 * dims not multiples of 128) fail here with SGS_E_UNSUPPORTED. */
sgs_status sgs_init(const sgs_model_cfg* m, const sgs_engine_cfg* e, const sgs_weights* weights, sgs_handle** out);
void sgs_destroy(sgs_handle* h);
const char* sgs_last_error(const sgs_handle* h); /* h may be NULL (init errors) */

/* Submit one RL batch: n prompts with ranker hints and forced
 * output lengths.  Every instance receives the SAME full batch;
 * Alg. 2 runs identically on each and the handle keeps the samples
 * dispatched to its instance_rank (no communication).  Validation: P >= 1,
 * hint >= 1, forced >= 1, tokens in [0, vocab), ids unique within the batch
 * and among the samples still queued or active on this handle (DESIGN.md
 * R22: an id may be reused once its sample has completed); violations ->
 * SGS_E_INVAL with no effect; a sample that can never fit -> SGS_E_CAPACITY.
 * n_mine (optional) receives how many samples this instance kept. */
sgs_status sgs_submit(sgs_handle* h, const sgs_prompt* prompts, int32_t n, const int32_t* output_len_hint,
                      const int32_t* forced_len, int32_t* n_mine);

/* Run one continuous-batching iteration (longest-first refill under B,
 * P:996-998; prefill of admitted prompts + one decode step of the running
 * samples) and return completed samples, ascending id within an iteration.
 * The device work is pipelined with the host: a call launches its iteration
 * and then waits for the previous call's iteration, returning that one's
 * completions (a call with nothing new to launch drains the last one); with
 * SGS_F_KEEP_LOGITS every call returns its own iteration's completions.  With
 * nothing queued, active or in flight: SGS_OK, *n_out = 0, no iteration is
 * counted.  Completions beyond cap stay queued and are returned (before any
 * new iteration) by the next call. */
sgs_status sgs_step(sgs_handle* h, sgs_completion* out, int32_t cap, int32_t* n_out);

/* Samples queued + active on this instance; active includes samples whose last
 * iteration is launched but not yet returned (sgs_step pipelines: it launches
 * iteration i+1 before waiting for iteration i, so a call returns the
 * completions of the previous iteration). */
sgs_status sgs_pending(const sgs_handle* h, int64_t* queued, int64_t* active);

/* Host-side state of the handle: sample records held, scheduler queue
 * entries held (consumed prefix included until compacted), and ids reserved
 * (queued or active).  Without SGS_F_TRACE all three stay bounded by the
 * samples in flight plus one batch, however many batches are served. */
sgs_status sgs_host_state(const sgs_handle* h, int64_t* records, int64_t* queue_entries, int64_t* live_ids);

/* Weight sync (SGS "update(weights)" P:595-596): the only
 * collective.  sgs_comm_unique_id on the root, share the 128 bytes (e.g.
 * torch.distributed), sgs_comm_init on every rank, then sgs_update_weights
 * on every rank: the root first copies src (the trainer's new weights,
 * canonical order, host or device; NULL = keep the root's current weights)
 * into its arena, then the root's weights are broadcast to all ranks
 * (ncclBroadcast over NVLink; at world size 1 the copy alone) and the weight
 * version increments.  Non-root ranks must pass src = NULL.  Requires no
 * sample in flight (SGS_E_STATE otherwise). */
sgs_status sgs_comm_unique_id(uint8_t out[128]);
sgs_status sgs_comm_init(sgs_handle* h, const uint8_t id[128], int32_t rank, int32_t world);
/* NEXT-2: the tensor-parallel communicator of a tp_size > 1 handle (unique id
 * from sgs_comm_unique_id on shard 0, shared by the caller); must precede the
 * first sgs_step.  Collective over the shards: it also allocates this shard's
 * peer-exchange buffer (cudaMalloc, freed by sgs_destroy; the one allocation
 * outside the arena), gathers the shards' CUDA IPC handles over the new
 * communicator and opens the peers' buffers.  SGS_E_CUDA when IPC is not
 * available (then set SGS_TP_NCCL_AR=1 on every shard). */
sgs_status sgs_tp_comm_init(sgs_handle* h, const uint8_t id[128]);
sgs_status sgs_update_weights(sgs_handle* h, const sgs_weights* src, int32_t root);
/* Trainer proxy: regenerate this handle's weights from a new seed on device
 * (the root does this before sgs_update_weights). */
sgs_status sgs_load_weights_seed(sgs_handle* h, uint64_t seed);
/* Asynchronous (overlapped) weight sync -- SURVEY NEXT-1, the paper's fully
 * asynchronous pipelining with staleness 1 over the weight
 * transmission of P:1022-1030.  Needs SGS_F_SHADOW_WEIGHTS.  The next weights
 * are written into the shadow buffer (by a trainer through
 * sgs_shadow_weights, or sgs_stage_weights_seed as the trainer proxy), then
 * sgs_update_weights_begin broadcasts the root's shadow buffer to every
 * rank's shadow buffer on a side stream while generation continues on the
 * current weights; sgs_update_weights_commit (RL-batch boundary: no sample in
 * flight, SGS_E_STATE otherwise) makes the engine stream wait for the
 * broadcast, copies shadow -> active on the device and increments the
 * version, so the samples of the next batch are generated with the new
 * weights and stamped with the new version.  One update may be in flight
 * (SGS_E_STATE for a second begin or a stage during it).  Ordering: staging
 * and the broadcast run on the library's side stream, which waits for the
 * previous commit's shadow -> active copy, so a stage or begin may follow a
 * commit immediately; a caller that writes the shadow buffer directly
 * (through sgs_shadow_weights) must first synchronise the handle's stream
 * after a commit, and writes the library's internal layout (the arena's
 * weight region byte for byte); sgs_stage_weights takes canonical tensors. */
sgs_status sgs_shadow_weights(sgs_handle* h, void** ptr, int64_t* bytes);
sgs_status sgs_stage_weights_seed(sgs_handle* h, uint64_t seed);
/* Trainer path of the asynchronous sync: copy src (canonical order, host or
 * device) into the shadow buffer on the side stream. */
sgs_status sgs_stage_weights(sgs_handle* h, const sgs_weights* src);
sgs_status sgs_update_weights_begin(sgs_handle* h, int32_t root);
/* *ready = 1 once the in-flight broadcast has completed on the device. */
sgs_status sgs_update_weights_ready(sgs_handle* h, int32_t* ready);
sgs_status sgs_update_weights_commit(sgs_handle* h);
/* Order-independent 64-bit checksum of one logical weight tensor (DESIGN.md
 * §3 tensor ids): sum_i bits16(w_i) * (2i+1) mod 2^64. */
sgs_status sgs_weight_checksum(sgs_handle* h, int64_t tensor_id, uint64_t* out);
sgs_status sgs_weight_version(const sgs_handle* h, int32_t* out);

/* Trace for schedule parity (DESIGN.md §5 format, int64 stream): iteration
 * records t,b,sumctx,nadm,ncomp,nalloc,nfree,adm...,comp...,alloc...,freed...
 * (which = 0) or per-sample records id,slot,admit,finish,npages,pages...
 * (which = 1, ascending id, samples admitted so far).  buf == NULL -> *n gets
 * the length.  The iteration trace can be cleared with sgs_trace_clear. */
sgs_status sgs_trace(const sgs_handle* h, int32_t which, int64_t* buf, int64_t cap, int64_t* n);
sgs_status sgs_trace_clear(sgs_handle* h);

/* fp32 logits of the last iteration (SGS_F_KEEP_LOGITS): rows = samples that
 * produced a token, in (prefill-first, then ascending slot) order; ids[r] and
 * pos[r] (index of the generated token, 0-based) identify each row. */
sgs_status sgs_last_logits(sgs_handle* h, float* logits, uint64_t* ids, int32_t* tok_idx, int32_t cap,
                           int32_t* rows);

/* Layer-by-layer parity hook: a standalone prefill forward of one prompt
 * (tokens host int32 [T], slot 0, idle handle only) that dumps the fp32
 * residual stream after the embedding and after every residual add into
 * dump (host, [(2*n_layers+1) x T x d_model]). */
sgs_status sgs_debug_forward(sgs_handle* h, const int32_t* tokens, int32_t T, float* dump);
/* Layer-local parity hook: run decoder layer `layer` of the CUDA path (prefill
 * form, positions 0..T-1, slot 0, idle handle only) on the fp32 residual
 * stream h_in (host [T x d_model]) and return the stream after the layer's
 * MLP residual add in h_out (host [T x d_model]).  layer == n_layers runs the
 * final RMSNorm + LM head on h_in instead: h_out is then fp32 logits
 * (host [T x vocab]). */
sgs_status sgs_debug_layer(sgs_handle* h, int32_t layer, const float* h_in, int32_t T, float* h_out);

/* Device-side timing of the last iteration's kernels (CUDA events), ms. */
sgs_status sgs_last_iter_ms(sgs_handle* h, float* ms);
/* Per kernel class (0 decode attention K1+K2, 1 decode GEMMs, 2 prefill
 * attention, 3 device time of the timed iterations, 4 prefill GEMMs, 5 other
 * decode kernels: RMSNorm, RoPE + KV append, embedding, sampler; the timed
 * iterations are ~1 in 64, chosen by a hash of the iteration counter); add 6
 * for the timed iterations with >= 129 decode rows only, 12 for those with
 * 1..32,
 * accumulated with SGS_F_KERNEL_TIMING: device ms (CUDA events on the
 * launching stream), algorithmic bytes and flops, launches.  reset != 0 clears. */
sgs_status sgs_kernel_stats(sgs_handle* h, int32_t cls, double* ms, double* bytes, double* flops, int64_t* launches,
                            int32_t reset);
/* Roofline denominators for sgs_kernel_stats' roofline time: every timed
 * launch contributes max(bytes / (bw_gbs GB/s), flops / (tflops TFLOP/s)). */
sgs_status sgs_set_roofline(sgs_handle* h, double bw_gbs, double tflops);
sgs_status sgs_kernel_roofline_ms(const sgs_handle* h, int32_t cls, double* ms);
/* Per-iteration log (T(b) profiling): 6 int64 per executed iteration
 * {t, b, admitted, prefill tokens, sum of contexts, device time in us}. */
sgs_status sgs_iter_log(const sgs_handle* h, int64_t* buf, int64_t cap, int64_t* n);

/* Host<->device bytes moved by the service calls so far (metadata, prompts, tokens). */
sgs_status sgs_io_bytes(const sgs_handle* h, int64_t* h2d, int64_t* d2h);

/* Count of kernel launches (or graph launches' kernels) issued so far. */
sgs_status sgs_kernel_launches(const sgs_handle* h, int64_t* n);

/* NEXT-4, elastic DP scale-out (§4.2 "Dynamic adjustment"): the
 * predicted generation time of this batch (n prompts, ranker hints as output
 * lengths) on e->n_instances = N instances and on N + 1 -- Alg. 2 dispatch,
 * then each instance's longest-first schedule timed with e->profile, makespan
 * over instances (R25) -- in t_gen_ps[2]; delta' = t_gen_ps[0] -
 * t_gen_ps[1]; *scale_out = delta' > 0 && delta_ps >= delta', delta_ps being
 * the measured generation time minus the measured training time.  pool_pages
 * is one instance's KV pool.  Pure host function. */
sgs_status sgs_elastic_plan(const sgs_engine_cfg* e, int32_t n, const uint64_t* ids, const int32_t* prompt_len,
                            const int32_t* hint, int64_t pool_pages, int64_t delta_ps, int64_t t_gen_ps[2],
                            int64_t* delta_prime_ps, int32_t* scale_out);
/* NEXT-2 two-dimensional dispatch (P:390-393 tensor parallelism for per-sample
 * latency, P:856-861 long-tail samples on dedicated instances; DESIGN.md
 * R27): the k longest samples by hint (ties: smaller id) go to one tp_size-GPU
 * tensor-parallel instance (max batch tp_max_batch, KV pool tp_pool_pages,
 * T(b) tp_profile), the other n - k to the e->n_instances DP instances
 * (e->dispatch policy, e->max_batch, e->profile, pool_pages each).  Both sides
 * are predicted like sgs_elastic_plan (longest-first schedule on the hints),
 * each iteration priced at T(b) + kv_ps (tp_kv_ps for the TP instance) times
 * the cached context tokens of its samples + pf_ps (tp_pf_ps) times the prompt
 * tokens it prefills (0, 0 = T(b) alone).
 * k is the smallest k in [0, n] with T_tp(k) >= T_dp(k) (binary search), or
 * k - 1 when that has the smaller max(T_tp, T_dp) (ties: k - 1).  Out:
 * *n_tail = k; t_ps = {T_tp(k), T_dp(k), T_all} with T_all the prediction for
 * all n samples on n_instances + tp_size DP instances (use TP iff
 * max(T_tp, T_dp) < T_all).  Pure host function. */
sgs_status sgs_tp_tail_plan(const sgs_engine_cfg* e, int64_t pool_pages, int32_t tp_size, int32_t tp_max_batch,
                            int64_t tp_pool_pages, const sgs_tb_profile* tp_profile, int64_t kv_ps, int64_t tp_kv_ps,
                            int64_t pf_ps, int64_t tp_pf_ps, int32_t n, const uint64_t* ids,
                            const int32_t* prompt_len, const int32_t* hint, int32_t* n_tail, int64_t t_ps[3]);
/* Change this handle's data-parallel layout (N instances, its rank) between
 * RL batches -- the elastic scale-out of NEXT-4; SGS_E_STATE while samples
 * are queued or in flight. */
sgs_status sgs_set_instances(sgs_handle* h, int32_t n_instances, int32_t instance_rank);

/* T(b) fit (C3): hinge least squares over n measured (b, T_ns)
 * points; out = {t0, k0, k1, t1, sse}, prof = rounded integer profile.
 * Returns SGS_E_INVAL when no breakpoint is identifiable. */
sgs_status sgs_fit_profile(int32_t n, const double* b, const double* T_ns, double out[5], sgs_tb_profile* prof);

/* Alg. 2 on its own (pure host function): instance per sample. */
sgs_status sgs_dispatch_plan(const sgs_engine_cfg* e, int32_t n, const uint64_t* ids, const int32_t* prompt_len,
                             const int32_t* hint, int64_t pool_pages, int32_t* instance, int32_t* n_l);

/* ------------------------------------------------------------------------
 * Kernel-level entry points (device pointers; launched on `stream`).  These
 * are the hot-path kernels the iteration is built from, exported so the
 * parity tests can drive each one against the oracle.
 * ------------------------------------------------------------------------ */

/* a8/K1+K2: paged GQA decode attention (P:361-363 memory-bound decode).
 * q:      device bf16 [b, nq, hd]
 * kv:     device bf16 page pool, one layer: [n_pages][nkv][2][page][hd] with
 *         16-byte chunks XOR-swizzled within each row
 * block_table: device int32 [b, max_pages_per_seq]; ctx: device int32 [b]
 * out:    device, [b, nq, hd], bf16 (out_fp32 = 0) or fp32 (out_fp32 = 1)
 * workspace: device, >= sgs_attn_workspace_bytes(...) bytes
 * Work is split over KV pages (split-K) and merged with the LSE combine. */
int64_t sgs_attn_workspace_bytes(int32_t b, int32_t nq, int32_t nkv, int32_t hd, int32_t max_pages_per_seq);
sgs_status sgs_op_decode_attention(const void* q, const void* kv, const int32_t* block_table, const int32_t* ctx,
                                   int32_t b, int32_t nq, int32_t nkv, int32_t hd, int32_t page,
                                   int32_t max_pages_per_seq, int32_t max_ctx_hint, void* out, int32_t out_fp32,
                                   void* workspace, int64_t workspace_bytes, int32_t split_pages, void* stream);

/* Config-5 measurement of the same kernel (no data-dependent host work in the
 * timed region): plans the work list once, launches the kernel reps times on
 * stream with CUDA events around each launch, writing l2_flush_bytes of
 * l2_flush (device scratch, may be NULL/0) between launches so that each
 * launch reads its KV from HBM; *ms = mean device time per launch. */
sgs_status sgs_op_decode_attention_timed(const void* q, const void* kv, const int32_t* block_table,
                                         const int32_t* ctx, int32_t b, int32_t nq, int32_t nkv, int32_t hd,
                                         int32_t page, int32_t max_pages_per_seq, void* out, void* workspace,
                                         int64_t workspace_bytes, int32_t reps, void* l2_flush,
                                         int64_t l2_flush_bytes, float* ms, void* stream);

/* K3/K4: tcgen05 bf16 GEMM, C[t, n] (+)= sum_k X[t, k] * W[n, k].
 * W device bf16 [N, K] row-major; X device bf16 [T, K]; C device fp32 [T, ldc].
 * mode 0: C = result; mode 1: C += result (atomic, split-K capable).
 * splits: K splits (mode 1 only; 0 = automatic).  N % 128 == 0, K % 64 == 0. */
sgs_status sgs_op_gemm(const void* W, const void* X, void* C, int32_t N, int32_t K, int32_t T, int32_t ldc,
                       int32_t mode, int32_t splits, void* stream);

/* a6/K6: y[t] = bf16(x[t] / sqrt(mean(x[t]^2) + eps) * w); x fp32 [T, d], w bf16 [d]. */
sgs_status sgs_op_rmsnorm(const float* x, const void* w, void* y, int32_t T, int32_t d, float eps, void* stream);

/* a7/K7: RoPE + KV append.  qkv fp32 [T, (nq+2nkv)*hd] (+ bias bf16),
 * pos int32 [T], slot int32 [T] -> q bf16 [T, nq, hd]; k, v written into the
 * page pool via block_table[slot][pos/page], pos % page (slot -1: row skipped).
 * cos_sin fp32 [max_pos, hd/2, 2] from sgs_rope_table.  qkv is zeroed after it
 * is read (it is the split-K accumulator of the next QKV GEMM). */
sgs_status sgs_op_rope_append(const float* qkv, const void* bias, const int32_t* pos, const int32_t* slot,
                              const int32_t* block_table, int32_t max_pages_per_seq, const float* cos_sin,
                              void* q_out, void* kv, int32_t T, int32_t nq, int32_t nkv, int32_t hd, int32_t page,
                              void* stream);
sgs_status sgs_rope_table(float* host_out, int32_t max_pos, int32_t hd, double theta);

/* a4/K10: causal prefill attention.  q device bf16 [T, nq, hd]; k, v device
 * bf16 [T, nkv, hd] (contiguous, not paged); prompt p spans rows
 * [offs[p], offs[p+1]) (offs device int32 [n_prompts+1]); out bf16 [T, nq, hd].
 * hd = 128 runs the tcgen05/TMEM kernel (P.V in fp16 on fp16(bf16 v), exact
 * conversion); other hd the mma.sync kernel.  workspace: device, >=
 * sgs_prefill_workspace_bytes(T, n_prompts, nkv, hd) bytes (query-block list
 * and the fp16 v copy); SGS_E_NOMEM when smaller.  Synchronises stream. */
int64_t sgs_prefill_workspace_bytes(int32_t T, int32_t n_prompts, int32_t nkv, int32_t hd);
sgs_status sgs_op_prefill_attention(const void* q, const void* k, const void* v, const int32_t* offs,
                                    int32_t n_prompts, int32_t nq, int32_t nkv, int32_t hd, void* out,
                                    void* workspace, int64_t workspace_bytes, void* stream);

/* a10 epilogue: m[t, i] = bf16(SiLU(gu[t, i]) * gu[t, f + i]); gu fp32 [T, 2f], m bf16 [T, f].
 * gu is zeroed after it is read. */
sgs_status sgs_op_silu_mul(const float* gu, void* m, int32_t T, int32_t f, void* stream);

/* K9 top-p (R18): p = softmax(logits/temperature) in fp32; nucleus =
 * shortest prefix in (p desc, id asc) order with mass >= top_p; u = 24-bit
 * uniform of Philox4x32-10(key = seed, ctr = (sample_id, step)) times the
 * nucleus mass; ids[r] = first token of that order whose cumulative mass > u.
 * sample_ids: device uint64 [rows]; steps: device int32 [rows]. */
sgs_status sgs_op_sample_top_p(const float* logits, int32_t rows, int32_t V, float temperature, float top_p,
                               uint64_t seed, const uint64_t* sample_ids, const int32_t* steps, int32_t* ids,
                               void* stream);

/* K9 greedy: ids[r] = argmax_v logits[r, v] (lowest index on ties). */
sgs_status sgs_op_argmax(const float* logits, int32_t rows, int32_t V, int32_t* ids, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SGS_H_ */
