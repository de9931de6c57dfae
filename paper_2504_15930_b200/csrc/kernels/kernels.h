// Host-side launchers of the sm_100a kernels (internal to libsgs).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace sgs {

// ---- GEMM (gemm.cu): C[t, n] (+)= X[t, :] . W[n, :]; mode 0 store, 1 atomic add, 2 add
// mode 3: fused SwiGLU epilogue for gate/up weights in the interleaved
// layout; C is then bf16 [T, ldc] with ldc = N/2 (requires splits == 1).
// mode 4: greedy sampling fused into the epilogue (LM head): every CTA folds
// its tile's (max logit, lowest vocab index) per token into keys[t] (packed
// 64-bit atomicMax); the last CTA to finish writes the argmax of row t to
// last_tok[slot[t]] and hist[slot[t] * max_gen + tok_idx[t]] (slot < 0: padding
// row) and re-zeroes keys and the arrival counter.  C (may be NULL) also gets
// the fp32 logits as in mode 0.
struct ArgmaxArgs {
  unsigned long long* keys;  // [>= T], zero between launches
  unsigned int* done;        // arrival counter, zero between launches
  const int32_t* slot;
  const int32_t* tok_idx;
  int32_t* last_tok;
  int32_t* hist;
  int max_gen;
  int vocab_off = 0;  // tensor-parallel shard: index of its first vocabulary row
  int finalize = 1;   // 0: leave the keys for a cross-shard all-reduce (argmax_keys_finalize)
};
// RMSNorm fused in front of a GEMM (decode program): before the GEMM reads its
// activation operand X, the CTAs of the (persistent, co-resident) grid compute
// X = bf16(h / sqrt(mean(h^2) + eps) * w) row by row (rows blockIdx.x, +grid;
// the arithmetic of the standalone rmsnorm kernel) and meet at a grid barrier;
// the activation TMA loads start after it, the weight loads before it.  The
// barrier counter bar[2 * site + parity] (zero-initialised) is armed by the
// last arrival resetting the other parity's counter; `parity` must alternate
// between consecutive launches of the same site.
struct PreNorm {
  const float* h;            // fp32 residual stream [T, K]
  const void* w;             // bf16 norm weight [K]
  void* x;                   // bf16 [T, K]: written here, the GEMM's X (set by gemm_bf16)
  float eps;
  unsigned int* bar;         // barrier counters
  int site;
  const int32_t* parity;     // device int: launch parity of this site (read after griddepcontrol.wait)
};
cudaError_t gemm_bf16(const void* W, const void* X, float* C, int N, int K, int T, int ldc, int mode, int splits,
                      cudaStream_t stream, const ArgmaxArgs* am = nullptr, const PreNorm* pn = nullptr,
                      int w_tiled = 0);  // 1: W in the tiled layout [N/128][K/64][128][64] (weight_layout below)
int gemm_auto_splits(int N, int K, int T);

// ---- decode attention (attention.cu)
struct AttnItem {
  int32_t row, kvh, p0, p1, part;  // part < 0: the item covers the whole row -> final output
  int32_t comb;                     // split items: index of their AttnComb
  int32_t slot, ctx;                // block-table row and context length of the sample
};
struct AttnComb {
  int32_t row, kvh, part0, nparts;
};
struct AttnPlan {
  std::vector<AttnItem> items;
  std::vector<AttnComb> combs;
  int n_parts = 0;
};
// Split-K plan over pages: about one wave of 2 CTAs per SM -- a (row, kv
// head) with np of the total pages gets floor(296 np / total) parts (>= 8
// pages each, <= 32 parts).  The item count is bounded by 296 + b*nkv (+ the
// split_pages override, <= 64 parts per row and kv head).
// slot[row] is the block-table row of each sample (NULL: the row index).
void attn_plan(const int32_t* ctx, const int32_t* slot, int b, int nkv, int page, int split_pages, AttnPlan* plan);
int64_t attn_workspace_bytes(int max_items, int max_parts, int g, int hd);
// items/combs are device arrays (already copied); part buffers in workspace.
// Each item carries its sample's block-table row (slot) and context length.
// Split items merge in-kernel: the last part of a (row, kv head) to finish
// combines (arrive = zero-initialised int[n_combs] counters, self re-arming).
// counts (device, optional): {n_items, n_combs} read by the kernels, in which
// case n_items / n_combs are only the launch capacities (CUDA-graph replay).
// PDL: items, counts, the block table and every KV page older than the one
// holding token ctx-1 are read before griddepcontrol.wait (they are written
// before the launching CUDA graph / stream segment starts, never by the
// predecessor kernels); q and the newest page are read after it.
cudaError_t attn_decode(const void* q, const void* kv, const int32_t* block_table, const int32_t* counts,
                        const AttnItem* items, int n_items, const AttnComb* combs, int n_combs, int nq, int nkv,
                        int hd, int page, int max_pages, void* out, int out_fp32, float* part_o, float* part_ml,
                        int* arrive, cudaStream_t stream);

// 2-byte-element row-major [rows, cols] matrix as a TMA map of (64 cols, box_rows,
// kc 64-col chunks) boxes with the 128-byte swizzle (cached per pointer/shape).
bool tmap_bf16_rows(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int box_rows, int kc);

// ---- prefill attention (prefill_attn.cu): causal within each prompt.
// q [T, nq, hd], k/v [T, nkv, hd] contiguous bf16; prompt p spans rows
// [offs[p], offs[p+1]).  out bf16 [T, nq, hd].
cudaError_t attn_prefill(const void* q, const void* k, const void* v, const int32_t* offs, const int32_t* qblocks,
                         int n_qblocks, int nq, int nkv, int hd, void* out, cudaStream_t stream);
// tcgen05/TMEM/TMA flash attention for hd = 128 (prefill_attn_tc.cu): same
// contract, except v is fp16 (= fp16(bf16 v), exact) and the work list holds
// (prompt, 128-query block) pairs; T = rows of q/k/v (TMA bounds).
cudaError_t attn_prefill_tc(const void* q, const void* k, const void* v_f16, const int32_t* offs,
                            const int32_t* qblocks128, int n_qblocks128, int T, int nq, int nkv, void* out,
                            cudaStream_t stream);

// ---- elementwise (elementwise.cu)
cudaError_t rmsnorm(const float* x, const void* w, void* y, const int32_t* rows, int T, int d, float eps,
                    cudaStream_t stream);
cudaError_t rope_append(const float* qkv, const void* bias, const int32_t* pos, const int32_t* slot,
                        const int32_t* block_table, int max_pages, const float* cos_sin, void* q_out, void* kv,
                        void* k_out, void* v_out, int T, int nq, int nkv, int hd, int page, cudaStream_t stream,
                        int v_f16 = 0);  // v_f16: the contiguous v copy as fp16(bf16 v)
cudaError_t embed(const void* E, const int32_t* tokens, const int32_t* slots, const int32_t* last_tok, float* h,
                  int T, int d, cudaStream_t stream);
cudaError_t silu_mul(const float* gu, void* m, int T, int f, cudaStream_t stream);
cudaError_t bf16_to_f16(const void* src, void* dst, int64_t n, cudaStream_t stream);
cudaError_t argmax_rows(const float* logits, int rows, int V, int32_t* ids, const int32_t* slot,
                        const int32_t* tok_idx, int32_t* last_tok, int32_t* out_hist, int max_gen,
                        cudaStream_t stream);
// Row-block mapping (blk, stride, off) for the interleaved gate/up weights; blk 0 = contiguous.
// top-p (nucleus) sampling, R18; sample_ids: uint32 pairs (lo, hi) per row.
cudaError_t sample_top_p(const float* logits, int rows, int V, float temperature, float top_p, uint64_t seed,
                         const uint32_t* sample_ids, int32_t* ids, const int32_t* slot, const int32_t* tok_idx,
                         int32_t* last_tok, int32_t* out_hist, int max_gen, cudaStream_t stream);
// tensor-parallel shard of a weight tensor: element i of the shard is element
// (row0 + i / lcols) * src_cols + col0 + i % lcols of the full tensor (src_cols 0: identity)
struct ShardMap {
  int64_t src_cols = 0, row0 = 0, col0 = 0, lcols = 1;
};
// Weight placement: element i = (r, c) of a row-major [n / cols, cols] tensor
// lands at row R = (r / blk) * stride + off + r % blk of its fused matrix
// (blk = 0: R = r; the interleaved gate/up rows), and, with tiled = 1, in the
// GEMM weight layout [R/128][cols/64][128][64] (16 KB blocks, one TMA box each).
cudaError_t hash_init(void* dst, uint64_t seed, uint64_t tensor_id, int64_t n, int is_norm, cudaStream_t stream,
                      int64_t cols = 1, int blk = 0, int stride = 0, int off = 0, ShardMap sm = ShardMap{},
                      int tiled = 0);
// dst[placement(i)] = src[i] for a canonical row-major bf16 tensor readable by the device
cudaError_t relayout_bf16(const void* src, void* dst, int64_t n, int64_t cols, int blk, int stride, int off, int tiled,
                          cudaStream_t stream);
cudaError_t argmax_keys_finalize(unsigned long long* keys, int rows, const int32_t* slot, const int32_t* tok_idx,
                                 int32_t* last_tok, int32_t* hist, int max_gen, cudaStream_t stream);
// ---- NEXT-2 tensor-parallel exchange over NVLink peer memory (tp_comm.cu)
constexpr int TPX_MAX = 8;     // shards
constexpr int TPX_CTAS = 296;  // CTAs of one exchange (two per SM, co-resident)
struct TpPeers {
  uint8_t* base[TPX_MAX];  // every shard's exchange buffer, mapped in this process (own at [me])
  int me, tp;
};
size_t tp_xch_bytes(int tp, int rows, int d);
// exchange epoch = *launch * per_launch + index + 1 (launch: device counter of
// the decode launch, index: the exchange's position in it, < per_launch)
cudaError_t tp_allreduce_rmsnorm(float* h, const void* w, void* y, int T, int d, float eps, const TpPeers& P,
                                 int rows_cap, const int32_t* launch, int index, int per_launch, cudaStream_t stream);
cudaError_t tp_argmax_exchange(unsigned long long* keys, int rows, const int32_t* slot, const int32_t* tok_idx,
                               int32_t* last_tok, int32_t* hist, int max_gen, const TpPeers& P, int rows_cap, int d,
                               const int32_t* launch, int index, int per_launch, cudaStream_t stream);
cudaError_t checksum_bf16(const void* src, int64_t n, unsigned long long* out_dev, cudaStream_t stream,
                          int64_t cols = 1, int blk = 0, int stride = 0, int off = 0, int tiled = 0);
cudaError_t apply_bt_deltas(int32_t* block_table, int max_pages, const int32_t* deltas, int n, cudaStream_t stream,
                            int32_t* last_tok = nullptr);
cudaError_t copy_kv_pages(void* pool, int64_t layer_stride, int64_t page_bytes, int n_layers, const int32_t* pairs,
                          int n_pairs, cudaStream_t stream);

}  // namespace sgs
