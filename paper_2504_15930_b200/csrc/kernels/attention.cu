// a8 / K1+K2: paged GQA decode attention with split-K over KV pages.
//
//   o_h = softmax(q_h K^T / sqrt(hd)) V     over the ctx cached tokens of a sample
//
// Decode is memory-bandwidth bound (§2.2); every byte of the KV
// cache is read once per layer.  One CTA = 4 warps handles one work item
// (sample row, kv head, page range).  Each warp streams its own pages
// (page, page+4, ...) through a private 3-stage shared-memory ring with 1-D
// bulk copies (TMA unit, completion on an mbarrier): one page-head = K and V
// of 16 tokens = 8 KB contiguous (hd = 128).  The g query heads of the group
// are the M = 16 rows of mma.sync.m16n8k16 (rows >= g are zero): S = Q K^T in
// bf16 with fp32 accumulation (ldmatrix from the XOR-swizzled page rows, bank
// conflict free), online softmax in fp32 with exp2 and quad shuffles, then
// O += P V with P in fp16 (V converted bf16 -> fp16 in registers) so the
// softmax weights keep 11 mantissa bits (the 1e-3 target).
// The 4 warps merge their (m, l, O) in shared memory; items that cover a
// whole row write o directly, split items write fp32 partials that the
// combine kernel merges with the log-sum-exp rule
//   o = sum_j 2^(m_j - M) O_j / sum_j 2^(m_j - M) l_j.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace sgs {

constexpr int ATTN_WARPS = 4;
constexpr int ATTN_STAGES = 3;
constexpr int PAGE_T = 16;
constexpr int ATTN_MAX_PARTS = 64;  // the planner never splits a (row, kv head) into more parts

__device__ __forceinline__ void combine_merge(const AttnComb& c, int nq, int nkv, int hd,
                                              const float* __restrict__ part_o, const float* __restrict__ part_ml,
                                              void* __restrict__ out, int out_fp32);

template <int HD>
__global__ void __launch_bounds__(128, 2)
    attn_decode_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ kv,
                       const int32_t* __restrict__ bt, const AttnItem* __restrict__ items, int n_items,
                       const int32_t* __restrict__ counts,
                       int nq, int nkv, int max_pages,
                       float scale_log2, void* __restrict__ out, int out_fp32, float* __restrict__ part_o,
                       float* __restrict__ part_ml, const AttnComb* __restrict__ combs, int* __restrict__ arrive) {
  constexpr int RC = HD / 8;                 // 16-byte chunks per row
  constexpr int HALF = PAGE_T * HD * 2;      // K (or V) bytes of one page-head
  constexpr int STAGE = 2 * HALF;
  constexpr int NT = HD / 8;                 // n8 tiles of the output
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[ATTN_WARPS][ATTN_STAGES];

  pdl_trigger();
  // Before griddepcontrol.wait: the work item, the block table and every KV
  // page that does not hold the newest token were written before this CUDA
  // graph (stream segment) started, so their loads overlap the predecessor
  // kernels; only q and the newest page (rope_append's output) wait.
  if ((int)blockIdx.x >= (counts ? counts[0] : n_items)) {
    pdl_wait();
    return;
  }
  const AttnItem it = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = nq / nkv;
  const int L = it.ctx;
  const int last_page = (L - 1) / PAGE_T;  // written by the predecessor this iteration
  const int32_t* btr = bt + (size_t)it.slot * max_pages;
  uint8_t* my = smem + (size_t)warp * ATTN_STAGES * STAGE;

  if (lane == 0) {
    for (int s = 0; s < ATTN_STAGES; ++s) mbar_init(&bars[warp][s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  const int npages = it.p1 - it.p0;
  const int n_my = npages > warp ? (npages - warp + ATTN_WARPS - 1) / ATTN_WARPS : 0;
  // the warp's block-table entries, 32 at a time in lane registers (lane k
  // holds the page of the warp's (32 j + k)-th page): the ring refill then
  // needs a shuffle, not a dependent global load, before each bulk copy
  auto bt_batch = [&](int j) {
    const int i = 32 * j + lane;
    return i < n_my ? btr[it.p0 + warp + ATTN_WARPS * i] : 0;
  };
  int my_pages = bt_batch(0);
  auto issue = [&](int i, int page) {
    const __nv_bfloat16* src = kv + ((size_t)page * nkv + it.kvh) * (size_t)(2 * PAGE_T * HD);
    uint64_t* b = &bars[warp][i % ATTN_STAGES];
    mbar_expect_tx(b, STAGE);
    bulk_g2s(my + (size_t)(i % ATTN_STAGES) * STAGE, src, STAGE, b);
  };
  const int first = n_my < ATTN_STAGES ? n_my : ATTN_STAGES;
  int pre = 0;  // ring slots whose page is complete (pages ascend with i)
  while (pre < first && it.p0 + warp + ATTN_WARPS * pre < last_page) ++pre;
  for (int i = 0; i < pre; ++i) {
    const int pg = __shfl_sync(0xffffffffu, my_pages, i);
    if (lane == 0) issue(i, pg);
  }
  pdl_wait();
  for (int i = pre; i < first; ++i) {
    const int pg = __shfl_sync(0xffffffffu, my_pages, i);
    if (lane == 0) issue(i, pg);
  }

  // Transposed formulation (tokens are the MMA's M dimension, the g <= 8
  // query heads its N): S^T = K Q^T and O^T += V^T P^T, so a 16-token page
  // step is 8 + 2x8 mma.m16n8k16 instead of 16 + 2x16 with heads as M.
  // Q^T fragments (B operand): head = lane/4, hd pairs 2(lane%4) (+8).
  const int hq = lane >> 2, cq = 2 * (lane & 3);
  uint32_t qb[HD / 16][2];
  {
    const uint32_t* qrow = reinterpret_cast<const uint32_t*>(q + ((size_t)it.row * nq + (size_t)it.kvh * g) * HD);
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      qb[kk][0] = hq < g ? qrow[(hq * HD + 16 * kk + cq) >> 1] : 0u;
      qb[kk][1] = hq < g ? qrow[(hq * HD + 16 * kk + 8 + cq) >> 1] : 0u;
    }
  }
  float o[HD / 16][4];  // O^T: rows hd 16 mt + lane/4 (+8), columns heads cq, cq + 1
#pragma unroll
  for (int i = 0; i < HD / 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // heads cq, cq + 1

  // ldmatrix lane coordinates: A fragments of K (tokens x hd) and V^T (hd x tokens)
  const int arow = (lane & 7) + (((lane >> 3) & 1) << 3), achk = lane >> 4;         // K, non-transposed
  const int vrow = (lane & 7) + (((lane >> 4) & 1) << 3), vchk = (lane >> 3) & 1;   // V, transposed

  for (int i = 0; i < n_my; ++i) {
    const int s = i % ATTN_STAGES;
    mbar_wait(&bars[warp][s], (i / ATTN_STAGES) & 1);
    const uint32_t kbase = smem_u32(my + (size_t)s * STAGE);
    const uint32_t vbase = kbase + HALF;
    const int tok0 = (it.p0 + warp + ATTN_WARPS * i) * PAGE_T;

    float sc[4] = {0.f, 0.f, 0.f, 0.f};  // S^T: tokens lane/4 (+8) x heads cq, cq + 1
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      const int ch = 2 * kk + achk;
      uint32_t a[4];
      ldmatrix_x4(a[0], a[1], a[2], a[3], kbase + arow * (HD * 2) + ((ch ^ kv_swz(arow, RC)) << 4));
      mma_bf16_16816(sc, a, qb[kk][0], qb[kk][1]);
    }
    // mask tokens beyond the context (only the last page is partial)
    if (tok0 + PAGE_T > L) {
      if (tok0 + hq >= L) sc[0] = sc[1] = -INFINITY;
      if (tok0 + hq + 8 >= L) sc[2] = sc[3] = -INFINITY;
    }
    // online softmax per head over the 16 tokens (base 2, pre-scaled scores):
    // the tokens of a head live in lanes with equal lane % 4
    float mx0 = fmaxf(sc[0], sc[2]) * scale_log2, mx1 = fmaxf(sc[1], sc[3]) * scale_log2;
#pragma unroll
    for (int x = 4; x < 32; x <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, x));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, x));
    }
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float a0 = exp2f(m0 - mn0), a1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    const float p00 = exp2f(fmaf(sc[0], scale_log2, -mn0)), p01 = exp2f(fmaf(sc[1], scale_log2, -mn1));
    const float p10 = exp2f(fmaf(sc[2], scale_log2, -mn0)), p11 = exp2f(fmaf(sc[3], scale_log2, -mn1));
    l0 = l0 * a0 + (p00 + p10);
    l1 = l1 * a1 + (p01 + p11);
    // P^T as the B operand (tokens x heads): transpose the two 8x8 blocks
    uint32_t h0, lo0, h1, lo1;
    split_bf16x2(p00, p01, h0, lo0);  // tokens 0..7
    split_bf16x2(p10, p11, h1, lo1);  // tokens 8..15
    const uint32_t bh0 = movmatrix_trans(h0), bh1 = movmatrix_trans(h1);
    const uint32_t bl0 = movmatrix_trans(lo0), bl1 = movmatrix_trans(lo1);
#pragma unroll
    for (int mt = 0; mt < HD / 16; ++mt) {
      o[mt][0] *= a0;
      o[mt][1] *= a1;
      o[mt][2] *= a0;
      o[mt][3] *= a1;
      const int ch = 2 * mt + vchk;
      uint32_t a[4];
      ldmatrix_x4_trans(a[0], a[1], a[2], a[3], vbase + vrow * (HD * 2) + ((ch ^ kv_swz(vrow, RC)) << 4));
      mma_bf16_16816(o[mt], a, bh0, bh1);
      mma_bf16_16816(o[mt], a, bl0, bl1);
    }
    __syncwarp();
    const int nx = i + ATTN_STAGES;
    if (nx < n_my) {  // warp-uniform
      if ((nx & 31) == 0) my_pages = bt_batch(nx >> 5);
      const int pg = __shfl_sync(0xffffffffu, my_pages, nx & 31);
      if (lane == 0) {
        fence_proxy_async_smem();
        issue(nx, pg);
      }
    }
  }
  // the row sums: reduce over the lanes holding the other tokens of each head
#pragma unroll
  for (int x = 4; x < 32; x <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, x);
    l1 += __shfl_xor_sync(0xffffffffu, l1, x);
  }

  // ---- merge the 4 warps through shared memory (stage buffers are idle now)
  __syncthreads();
  float* sO = reinterpret_cast<float*>(smem);                 // [4][16][HD] (rows = heads)
  float* sM = sO + ATTN_WARPS * 16 * HD;                       // [4][16]
  float* sL = sM + ATTN_WARPS * 16;                            // [4][16]
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) {
    const int e0 = 16 * mt + hq;
    sO[(warp * 16 + cq) * HD + e0] = o[mt][0];
    sO[(warp * 16 + cq + 1) * HD + e0] = o[mt][1];
    sO[(warp * 16 + cq) * HD + e0 + 8] = o[mt][2];
    sO[(warp * 16 + cq + 1) * HD + e0 + 8] = o[mt][3];
  }
  if (lane < 4) {
    sM[warp * 16 + cq] = m0;
    sM[warp * 16 + cq + 1] = m1;
    sL[warp * 16 + cq] = l0;
    sL[warp * 16 + cq + 1] = l1;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < g * HD; idx += blockDim.x) {
    const int r = idx / HD, e = idx % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < ATTN_WARPS; ++w) M = fmaxf(M, sM[w * 16 + r]);
    float so = 0.f, sl = 0.f;
#pragma unroll
    for (int w = 0; w < ATTN_WARPS; ++w) {
      const float f = exp2f(sM[w * 16 + r] - M);  // empty warps: 2^-inf = 0
      so += f * sO[(w * 16 + r) * HD + e];
      sl += f * sL[w * 16 + r];
    }
    if (it.part < 0) {
      const size_t oi = ((size_t)it.row * nq + (size_t)it.kvh * g + r) * HD + e;
      const float v = so / sl;
      if (out_fp32)
        reinterpret_cast<float*>(out)[oi] = v;
      else
        reinterpret_cast<__nv_bfloat16*>(out)[oi] = __float2bfloat16_rn(v);
    } else {
      part_o[((size_t)it.part * g + r) * HD + e] = so;
      if (e == 0) {
        part_ml[((size_t)it.part * g + r) * 2 + 0] = M;
        part_ml[((size_t)it.part * g + r) * 2 + 1] = sl;
      }
    }
  }
  if (it.part >= 0) {
    // split item: the last of the (row, kv head)'s parts to arrive merges them
    // (threadfence reduction; the counter re-arms itself for the next launch)
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&arrive[it.comb], 1) == combs[it.comb].nparts - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      combine_merge(combs[it.comb], nq, nkv, HD, part_o, part_ml, out, out_fp32);
      if (threadIdx.x == 0) arrive[it.comb] = 0;
    }
  }
}

// LSE merge of the split-K partials of one (row, kv head): the per-part
// weights 2^(m_j - M) and the denominator are computed once per row into
// shared memory (one warp per query row), then every output element sums its
// column over the parts with independent, coalesced (L2) loads.
__device__ __forceinline__ void combine_merge(const AttnComb& c, int nq, int nkv, int hd,
                                              const float* __restrict__ part_o, const float* __restrict__ part_ml,
                                              void* __restrict__ out, int out_fp32) {
  __shared__ float w[16][ATTN_MAX_PARTS];
  __shared__ float inv_l[16];
  const int g = nq / nkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < g; r += blockDim.x >> 5) {
    float m[2], l[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int j = lane + 32 * k;
      const bool ok = j < c.nparts;
      const size_t pj = ((size_t)(c.part0 + (ok ? j : 0)) * g + r) * 2;
      m[k] = ok ? __ldcg(part_ml + pj) : -INFINITY;
      l[k] = ok ? __ldcg(part_ml + pj + 1) : 0.f;
    }
    const float M = warp_max(fmaxf(m[0], m[1]));
    float L = 0.f;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int j = lane + 32 * k;
      const float f = j < c.nparts ? exp2f(m[k] - M) : 0.f;
      if (j < ATTN_MAX_PARTS) w[r][j] = f;
      L += f * l[k];
    }
    L = warp_sum(L);
    if (lane == 0) inv_l[r] = 1.f / L;
  }
  __syncthreads();
  // Every thread owns float4 columns v and v + blockDim.x of the [g][hd] block
  // and keeps 2 x 8 partial loads in flight per batch: the merge costs about
  // ceil(nparts / 8) L2 round trips instead of one per part and element.
  const int nvec = g * hd / 4;
  const size_t stride = (size_t)nvec;  // float4s per part
  const float4* base = reinterpret_cast<const float4*>(part_o + (size_t)c.part0 * g * hd);
  for (int v0 = threadIdx.x; v0 < nvec; v0 += 2 * blockDim.x) {
    const int v1 = v0 + blockDim.x;
    const bool has1 = v1 < nvec;
    const int r0 = (4 * v0) / hd, r1 = has1 ? (4 * v1) / hd : r0;
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
    for (int j = 0; j < c.nparts; j += 8) {
      float4 x0[8], x1[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const bool ok = j + k < c.nparts;
        x0[k] = ok ? __ldcg(base + (size_t)(j + k) * stride + v0) : make_float4(0.f, 0.f, 0.f, 0.f);
        x1[k] = ok && has1 ? __ldcg(base + (size_t)(j + k) * stride + v1) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (j + k < c.nparts) {
          const float w0 = w[r0][j + k], w1 = w[r1][j + k];
          a0.x += w0 * x0[k].x, a0.y += w0 * x0[k].y, a0.z += w0 * x0[k].z, a0.w += w0 * x0[k].w;
          a1.x += w1 * x1[k].x, a1.y += w1 * x1[k].y, a1.z += w1 * x1[k].z, a1.w += w1 * x1[k].w;
        }
      }
    }
    auto store = [&](int v, int r, float4 a) {
      const int e = 4 * v - r * hd;
      const float il = inv_l[r];
      const size_t oi = ((size_t)c.row * nq + (size_t)c.kvh * g + r) * hd + e;
      if (out_fp32) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + oi) =
            make_float4(a.x * il, a.y * il, a.z * il, a.w * il);
      } else {
        uint2 o;
        o.x = pack_bf16x2(a.x * il, a.y * il);
        o.y = pack_bf16x2(a.z * il, a.w * il);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + oi) = o;
      }
    };
    store(v0, r0, a0);
    if (has1) store(v1, r1, a1);
  }
}

// ------------------------------------------------------------------ host side
void attn_plan(const int32_t* ctx, const int32_t* slot, int b, int nkv, int page, int split_pages, AttnPlan* plan) {
  plan->items.clear();
  plan->combs.clear();
  plan->n_parts = 0;
  int64_t total = 0;
  for (int i = 0; i < b; ++i) total += (int64_t)((ctx[i] + page - 1) / page) * nkv;
  // One wave of 2 CTAs per SM (296 slots): a (row, kv head) with np pages
  // gets floor(296 np / total) parts, so the items never spill into a second,
  // nearly empty wave; parts keep >= 4 pages per warp (measured: 8 pages per part ->
  // 16 saves ~1% of T(b) at b <= 16, profiles/r02/attn_planner) and there are at most
  // ATTN_SPLIT_CAP of them (the last-arriving CTA merges them serially).
  // SGS_ATTN_SLOTS / SGS_ATTN_MINPG: planner experiments (tools/attn_sweep.py)
  static const int64_t kSlots = std::getenv("SGS_ATTN_SLOTS") ? std::atoll(std::getenv("SGS_ATTN_SLOTS")) : 2 * 148;
  static const int kMinPg = std::getenv("SGS_ATTN_MINPG") ? std::atoi(std::getenv("SGS_ATTN_MINPG")) : 4 * ATTN_WARPS;
  constexpr int ATTN_SPLIT_CAP = 32;
  auto cap = [&](int np, int nch) {
    const int by_pages = np / kMinPg;
    if (nch > by_pages) nch = by_pages;
    if (nch > ATTN_SPLIT_CAP) nch = ATTN_SPLIT_CAP;
    return nch < 1 ? 1 : nch;
  };
  // parts per row: floor(slots * np / total), then the slots the floors leave
  // empty go to the rows with the largest remainders (one part each), so a
  // one-wave plan uses the whole wave
  std::vector<int> nparts(b, 0);
  {
    std::vector<std::pair<int64_t, int>> rem;
    int64_t used = 0;
    for (int i = 0; i < b; ++i) {
      const int np = (ctx[i] + page - 1) / page;
      if (np == 0) continue;
      const int64_t q = kSlots * np * nkv;  // this row's share of the slots, times total
      nparts[i] = cap(np, (int)(q / total / nkv));
      used += (int64_t)nparts[i] * nkv;
      rem.push_back({(q / nkv) % total, i});
    }
    if (used < kSlots && split_pages <= 0) {
      std::stable_sort(rem.begin(), rem.end(), [](const std::pair<int64_t, int>& a, const std::pair<int64_t, int>& c) {
        return a.first > c.first;
      });
      for (const auto& r : rem) {
        const int i = r.second, np = (ctx[i] + page - 1) / page;
        if (used + nkv > kSlots) break;
        const int n2 = cap(np, nparts[i] + 1);
        if (n2 > nparts[i]) used += (int64_t)(n2 - nparts[i]) * nkv, nparts[i] = n2;
      }
    }
  }
  for (int i = 0; i < b; ++i) {
    const int np = (ctx[i] + page - 1) / page;
    if (np == 0) continue;
    int nch;
    if (split_pages > 0) {
      nch = (np + split_pages - 1) / split_pages;
      if (nch > ATTN_MAX_PARTS) nch = ATTN_MAX_PARTS;
    } else {
      nch = nparts[i];
    }
    for (int h = 0; h < nkv; ++h) {
      if (nch == 1) {
        plan->items.push_back(AttnItem{i, h, 0, np, -1, -1, slot ? slot[i] : i, ctx[i]});
        continue;
      }
      const int part0 = plan->n_parts;
      for (int c = 0; c < nch; ++c) {
        const int p0 = (int)((int64_t)np * c / nch), p1 = (int)((int64_t)np * (c + 1) / nch);
        plan->items.push_back(
            AttnItem{i, h, p0, p1, plan->n_parts++, (int32_t)plan->combs.size(), slot ? slot[i] : i, ctx[i]});
      }
      plan->combs.push_back(AttnComb{i, h, part0, nch});
    }
  }
  // longest items first (tail balance)
  std::stable_sort(plan->items.begin(), plan->items.end(),
                   [](const AttnItem& a, const AttnItem& c) { return (a.p1 - a.p0) > (c.p1 - c.p0); });
}

int64_t attn_workspace_bytes(int max_items, int max_parts, int g, int hd) {
  // items + combs (op path) | part_o | part_ml | arrival counters
  return (int64_t)max_items * sizeof(AttnItem) + (int64_t)max_items * sizeof(AttnComb) +
         (int64_t)max_parts * g * (hd + 2) * sizeof(float) + (int64_t)max_items * sizeof(int) + 2048;
}

template <int HD>
static cudaError_t launch_decode(const void* q, const void* kv, const int32_t* bt, const AttnItem* items,
                                 int n_items, const int32_t* counts,
                                 int nq, int nkv, int max_pages, void* out, int out_fp32, float* part_o,
                                 float* part_ml, const AttnComb* combs, int* arrive, cudaStream_t stream) {
  constexpr int STAGE = 2 * PAGE_T * HD * 2;
  const size_t ring = (size_t)ATTN_WARPS * ATTN_STAGES * STAGE;
  const size_t merge = (size_t)ATTN_WARPS * 16 * (HD + 2) * sizeof(float);
  const size_t smem = ring > merge ? ring : merge;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(attn_decode_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    set = true;
  }
  const float scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)HD));
  return launch_pdl(attn_decode_kernel<HD>, dim3(n_items), dim3(128), smem, stream,
                    reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(kv), bt,
                    items, n_items, counts, nq, nkv, max_pages, scale_log2, out, out_fp32, part_o, part_ml,
                    combs, arrive);
}

cudaError_t attn_decode(const void* q, const void* kv, const int32_t* bt, const int32_t* counts,
                        const AttnItem* items, int n_items, const AttnComb* combs, int n_combs,
                        int nq, int nkv, int hd, int page, int max_pages, void* out, int out_fp32, float* part_o,
                        float* part_ml, int* arrive, cudaStream_t stream) {
  (void)n_combs;
  if (page != PAGE_T) return cudaErrorInvalidValue;
  if (nq % nkv != 0 || nq / nkv > 8) return cudaErrorInvalidValue;  // the g query heads are the MMA's N = 8
  if (n_items <= 0) return cudaSuccess;
  switch (hd) {
    case 32:
      return launch_decode<32>(q, kv, bt, items, n_items, counts, nq, nkv, max_pages, out, out_fp32,
                               part_o, part_ml, combs, arrive, stream);
    case 64:
      return launch_decode<64>(q, kv, bt, items, n_items, counts, nq, nkv, max_pages, out, out_fp32,
                               part_o, part_ml, combs, arrive, stream);
    case 128:
      return launch_decode<128>(q, kv, bt, items, n_items, counts, nq, nkv, max_pages, out, out_fp32,
                                part_o, part_ml, combs, arrive, stream);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace sgs
