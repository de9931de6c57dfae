// K3/K4: bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   C[t, n] (+)= sum_k X[t, k] * W[n, k]        (the projections / MLP / LM head,
//                                               SURVEY §8a rows a7, a9-a12)
//
// Swap-AB: the weight tile (128 output features x 64 K) is the UMMA "A"
// operand (M = 128) and the token tile (BN tokens x 64 K) is "B" (N = BN,
// 16..256), so the same kernel serves decode (b <= 256 tokens: weight
// streaming, one N tile, HBM bound) and prefill (thousands of tokens,
// tensor bound).  Accumulators live in TMEM; one elected thread issues TMA
// loads into a multi-stage shared-memory ring, one elected thread issues
// tcgen05.mma, four epilogue warps read TMEM (tcgen05.ld) and write fp32
// rows of C (coalesced: lane = output feature).  Split-K over gridDim.z with
// fp32 red.add when mode == 1.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "kernels.h"

namespace sgs {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;  // one 128-byte swizzle atom of bf16
constexpr int GEMM_A_BYTES = GEMM_BM * GEMM_BK * 2;
constexpr int GEMM_SMEM_BUDGET = 200 * 1024;
constexpr int GEMM_GROUP = 16;  // weight tiles (pairs) per rasterisation group

// CG = 1: one CTA per 128-row weight tile.  CG = 2: a CTA pair (cluster of
// 2) computes a 256-row tile with tcgen05.mma.cta_group::2: each CTA stages
// its 128 weight rows and half of the token tile, the leader issues the MMAs,
// and the accumulator rows land in each CTA's own TMEM.  Per SM this halves
// the token-tile shared-memory and L2 traffic of the 1-CTA kernel.
//
// Persistent: a CTA (pair) walks the work units u = blockIdx/CG, +grid/CG, ...
// (unit = weight tile x token tile x K split, grouped rasterisation).  The
// shared-memory ring runs continuously across units, and with nbuf = 2 the
// TMEM accumulator is double-buffered so the epilogue of unit i overlaps the
// MMAs of unit i+1 (tmem_full / tmem_empty barrier pair per buffer).
// One instantiation per (CG, epilogue MODE, k-chunks per stage KCS): each
// kernel carries only its own producer and epilogue code, which keeps it
// under the ~40 KB instruction-cache knee (a 46 KB all-modes kernel measured
// 14% slower on decode-sized GEMMs).
// ---- fused RMSNorm pre-phase (PreNorm) helpers
__device__ __forceinline__ uint32_t ld_acquire_u32(const unsigned int* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// epilogue warps (128 threads, e = warp - 4): X rows of this CTA, then one arrival
__device__ __forceinline__ void prenorm_rows(const PreNorm& pn, __nv_bfloat16* __restrict__ X, int T, int d, int e,
                                             int lane, double* red) {
  const int tid = e * 32 + lane;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const float* hr = pn.h + (size_t)t * d;
    double ss = 0.0;
    for (int i = 4 * tid; i < d; i += 512) {
      const float4 v = *reinterpret_cast<const float4*>(hr + i);
      ss += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[e] = ss;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const double r = 1.0 / sqrt((red[0] + red[1] + red[2] + red[3]) / (double)d + (double)pn.eps);
    asm volatile("bar.sync 1, 128;" ::: "memory");  // red[] is reused by the next row
    const uint32_t* w = reinterpret_cast<const uint32_t*>(pn.w);
    for (int i = 4 * tid; i < d; i += 512) {
      const float4 v = *reinterpret_cast<const float4*>(hr + i);
      const uint32_t w0 = w[i >> 1], w1 = w[(i >> 1) + 1];
      auto f = [&](float x, uint32_t wbits) { return (float)((double)x * r * (double)__uint_as_float(wbits)); };
      uint2 o;
      o.x = pack_bf16x2(f(v.x, w0 << 16), f(v.y, w0 & 0xffff0000u));
      o.y = pack_bf16x2(f(v.z, w1 << 16), f(v.w, w1 & 0xffff0000u));
      *reinterpret_cast<uint2*>(X + (size_t)t * d + i) = o;
    }
  }
  fence_proxy_async_global();  // X is read by other CTAs' TMA (async proxy)
  __threadfence();
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (tid == 0) {
    const int p = *pn.parity & 1;
    unsigned int* cnt = pn.bar + 2 * pn.site + p;
    if (atomicAdd(cnt, 1u) == gridDim.x - 1) pn.bar[2 * pn.site + (p ^ 1)] = 0u;  // re-arm the other parity
  }
}
// the activation producer: wait until every CTA wrote its X rows
__device__ __forceinline__ void prenorm_wait(const PreNorm& pn) {
  const unsigned int* cnt = pn.bar + 2 * pn.site + (*pn.parity & 1);
  while (ld_acquire_u32(cnt) < gridDim.x) __nanosleep(32);
  fence_proxy_async_global();
}

// <= 128 registers per thread: two decode-tile CTAs (and their PreNorm grid
// barrier) must be co-resident on an SM
template <int CG, int MODE, int KCS>
__global__ void __launch_bounds__(256, 2)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                        float* __restrict__ C, int T, int ldc, int BN, int stages, int k_chunks_total,
                        int chunks_per_split, int tmem_cols, int n_acc, int acc_stride, int num_mp, int num_n,
                        int units, int nbuf, int xbufs, const ArgmaxArgs am, const PreNorm pn, int K,
                        int w_tiled) {
  constexpr int mode = MODE, kcs = KCS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int bl = BN / CG;  // token rows staged by this CTA
  const int b_bytes = bl * GEMM_BK * 2;  // one k-chunk of the token tile
  // a stage holds kcs consecutive k-chunks of each operand (one 3-D TMA box)
  const int a_stage = kcs * GEMM_A_BYTES, b_stage = kcs * b_bytes;
  uint8_t* sA = smem;
  uint8_t* sB = smem + (size_t)stages * a_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)stages * b_stage);
  uint64_t* empty = full + stages;
  uint64_t* tmem_full = empty + stages;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  // 2 x [4 warps][32][17]: per-warp transpose (features x tokens -> tokens x
  // feature quads) for the vectorised epilogue; both halves serve as the
  // double-buffered SwiGLU exchange (mode 3); rows 0..63 double as the
  // SwiGLU exchange (mode 3)
  float* xch = reinterpret_cast<float*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int pair = blockIdx.x / CG, npairs = gridDim.x / CG;
  const uint32_t buf_stride = nbuf == 2 ? (uint32_t)tmem_cols / 2 : 0u;

  // unit -> (m0, n0, first k chunk, k chunks).  Grouped rasterisation:
  // consecutive units walk GEMM_GROUP weight tiles (pairs) of one token tile,
  // then the same weight tiles for the next token tile, so concurrently
  // running units share weight tiles through L2.
  auto coords = [&](int u, int& m0, int& n0, int& kc0, int& nk) {
    const int per_split = num_mp * num_n;
    const int sp = u / per_split, r = u - sp * per_split;
    const int per_group = GEMM_GROUP * num_n;
    const int first = (r / per_group) * GEMM_GROUP;
    const int gsize = min(num_mp - first, GEMM_GROUP);
    const int mt = first + (r % per_group) % gsize;
    const int nt = (r % per_group) / gsize;
    m0 = (mt * CG + (int)rank) * GEMM_BM;
    n0 = nt * BN;
    kc0 = sp * chunks_per_split;
    nk = min(kc0 + chunks_per_split, k_chunks_total) - kc0;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], kcs > 1 ? 2 : 1);  // split producers: the weight and the activation thread each arrive
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 4 * CG);  // one arrival per epilogue warp of the pair
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    if (CG == 2)
      tmem_alloc_2sm(tmem_slot, tmem_cols);
    else
      tmem_alloc(tmem_slot, tmem_cols);
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();  // the peer's barriers exist before any cross-CTA arrival
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  pdl_trigger();
  if (kcs == 1 && warp == 0 && lane == 0) {
    // ---------------- TMA producer, decode-sized tiles: one thread, 2-D boxes
    // (both CTAs; the leader's barrier counts both CTAs' bytes).  The weight
    // tiles do not depend on the previous kernel: the ring is filled with
    // them before griddepcontrol.wait (overlapping the predecessor's tail),
    // then the activation tiles follow.
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmX);
    const uint32_t tx = (uint32_t)CG * (GEMM_A_BYTES + b_bytes);
    int it = 0;  // position in the ring, continuous across units
    for (int u = pair; u < units; u += npairs) {
      int m0, n0, kc0, nk;
      coords(u, m0, n0, kc0, nk);
      auto load_a = [&](int s, int i) {
        if (w_tiled) {  // one contiguous 16 KB block of the tiled weights
          if (CG == 2)
            tma_load_4d_2sm(sA + (size_t)s * GEMM_A_BYTES, &tmW, kc0 + i, m0 / GEMM_BM, &full[s]);
          else
            tma_load_4d(sA + (size_t)s * GEMM_A_BYTES, &tmW, kc0 + i, m0 / GEMM_BM, &full[s]);
        } else if (CG == 2) {
          tma_load_2d_2sm(sA + (size_t)s * GEMM_A_BYTES, &tmW, (kc0 + i) * GEMM_BK, m0, &full[s]);
        } else {
          tma_load_2d(sA + (size_t)s * GEMM_A_BYTES, &tmW, (kc0 + i) * GEMM_BK, m0, &full[s]);
        }
      };
      auto load_b = [&](int s, int i) {
        if (CG == 2)
          tma_load_2d_2sm(sB + (size_t)s * b_bytes, &tmX, (kc0 + i) * GEMM_BK, n0 + (int)rank * bl, &full[s]);
        else
          tma_load_2d(sB + (size_t)s * b_bytes, &tmX, (kc0 + i) * GEMM_BK, n0, &full[s]);
      };
      int i0 = 0;
      if (u == pair) {
        const int pre = nk < stages ? nk : stages;
        for (int i = 0; i < pre; ++i) {
          if (leader) mbar_expect_tx(&full[i], tx);
          load_a(i, i);
        }
        pdl_wait();
        if (pn.h) prenorm_wait(pn);
        for (int i = 0; i < pre; ++i) load_b(i, i);
        i0 = pre;
        it = pre;
      }
      for (int i = i0; i < nk; ++i, ++it) {
        const int s = it % stages;
        if (it >= stages) mbar_wait(&empty[s], ((it / stages) - 1) & 1);
        if (leader) mbar_expect_tx(&full[s], tx);
        load_a(s, i);
        load_b(s, i);
      }
    }
  } else if (kcs > 1 && (warp == 0 || warp == 3) && lane == 0) {
    // ---------------- TMA producers, compute-bound tiles (both CTAs): warp 0
    // streams the weight tiles, warp 3 the activation tiles, one 3-D box of
    // kcs k-chunks per stage each (fewer, larger requests).  The leader's
    // full barrier counts both producers and both CTAs' bytes.  The weights
    // do not depend on the previous kernel, so warp 0 never waits for it.
    const bool is_w = warp == 0;
    const CUtensorMap* tm = is_w ? &tmW : &tmX;
    prefetch_tmap(tm);
    if (!is_w) {
      pdl_wait();
      if (pn.h) prenorm_wait(pn);
    }
    const uint32_t tx = (uint32_t)CG * (is_w ? a_stage : b_stage);
    uint8_t* base = is_w ? sA : sB;
    const int sbytes = is_w ? a_stage : b_stage;
    int it = 0;  // position in the ring, continuous across units
    for (int u = pair; u < units; u += npairs) {
      int m0, n0, kc0, nk;
      coords(u, m0, n0, kc0, nk);
      const int row = is_w ? m0 : n0 + (int)rank * bl;
      for (int i = 0; i < nk; i += kcs, ++it) {
        const int s = it % stages;
        if (it >= stages) mbar_wait(&empty[s], ((it / stages) - 1) & 1);
        if (leader) mbar_expect_tx(&full[s], tx);
        if (is_w && w_tiled) {
          if (CG == 2)
            tma_load_4d_2sm(base + (size_t)s * sbytes, tm, kc0 + i, row / GEMM_BM, &full[s]);
          else
            tma_load_4d(base + (size_t)s * sbytes, tm, kc0 + i, row / GEMM_BM, &full[s]);
        } else if (CG == 2) {
          tma_load_3d_2sm(base + (size_t)s * sbytes, tm, row, (kc0 + i), &full[s]);
        } else {
          tma_load_3d(base + (size_t)s * sbytes, tm, row, (kc0 + i), &full[s]);
        }
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ---------------- MMA issuer (single thread of the leader CTA)
    const uint32_t idesc = umma_idesc_bf16(GEMM_BM * CG, BN);
    int it = 0, tc = 0;
    for (int u = pair; u < units; u += npairs, ++tc) {
      int m0, n0, kc0, nk;
      coords(u, m0, n0, kc0, nk);
      const int buf = nbuf == 2 ? (tc & 1) : 0, use = nbuf == 2 ? (tc >> 1) : tc;
      if (use > 0) {  // the epilogue of this buffer's previous unit has drained it
        mbar_wait(&tmem_empty[buf], (use - 1) & 1);
        tc_fence_after();
      }
      const uint32_t base = tmem + (uint32_t)buf * buf_stride;
      for (int i = 0; i < nk; i += kcs, ++it) {
        const int s = it % stages;
        mbar_wait(&full[s], (it / stages) & 1);
        tc_fence_after();
        for (int kk = 0; kk < kcs; ++kk) {
          const int ci = i + kk;  // k-chunk index within the unit
          const uint64_t ad = umma_desc_sw128(smem_u32(sA + (size_t)s * a_stage + (size_t)kk * GEMM_A_BYTES));
          const uint64_t bd = umma_desc_sw128(smem_u32(sB + (size_t)s * b_stage + (size_t)kk * b_bytes));
          // k-chunk ci accumulates into TMEM accumulator ci % n_acc: the
          // tensor-core fp32 accumulation truncates, so short chains + an IEEE
          // fp32 sum of the accumulators in the epilogue keep the error at
          // fp32-GEMM level.
          const uint32_t d = base + (uint32_t)((ci % n_acc) * acc_stride);
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {  // K = 16 per MMA: advance 32 B inside the swizzle atom
            if (CG == 2)
              umma_bf16_2sm(d, ad + 2 * k, bd + 2 * k, idesc, (ci >= n_acc || k > 0) ? 1u : 0u);
            else
              umma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (ci >= n_acc || k > 0) ? 1u : 0u);
          }
        }
        if (CG == 2)
          umma_commit_2sm(&empty[s]);
        else
          umma_commit(&empty[s]);
      }
      if (CG == 2)
        umma_commit_2sm(&tmem_full[buf]);
      else
        umma_commit(&tmem_full[buf]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> global (lane = output feature)
    const int e = warp - 4;
    pdl_wait();  // C may still be read by the predecessor (write-after-read)
    if (pn.h) {
      double* red = reinterpret_cast<double*>(xch + (size_t)xbufs * 4 * 32 * 17 + 128);  // past the mode-4 keys
      prenorm_rows(pn, reinterpret_cast<__nv_bfloat16*>(pn.x), T, K, e, lane, red);
    }
    int tc = 0;
    for (int u = pair; u < units; u += npairs, ++tc) {
      int m0, n0, kc0, nk;
      coords(u, m0, n0, kc0, nk);
      const int buf = nbuf == 2 ? (tc & 1) : 0, use = nbuf == 2 ? (tc >> 1) : tc;
      mbar_wait(&tmem_full[buf], use & 1);
      tc_fence_after();
      const uint32_t base = tmem + (uint32_t)buf * buf_stride + ((uint32_t)(32 * e) << 16);
      const int used = nk < n_acc ? nk : n_acc;
      for (int c = 0; c < BN; c += 16) {
        float acc[16];
        {
          uint32_t r[16];
          tmem_ld16(base + (uint32_t)c, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = __uint_as_float(r[j]);
        }
        for (int a = 1; a < used; ++a) {
          uint32_t r[16];
          tmem_ld16(base + (uint32_t)(a * acc_stride + c), r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] += __uint_as_float(r[j]);
        }
        if (mode == 4) {
          // fused greedy sampling: per token, the (value desc, vocab index asc)
          // maximum over this warp's 32 rows, then over the 4 epilogue warps
          // (shared memory), then one 64-bit atomicMax per token and tile
          const int feat = am.vocab_off + m0 + 32 * e + lane;
          // [4][16] keys, after the exchange buffers (the store path below reuses those)
          unsigned long long* sk = reinterpret_cast<unsigned long long*>(xch + (size_t)xbufs * 4 * 32 * 17);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const uint32_t u = __float_as_uint(acc[j]);
            const uint32_t ord = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
            unsigned long long key = ((unsigned long long)ord << 32) | (uint32_t)(~(uint32_t)feat);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
              key = ok > key ? ok : key;
            }
            if (lane == j) sk[e * 16 + j] = key;
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (e == 0 && lane < 16 && n0 + c + lane < T) {
            unsigned long long k = sk[lane];
#pragma unroll
            for (int w = 1; w < 4; ++w) k = sk[w * 16 + lane] > k ? sk[w * 16 + lane] : k;
            atomicMax(am.keys + n0 + c + lane, k);
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (C == nullptr) continue;
        }
        if (mode == 3) {
          // fused SwiGLU: tile rows 0..63 are gate rows and 64..127 the up rows
          // of the same 64 features (warps 0-1: g, warps 2-3: u).  All four
          // warps publish their 16 tokens to shared memory (double-buffered
          // by chunk parity when xbufs == 2: one barrier per chunk); warp w
          // then writes m = bf16(SiLU(g) * u) for features 32 (w & 1) + lane
          // and tokens 8 (w >> 1) + 0..7 (lane = feature: 64-byte stores).
          __nv_bfloat16* M = reinterpret_cast<__nv_bfloat16*>(C);
          float* xb = xch + (size_t)((c >> 4) & (xbufs - 1)) * (4 * 32 * 17);
#pragma unroll
          for (int j = 0; j < 16; ++j) xb[(e * 32 + lane) * 17 + j] = acc[j];
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const int fg = e & 1, th = e >> 1;
          const int feat = (m0 >> 1) + 32 * fg + lane;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int j = 8 * th + k, t = n0 + c + j;
            const float g = xb[(fg * 32 + lane) * 17 + j], uu = xb[((2 + fg) * 32 + lane) * 17 + j];
            if (t < T) M[(size_t)t * ldc + feat] = __float2bfloat16_rn(g / (1.f + expf(-g)) * uu);
          }
          if (xbufs == 1) asm volatile("bar.sync 1, 128;" ::: "memory");  // single buffer: drain before reuse
          continue;
        }
        // transpose through shared memory so each thread owns 4 consecutive
        // features of one token: 16-byte stores / red.global.add.v4.f32
        // (a quarter of the scalar atomics of split-K)
        float* xt = xch + (size_t)e * 32 * 17;
#pragma unroll
        for (int j = 0; j < 16; ++j) xt[lane * 17 + j] = acc[j];
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int item = lane + 32 * it, j = item >> 3, qd = item & 7;
          const int t = n0 + c + j;
          if (t < T) {
            float4 v;
            v.x = xt[(4 * qd + 0) * 17 + j], v.y = xt[(4 * qd + 1) * 17 + j];
            v.z = xt[(4 * qd + 2) * 17 + j], v.w = xt[(4 * qd + 3) * 17 + j];
            float* p = C + (size_t)t * ldc + m0 + 32 * e + 4 * qd;
            if (mode == 0 || mode == 4) {
              *reinterpret_cast<float4*>(p) = v;
            } else if (mode == 1) {
              red_add_v4(p, v);
            } else {
              float4 o = *reinterpret_cast<float4*>(p);
              o.x += v.x, o.y += v.y, o.z += v.z, o.w += v.w;
              *reinterpret_cast<float4*>(p) = o;
            }
          }
        }
        __syncwarp();
      }
      // hand the accumulator buffer back to the MMA issuer (leader CTA)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2)
          mbar_arrive_cluster(&tmem_empty[buf], 0);
        else
          mbar_arrive(&tmem_empty[buf]);
      }
    }
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();  // the leader's MMAs read the peer's shared memory until tmem_full
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2)
      tmem_dealloc_2sm(tmem, tmem_cols);
    else
      tmem_dealloc(tmem, tmem_cols);
  }
  if (mode == 4 && am.finalize) {
    // the last CTA to arrive turns the packed keys into tokens (all atomics of
    // every CTA precede its fenced arrival)
    // (no static shared memory in this kernel: the dynamic allocation takes the
    // full 227 KB; tmem_slot[2] is a free word of the dynamic area)
    volatile uint32_t* s_last = tmem_slot + 2;
    if (threadIdx.x == 0) {
      __threadfence();
      *s_last = atomicAdd(am.done, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (*s_last) {
      __threadfence();
      for (int t = threadIdx.x; t < T; t += blockDim.x) {
        const unsigned long long k = atomicExch(am.keys + t, 0ull);
        const int s = am.slot[t];
        if (s >= 0) {
          const int32_t tok = (int32_t)(~(uint32_t)k);
          am.last_tok[s] = tok;
          am.hist[(size_t)s * am.max_gen + am.tok_idx[t]] = tok;
        }
      }
      if (threadIdx.x == 0) *am.done = 0u;
    }
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// Row-major bf16 [rows, cols] matrix viewed as (64, rows, cols/64) with
// strides (2 cols, row pitch, 128 B): box (64, box_rows, kc) = kc consecutive
// k-chunks of box_rows rows, 128-byte swizzle.
static bool make_tmap(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int box_rows, int kc,
                      int tiled = 0) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  if (tiled) {
    // tiled weights [rows/128][cols/64][128][64] (the engine's layout)
    // viewed as (64, 128, cols/64, rows/128): box (64, 128, kc, 1) is kc
    // consecutive 16 KB blocks of global memory, the same shared-memory image
    // as the row-major box
    if (box_rows != 128 || rows % 128 || cols % GEMM_BK) return false;
    cuuint64_t dims[4] = {(cuuint64_t)GEMM_BK, 128, (cuuint64_t)(cols / GEMM_BK), (cuuint64_t)(rows / 128)};
    cuuint64_t strides[3] = {(cuuint64_t)GEMM_BK * 2, (cuuint64_t)128 * GEMM_BK * 2,
                             (cuuint64_t)(cols / GEMM_BK) * 128 * GEMM_BK * 2};
    cuuint32_t box[4] = {(cuuint32_t)GEMM_BK, 128, (cuuint32_t)kc, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  if (kc == 1) {  // 2-D [rows, cols], box [box_rows, 64]
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)GEMM_BK, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  cuuint64_t dims[3] = {(cuuint64_t)GEMM_BK, (cuuint64_t)rows, (cuuint64_t)(cols / GEMM_BK)};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)GEMM_BK * 2};
  cuuint32_t box[3] = {(cuuint32_t)GEMM_BK, (cuuint32_t)box_rows, (cuuint32_t)kc};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct TmapKey {
  const void* p;
  int64_t rows, cols;
  int box, kc, tiled;
  bool operator==(const TmapKey& o) const {
    return p == o.p && rows == o.rows && cols == o.cols && box == o.box && kc == o.kc && tiled == o.tiled;
  }
};
struct TmapKeyHash {
  size_t operator()(const TmapKey& k) const {
    return std::hash<const void*>()(k.p) ^ (size_t)(k.rows * 1315423911u) ^ (size_t)(k.cols * 2654435761u) ^
           (size_t)k.box ^ ((size_t)k.kc << 20) ^ ((size_t)k.tiled << 28);
  }
};

static bool cached_tmap(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int box_rows, int kc,
                        int tiled = 0) {
  static std::mutex mu;
  static std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> cache;
  TmapKey k{ptr, rows, cols, box_rows, kc, tiled};
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(k);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  if (!make_tmap(out, ptr, rows, cols, box_rows, kc, tiled)) return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(k, *out);
  return true;
}

// shared with the other tcgen05 kernels (prefill attention)
bool tmap_bf16_rows(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int box_rows, int kc) {
  return cached_tmap(out, ptr, rows, cols, box_rows, kc);
}

static int sm_count() {
  static int n[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

// Split-K factor for launches that would leave the GPU under-filled: the
// units (tiles x splits) fill the resident slots -- 2 CTAs per SM for decode
// tiles (BN <= 128), 1 for the 200 KB compute-bound tiles -- up to 8 splits
// and >= 4 k-chunks per split (tools/split_sweep.py: at T <= 128, 8 splits
// beat 5 by 8-15%; at T = 256 the red.add traffic makes ~148/tiles optimal).
int gemm_auto_splits(int N, int K, int T) {
  const int bn = T >= 256 ? 256 : ((T + 15) / 16) * 16;
  const int tiles = (N / GEMM_BM) * ((T + bn - 1) / bn);
  const int slots = bn <= 128 ? 2 * 148 : 148;
  const int kc = K / GEMM_BK;
  int s = slots / tiles;
  if (s > 8) s = 8;
  const int maxs = kc / 4 > 0 ? kc / 4 : 1;  // keep >= 4 K chunks per split
  if (s > maxs) s = maxs;
  return s < 1 ? 1 : s;
}

template <int CG, int MODE, int KCS>
static int occupancy_of(size_t smem) {
  static std::mutex mu;
  static std::unordered_map<size_t, int> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(smem);
  if (it != cache.end()) return it->second;
  auto kern = gemm_bf16_tc_kernel<CG, MODE, KCS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, 256, smem) != cudaSuccess) n = 0;
  cache.emplace(smem, n);
  return n;
}

static int gemm_occupancy(int cg, int mode, int kcs, size_t smem) {
  switch ((cg - 1) * 10 + mode * 2 + (kcs - 1)) {
#define SGS_OCC_CASE(c, md, kk) \
  case (c - 1) * 10 + md * 2 + (kk - 1): return occupancy_of<c, md, kk>(smem);
    SGS_OCC_CASE(1, 0, 1) SGS_OCC_CASE(1, 0, 2) SGS_OCC_CASE(1, 1, 1) SGS_OCC_CASE(1, 1, 2)
    SGS_OCC_CASE(1, 2, 1) SGS_OCC_CASE(1, 2, 2) SGS_OCC_CASE(1, 3, 1) SGS_OCC_CASE(1, 3, 2)
    SGS_OCC_CASE(1, 4, 1) SGS_OCC_CASE(1, 4, 2)
    SGS_OCC_CASE(2, 0, 1) SGS_OCC_CASE(2, 0, 2) SGS_OCC_CASE(2, 1, 1) SGS_OCC_CASE(2, 1, 2)
    SGS_OCC_CASE(2, 2, 1) SGS_OCC_CASE(2, 2, 2) SGS_OCC_CASE(2, 3, 1) SGS_OCC_CASE(2, 3, 2)
    SGS_OCC_CASE(2, 4, 1) SGS_OCC_CASE(2, 4, 2)
#undef SGS_OCC_CASE
    default:
      return 0;
  }
}

// Launch one instantiation: PDL always, plus a 2-CTA cluster for CG == 2.
template <typename Kern, typename... Args>
static cudaError_t launch_gemm(Kern kern, int cg, dim3 grid, size_t smem, cudaStream_t stream, Args... args) {
  static thread_local std::unordered_map<const void*, bool> attr;  // per instantiation
  bool& done = attr[reinterpret_cast<const void*>(kern)];
  if (!done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    done = true;
  }
  if (cg == 1) return launch_pdl(kern, grid, dim3(256), smem, stream, args...);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

cudaError_t gemm_bf16(const void* W, const void* X, float* C, int N, int K, int T, int ldc, int mode, int splits,
                      cudaStream_t stream, const ArgmaxArgs* am, const PreNorm* pn, int w_tiled) {
  if (T <= 0) return cudaSuccess;
  if (N % GEMM_BM != 0 || K % GEMM_BK != 0) return cudaErrorInvalidValue;
  // SGS_GEMM_BN_CAP (experiments, tools/gemm_explore.py): largest token tile
  static const int bn_cap = std::getenv("SGS_GEMM_BN_CAP") ? std::atoi(std::getenv("SGS_GEMM_BN_CAP")) : 256;
  int BN = std::min(bn_cap, T >= 256 ? 256 : ((T + 15) / 16) * 16);
  // small split-K projections (QKV, O: N*K <= 16.5M) at T >= 256: 128-token
  // tiles (twice the units per split) measured 7-8% faster than 256-token ones
  // (profiles/r02/gemm_explore_*.log: QKV 13.7 vs 14.6 us, O 12.6 vs 13.6 us)
  if (mode == 1 && T >= 256 && (int64_t)N * K <= 4608LL * 3584 && bn_cap >= 256) BN = 128;
  // CTA pairs for compute-bound token tiles (BN >= 128) when the 256-row pair tiles N
  const int CG = (BN >= 128 && N % (2 * GEMM_BM) == 0) ? 2 : 1;
  const int kc = K / GEMM_BK;
  if (splits <= 0) splits = mode == 1 ? gemm_auto_splits(N, K, T) : 1;
  if (splits > 1 && mode != 1) return cudaErrorInvalidValue;
  if (mode == 4 && !am) return cudaErrorInvalidValue;
  const ArgmaxArgs amv = am ? *am : ArgmaxArgs{};
  PreNorm pnv = pn ? *pn : PreNorm{};
  if (pn) {
    if (K % 4 != 0) return cudaErrorInvalidValue;
    pnv.x = const_cast<void*>(X);
  }
  // decode-sized tiles (BN <= 128) use half the shared memory and TMEM so two
  // CTAs fit on an SM: the next tile (or the next GEMM, via PDL) streams its
  // weights while the current one drains
  const bool small = BN <= 128;
  // k-chunks per stage (one 3-D TMA box per operand): 2 for the compute-bound
  // tiles (fewer, larger TMA requests), 1 for decode tiles (deeper ring)
  static const int kcs_env = std::getenv("SGS_GEMM_KCS") ? std::atoi(std::getenv("SGS_GEMM_KCS")) : 2;
  const int kcs = (!small && kc % kcs_env == 0) ? kcs_env : 1;
  int per = (kc + splits - 1) / splits;
  per = (per + kcs - 1) / kcs * kcs;  // every split covers whole stages
  splits = (kc + per - 1) / per;      // every split has >= 1 chunk
  CUtensorMap tw, tx;
  if (!cached_tmap(&tw, W, N, K, GEMM_BM, kcs, w_tiled)) return cudaErrorInvalidValue;
  if (!cached_tmap(&tx, X, T, K, BN / CG, kcs)) return cudaErrorInvalidValue;
  const int stage_bytes = kcs * (GEMM_A_BYTES + (BN / CG) * GEMM_BK * 2);
  // experiment (SGS_GEMM_ONE_CTA=<modes bitmask>): decode tiles of the listed
  // modes with one CTA per SM and the whole shared-memory ring, so a CTA walks
  // several units and streams the next unit's weights during an epilogue
  static const int one_cta_modes = std::getenv("SGS_GEMM_ONE_CTA") ? std::atoi(std::getenv("SGS_GEMM_ONE_CTA")) : 0;
  const bool one_cta = small && CG == 1 && ((one_cta_modes >> mode) & 1) && !pn;
  int stages = (small && !one_cta ? GEMM_SMEM_BUDGET / 2 : GEMM_SMEM_BUDGET) / stage_bytes;
  if (stages > 12) stages = 12;
  const int kst = kc / kcs;  // stages-worth of chunks in the whole K
  if (stages > kst) stages = kst < 2 ? 2 : kst;
  if (C && (ldc % 4 != 0 || (reinterpret_cast<uintptr_t>(C) & 15) != 0)) return cudaErrorInvalidValue;  // float4 epilogue
  // epilogue exchange: double-buffered for compute-bound tiles (mode 3 then
  // needs one barrier per 16-token chunk); decode tiles keep the smem for stages
  const int xbufs = small ? 1 : 2;
  const size_t smem = 1024 + (size_t)stages * stage_bytes + (2 * stages + 4) * 8 + 16 + (size_t)xbufs * 4 * 32 * 17 * 4 +
                      4 * 16 * 8 + 64;  // + mode-4 keys [4][16] + PreNorm reduction [4] (fp64)
  // persistent grid: one CTA (pair) per resident slot, at most one per unit
  const int num_mp = N / GEMM_BM / CG, num_n = (T + BN - 1) / BN;
  const int units = num_mp * num_n * splits;
  int slots = sm_count() * (small && !one_cta ? 2 : 1) / CG;
  if (pn) {
    // a PreNorm grid barrier needs every CTA co-resident: never more CTAs than fit
    const int occ = gemm_occupancy(CG, mode, kcs, smem);
    if (occ <= 0) return cudaErrorInvalidConfiguration;
    if (sm_count() * occ / CG < slots) slots = sm_count() * occ / CG;
  }
  const int pairs = units < slots ? units : slots;
  // double-buffer TMEM when a CTA runs several compute-bound units; decode-
  // sized units (BN <= 64) keep all accumulators for precision (their
  // epilogue is short and the co-resident CTA keeps HBM busy meanwhile)
  const int nbuf = (units > pairs && BN >= 128) ? 2 : 1;
  // accumulator interleave: as many TMEM accumulators as fit (<= 8), each 32-column aligned
  const int budget = small ? 256 : 512;
  const int acc_stride = (BN + 31) / 32 * 32;
  int n_acc = budget / (nbuf * acc_stride);
  if (n_acc > 8) n_acc = 8;
  if (n_acc > per) n_acc = per;
  if (n_acc < 1) n_acc = 1;
  int tmem_cols = 32;
  while (tmem_cols < nbuf * n_acc * acc_stride) tmem_cols <<= 1;
  if (nbuf == 2 && tmem_cols / 2 < n_acc * acc_stride) tmem_cols <<= 1;
  if (tmem_cols > 512) return cudaErrorInvalidValue;
  const dim3 grid(pairs * CG);
  switch ((CG - 1) * 10 + mode * 2 + (kcs - 1)) {
#define SGS_GEMM_CASE(cg, md, kk)                                                                                     \
  case (cg - 1) * 10 + md * 2 + (kk - 1):                                                                           \
    return launch_gemm(gemm_bf16_tc_kernel<cg, md, kk>, cg, grid, smem, stream, tw, tx, C, T, ldc, BN, stages, kc, \
                       per, tmem_cols, n_acc, acc_stride, num_mp, num_n, units, nbuf, xbufs, amv, pnv, K, w_tiled);
    SGS_GEMM_CASE(1, 0, 1) SGS_GEMM_CASE(1, 0, 2) SGS_GEMM_CASE(1, 1, 1) SGS_GEMM_CASE(1, 1, 2)
    SGS_GEMM_CASE(1, 2, 1) SGS_GEMM_CASE(1, 2, 2) SGS_GEMM_CASE(1, 3, 1) SGS_GEMM_CASE(1, 3, 2)
    SGS_GEMM_CASE(1, 4, 1) SGS_GEMM_CASE(1, 4, 2)
    SGS_GEMM_CASE(2, 0, 1) SGS_GEMM_CASE(2, 0, 2) SGS_GEMM_CASE(2, 1, 1) SGS_GEMM_CASE(2, 1, 2)
    SGS_GEMM_CASE(2, 2, 1) SGS_GEMM_CASE(2, 2, 2) SGS_GEMM_CASE(2, 3, 1) SGS_GEMM_CASE(2, 3, 2)
    SGS_GEMM_CASE(2, 4, 1) SGS_GEMM_CASE(2, 4, 2)
#undef SGS_GEMM_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace sgs
