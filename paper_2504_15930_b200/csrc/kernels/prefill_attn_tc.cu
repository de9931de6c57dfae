// a4 / K10 on the 5th-generation tensor cores: causal prefill attention of the
// admitted prompts (the prompt tokens "establish the KV cache", P:303-306,
// §2.1), head_dim 128.
//
//   o_i = sum_{j <= i} softmax_j(q_i . k_j / sqrt(hd)) v_j        per prompt, per query head
//
// One CTA = (prompt, 128-query block, query head); KV tiles of 128 keys up to
// the causal diagonal.  tcgen05/TMEM/TMA flash attention:
//   warp 0      TMA producer: Q once, K and V tiles double-buffered (3-D boxes
//               of two 64-column chunks, 128-byte swizzle)
//   warp 1      MMA issuer (one elected thread): S_j = Q K_j^T (bf16, fp32 in
//               TMEM, two S buffers so S_{j+1} overlaps the softmax of S_j),
//               then O += P_j V_j (fp16, fp32 accumulator in TMEM)
//   warps 2-5   softmax: thread = query row = TMEM lane; tcgen05.ld of its S
//               row, causal/prompt mask, online max in the exp2 domain, the O
//               rescale in TMEM (tcgen05.ld/st) when the max moves, P = 2^(s -
//               m) as fp16 into shared memory (K-major, swizzled), then the
//               final O / l as bf16.
// Numerics: V arrives as fp16(bf16 v) (exact); P is split P_hi + P_lo in fp16
// (two MMAs, ~22 significant bits, as the mma.sync kernel does), so P.V keeps
// the fp32 softmax weights' precision (a single fp16 P moved a 1-layer 7B-width
// logit by 0.021 against the fp64 oracle; tolerance 2e-2).
// V is the MN-major B operand (keys x dims in shared memory), so no transpose.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace sgs {

constexpr int PF_M = 128;                   // queries per CTA
constexpr int PF_N = 128;                   // keys per KV tile
constexpr int PF_CHUNK = 128 * 64 * 2;      // [128 rows][64 cols] 2-byte, 128-byte swizzle = 16 KB
constexpr int PF_TILE = 2 * PF_CHUNK;       // 128 x 128 = 32 KB
constexpr int PF_SMEM = 1024 + 7 * PF_TILE + 512;  // Q, K[2], V[2], P hi, P lo

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor of an MN-major operand with the 128-byte
// swizzle: atoms of 64 MN elements (128 B) x 8 K rows (1024 B); lbo = bytes
// between MN atoms, sbo = bytes between 8-row K groups.
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // sm_100 descriptor version
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// bf16 x bf16 -> fp32, both K-major (S = Q K^T); fp16 x fp16 -> fp32 with B
// MN-major (O += P V); M = N = 128
constexpr uint32_t PF_IDESC_QK = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(PF_N >> 3) << 17) |
                                 ((uint32_t)(PF_M >> 4) << 24);
constexpr uint32_t PF_IDESC_PV = (1u << 4) | (1u << 16) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(PF_M >> 4) << 24);

// Persistent: one CTA per SM walks the work items (query block, head) with a
// stride of gridDim.x; barrier phases run on global tile / item counters, so
// the next item's Q, K and V loads overlap the current item's softmax.
__global__ void __launch_bounds__(192, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, const int32_t* __restrict__ offs,
                           const int32_t* __restrict__ qblocks, int n_items, int nq, int nkv, float scale_log2,
                           __nv_bfloat16* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + PF_TILE;       // [2]
  uint8_t* sV = sK + 2 * PF_TILE;   // [2]
  uint8_t* sP = sV + 2 * PF_TILE;
  uint8_t* sPl = sP + PF_TILE;      // P = P_hi + P_lo (fp16 each, ~22 significant bits)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sPl + PF_TILE);
  uint64_t *q_full = bars, *k_full = bars + 1, *k_empty = bars + 3, *v_full = bars + 5, *v_empty = bars + 7,
           *s_full = bars + 9, *s_empty = bars + 11, *p_full = bars + 13, *pv_done = bars + 14, *q_empty = bars + 15,
           *o_free = bars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g_sz = nq / nkv;
  // work item -> (prompt, query block, head); consecutive items are the heads
  // of one query block, so co-running CTAs share the K/V tiles in L2
  struct Item {
    int h, hk, off, P, q0, qrows, nt;
  };
  auto item = [&](int it) {
    Item x;
    const int e = it / nq;
    x.h = it - e * nq;
    x.hk = x.h / g_sz;
    const int p = qblocks[2 * e], qb = qblocks[2 * e + 1];
    x.off = offs[p];
    x.P = offs[p + 1] - x.off;
    x.q0 = qb * PF_M;
    x.qrows = min(PF_M, x.P - x.q0);
    x.nt = (x.q0 + x.qrows - 1) / PF_N + 1;  // KV tiles up to the causal diagonal
    return x;
  };

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1), mbar_init(&k_empty[s], 1), mbar_init(&v_full[s], 1), mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1), mbar_init(&s_empty[s], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(pv_done, 1);
    mbar_init(o_free, 4);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S buffers at columns 0 and 128, O at 256
  pdl_trigger();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (q, k, v were written by the predecessor)
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    pdl_wait();
    int gt = 0, ni = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++ni) {
      const Item x = item(it);
      if (ni >= 1) mbar_wait(q_empty, (ni - 1) & 1);  // the previous item's S MMAs are done with Q
      mbar_expect_tx(q_full, PF_TILE);
      tma_load_3d(sQ, &tmQ, x.off + x.q0, 2 * x.h, q_full);
      for (int j = 0; j < x.nt; ++j, ++gt) {
        const int s = gt & 1;
        if (gt >= 2) mbar_wait(&k_empty[s], ((gt >> 1) - 1) & 1);
        mbar_expect_tx(&k_full[s], PF_TILE);
        tma_load_3d(sK + s * PF_TILE, &tmK, x.off + j * PF_N, 2 * x.hk, &k_full[s]);
        if (gt >= 2) mbar_wait(&v_empty[s], ((gt >> 1) - 1) & 1);
        mbar_expect_tx(&v_full[s], PF_TILE);
        tma_load_3d(sV + s * PF_TILE, &tmV, x.off + j * PF_N, 2 * x.hk, &v_full[s]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer: S_j, then O += P_{j-1} V_{j-1}
    const uint32_t qa = smem_u32(sQ), pa = smem_u32(sP), pla = smem_u32(sPl);
    int gs = 0, gp = 0, ni = 0;  // global S tile, global PV tile, item
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++ni) {
      const Item x = item(it);
      mbar_wait(q_full, ni & 1);
      tc_fence_after();
      for (int j = 0; j <= x.nt; ++j) {
        if (j < x.nt) {
          const int s = gs & 1;
          mbar_wait(&k_full[s], (gs >> 1) & 1);
          if (gs >= 2) mbar_wait(&s_empty[s], ((gs >> 1) - 1) & 1);  // the softmax has read S two tiles ago
          tc_fence_after();
          const uint32_t kb = smem_u32(sK + s * PF_TILE);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {  // head dims 16 kk .. 16 kk + 15
            const uint64_t ad = umma_desc_sw128(qa + (kk >> 2) * PF_CHUNK) + 2 * (kk & 3);
            const uint64_t bd = umma_desc_sw128(kb + (kk >> 2) * PF_CHUNK) + 2 * (kk & 3);
            umma_bf16(tmem + (uint32_t)(s * PF_N), ad, bd, PF_IDESC_QK, kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[s]);
          umma_commit(&k_empty[s]);
          if (j == x.nt - 1) umma_commit(q_empty);
          ++gs;
        }
        if (j >= 1) {
          const int s = gp & 1;
          mbar_wait(p_full, gp & 1);  // P written, O rescaled
          mbar_wait(&v_full[s], (gp >> 1) & 1);
          if (j == 1 && ni >= 1) mbar_wait(o_free, (ni - 1) & 1);  // the previous item's O is read out
          tc_fence_after();
          const uint32_t vb = smem_u32(sV + s * PF_TILE);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {  // keys 16 kk .. 16 kk + 15: O += P_hi V, then P_lo V
            const uint64_t bd = umma_desc_sw128_mn(vb + kk * 2048, PF_CHUNK, 1024);
            const uint64_t ad = umma_desc_sw128(pa + (kk >> 2) * PF_CHUNK) + 2 * (kk & 3);
            umma_bf16(tmem + 256u, ad, bd, PF_IDESC_PV, (j > 1 || kk > 0) ? 1u : 0u);
            const uint64_t al = umma_desc_sw128(pla + (kk >> 2) * PF_CHUNK) + 2 * (kk & 3);
            umma_bf16(tmem + 256u, al, bd, PF_IDESC_PV, 1u);
          }
          umma_commit(pv_done);
          umma_commit(&v_empty[s]);
          ++gp;
        }
      }
    }
  } else if (warp >= 2) {
    // ---------------- softmax + epilogue: thread = query row = TMEM lane
    const int g = warp & 3;  // TMEM lane quarter this warp may access
    const int row = 32 * g + lane;
    const uint32_t lane_off = (uint32_t)(32 * g) << 16;
    const uint32_t o_addr = tmem + 256u + lane_off;
    int gt = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const Item x = item(it);
      const int qi = x.q0 + row;  // query index within the prompt
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < x.nt; ++j, ++gt) {
        const int s = gt & 1;
        mbar_wait(&s_full[s], (gt >> 1) & 1);
        tc_fence_after();
        const uint32_t s_addr = tmem + (uint32_t)(s * PF_N) + lane_off;
        uint32_t r[8][16];
#pragma unroll
        for (int c = 0; c < 8; ++c) tmem_ld16(s_addr + 16 * c, r[c]);
        tmem_wait_ld();
        const int kbase = j * PF_N;
        const bool full_tile = kbase + PF_N - 1 <= x.q0 && kbase + PF_N <= x.P;  // no mask in this tile
        const int kmax = full_tile ? kbase + PF_N - 1 : min(qi, x.P - 1);       // last valid key of the row
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
          for (int i = 0; i < 16; ++i)
            mx = (kbase + 16 * c + i <= kmax) ? fmaxf(mx, __uint_as_float(r[c][i])) : mx;
        const float m_new = fmaxf(m, mx * scale_log2);
        if (j >= 1) {  // PV of the previous tile done: O is stable and the P buffer free
          mbar_wait(pv_done, (gt - 1) & 1);
          tc_fence_after();
        }
        const float alpha = exp2f(m - m_new);  // m = -inf at j = 0: alpha = 0, l = 0
        if (j >= 1 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
          for (int c = 0; c < 8; ++c) {
            uint32_t o[16];
            tmem_ld16(o_addr + 16 * c, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16(o_addr + 16 * c, o);
          }
          tmem_wait_st();
        }
        l *= alpha;
        // P = 2^(s * scale - m_new) split as P_hi + P_lo (fp16 each: ~22 significant bits,
        // the precision of the fp32 softmax weights), rows of the K-major swizzled P tiles
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t ph[8], pl[8];
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const int key = kbase + 16 * c + i;
            const float p0 = key <= kmax ? exp2f(fmaf(__uint_as_float(r[c][i]), scale_log2, -m_new)) : 0.f;
            const float p1 = key + 1 <= kmax ? exp2f(fmaf(__uint_as_float(r[c][i + 1]), scale_log2, -m_new)) : 0.f;
            l += p0 + p1;
            split_f16x2(p0, p1, ph[i >> 1], pl[i >> 1]);
          }
          const int u0 = 2 * (c & 3);  // 16-byte units (8 keys) within the 128-byte row
          const size_t o0 = (size_t)(c >> 2) * PF_CHUNK + row * 128;
          *reinterpret_cast<uint4*>(sP + o0 + ((u0 ^ (row & 7)) << 4)) = make_uint4(ph[0], ph[1], ph[2], ph[3]);
          *reinterpret_cast<uint4*>(sP + o0 + (((u0 + 1) ^ (row & 7)) << 4)) = make_uint4(ph[4], ph[5], ph[6], ph[7]);
          *reinterpret_cast<uint4*>(sPl + o0 + ((u0 ^ (row & 7)) << 4)) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
          *reinterpret_cast<uint4*>(sPl + o0 + (((u0 + 1) ^ (row & 7)) << 4)) = make_uint4(pl[4], pl[5], pl[6], pl[7]);
        }
        m = m_new;
        tc_fence_before();
        fence_proxy_async_smem();  // P is read by the tensor core (async proxy)
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&s_empty[s]);
          mbar_arrive(p_full);
        }
      }
      mbar_wait(pv_done, (gt - 1) & 1);
      tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* orow = out + ((size_t)(x.off + qi) * nq + x.h) * 128;
      uint32_t o[8][16];
#pragma unroll
      for (int c = 0; c < 8; ++c) tmem_ld16(o_addr + 16 * c, o[c]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_free);  // the next item's first PV may overwrite O
      if (row < x.qrows) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t w[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
            w[i] = pack_bf16x2(__uint_as_float(o[c][2 * i]) * inv, __uint_as_float(o[c][2 * i + 1]) * inv);
          *reinterpret_cast<uint4*>(orow + 16 * c) = make_uint4(w[0], w[1], w[2], w[3]);
          *reinterpret_cast<uint4*>(orow + 16 * c + 8) = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

cudaError_t attn_prefill_tc(const void* q, const void* k, const void* v_f16, const int32_t* offs,
                            const int32_t* qblocks128, int n_qblocks128, int T, int nq, int nkv, void* out,
                            cudaStream_t stream) {
  if (n_qblocks128 <= 0 || T <= 0) return cudaSuccess;
  if (nq % nkv != 0) return cudaErrorInvalidValue;
  CUtensorMap tq, tk, tv;
  if (!tmap_bf16_rows(&tq, q, T, (int64_t)nq * 128, 128, 2) || !tmap_bf16_rows(&tk, k, T, (int64_t)nkv * 128, 128, 2) ||
      !tmap_bf16_rows(&tv, v_f16, T, (int64_t)nkv * 128, 128, 2))
    return cudaErrorInvalidValue;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(attn_prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PF_SMEM);
    if (e != cudaSuccess) return e;
    set = true;
  }
  const float sl2 = (float)(1.4426950408889634 / std::sqrt(128.0));
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int n_items = n_qblocks128 * nq;
  return launch_pdl(attn_prefill_tc_kernel, dim3(n_items < sms ? n_items : sms), dim3(192), (size_t)PF_SMEM, stream,
                    tq, tk, tv, offs, qblocks128, n_items, nq, nkv, sl2, reinterpret_cast<__nv_bfloat16*>(out));
}

}  // namespace sgs
