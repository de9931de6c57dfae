// a4 / K10: causal prefill attention over each admitted prompt (the prompt
// tokens "establish the KV cache", §2.1).  Flash-style: one CTA =
// (prompt, kv head, 16 queries) with one warp per query head of the GQA group
// sharing the key/value tiles; tiles of 64 tokens are double-buffered in
// shared memory with cp.async (XOR-swizzled rows), S = Q K^T on mma.sync bf16
// with fp32 accumulation, online softmax in fp32 (exp2), O += P V with P split
// into two fp16 parts.  The prompt K/V come from the contiguous copy the
// RoPE/append kernel writes for prefill rows.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace sgs {

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One CTA = (prompt, kv head, 16 consecutive queries); warp w handles q head
// kh * G + w of the group, so the K/V tiles staged in shared memory serve all
// G query heads that read them (GQA).  Key/value tiles of 64 tokens are
// double-buffered with cp.async (zero-filled past the prompt end).
template <int HD>
__global__ void __launch_bounds__(256, 2)
    attn_prefill_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                        const __nv_bfloat16* __restrict__ v, const int32_t* __restrict__ offs,
                        const int32_t* __restrict__ qblocks, int nq, int nkv, float scale_log2,
                        __nv_bfloat16* __restrict__ out) {
  constexpr int BK = 64, RC = HD / 8, NT = HD / 8;
  constexpr int TILE = BK * HD * 2;  // bytes of K (or V) per tile
  extern __shared__ __align__(128) uint8_t sm[];  // [2 buffers][K | V]
  pdl_trigger();
  pdl_wait();
  const int e = blockIdx.x >> 2, sub = blockIdx.x & 3;
  const int p = qblocks[2 * e], qb = qblocks[2 * e + 1];
  const int kh = blockIdx.y, G = nq / nkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = kh * G + warp;
  const int off = offs[p], P = offs[p + 1] - off;
  const int q0 = qb * 64 + sub * 16;
  if (q0 >= P) return;
  const int kend = min(P, q0 + 16);
  const int ntiles = (kend + BK - 1) / BK;
  const uint32_t sbase = smem_u32(sm);

  auto load_tile = [&](int kt, int buf) {
    const uint32_t kb = sbase + (uint32_t)(buf * 2 * TILE), vb = kb + TILE;
    for (int c = threadIdx.x; c < BK * RC; c += blockDim.x) {
      const int r = c / RC, ch = c % RC, key = kt * BK + r;
      const bool ok = key < P;
      const size_t src = ((size_t)(off + (ok ? key : 0)) * nkv + kh) * HD + ch * 8;
      const uint32_t dst = (uint32_t)(r * HD * 2 + ((ch ^ kv_swz(r, RC)) << 4));
      cp_async16(kb + dst, k + src, ok ? 16 : 0);
      cp_async16(vb + dst, v + src, ok ? 16 : 0);
    }
    cp_async_commit();
  };
  load_tile(0, 0);

  const int r0 = lane >> 2, r1 = r0 + 8, cq = 2 * (lane & 3);
  uint32_t qa[HD / 16][4];
  {
    const uint32_t* Q = reinterpret_cast<const uint32_t*>(q);
    const bool v0 = q0 + r0 < P, v1 = q0 + r1 < P;
    const size_t b0 = (((size_t)(off + q0 + r0) * nq + h) * HD) >> 1;
    const size_t b1 = (((size_t)(off + q0 + r1) * nq + h) * HD) >> 1;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      qa[kk][0] = v0 ? Q[b0 + ((16 * kk + cq) >> 1)] : 0u;
      qa[kk][1] = v1 ? Q[b1 + ((16 * kk + cq) >> 1)] : 0u;
      qa[kk][2] = v0 ? Q[b0 + ((16 * kk + 8 + cq) >> 1)] : 0u;
      qa[kk][3] = v1 ? Q[b1 + ((16 * kk + 8 + cq) >> 1)] : 0u;
    }
  }
  float o[NT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int ktok = ((lane >> 4) << 3) + (lane & 7), kchk = (lane >> 3) & 1;
  const int vtok = (((lane >> 3) & 1) << 3) + (lane & 7), vchk = lane >> 4;

  for (int kt = 0; kt < ntiles; ++kt) {
    if (kt + 1 < ntiles) {
      load_tile(kt + 1, (kt + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint32_t kbase = sbase + (uint32_t)((kt & 1) * 2 * TILE), vbase = kbase + TILE;
#pragma unroll
    for (int j = 0; j < BK / 16; ++j) {
      if (kt * BK + 16 * j > q0 + 15) break;  // sub-tile entirely in the future of these queries
      float sc[2][4];
#pragma unroll
      for (int t = 0; t < 2; ++t) sc[t][0] = sc[t][1] = sc[t][2] = sc[t][3] = 0.f;
      const int kr = 16 * j + ktok;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int ch = 2 * kk + kchk;
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4(b0, b1, b2, b3, kbase + kr * (HD * 2) + ((ch ^ kv_swz(kr, RC)) << 4));
        mma_bf16_16816(sc[0], qa[kk], b0, b1);
        mma_bf16_16816(sc[1], qa[kk], b2, b3);
      }
      if (kt * BK + 16 * j + 15 > q0 || kt * BK + 16 * j + 15 >= P) {  // diagonal / ragged sub-tile
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int el = 0; el < 4; ++el) {
            const int key = kt * BK + 16 * j + 8 * t + cq + (el & 1);
            const int qry = q0 + (el < 2 ? r0 : r1);
            if (key > qry || key >= P) sc[t][el] = -INFINITY;
          }
      }
      float mx0 = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1])) * scale_log2;
      float mx1 = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3])) * scale_log2;
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      // rows whose keys are all masked so far keep m = -inf; guard the rescale
      const float a0 = mn0 == -INFINITY ? 1.f : exp2f(m0 - mn0);
      const float a1 = mn1 == -INFINITY ? 1.f : exp2f(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
      float pp[2][4];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        pp[t][0] = mn0 == -INFINITY ? 0.f : exp2f(fmaf(sc[t][0], scale_log2, -mn0));
        pp[t][1] = mn0 == -INFINITY ? 0.f : exp2f(fmaf(sc[t][1], scale_log2, -mn0));
        pp[t][2] = mn1 == -INFINITY ? 0.f : exp2f(fmaf(sc[t][2], scale_log2, -mn1));
        pp[t][3] = mn1 == -INFINITY ? 0.f : exp2f(fmaf(sc[t][3], scale_log2, -mn1));
      }
      uint32_t pa[4], pl[4];  // P = P_hi + P_lo in fp16 (~22 significant bits)
      split_f16x2(pp[0][0], pp[0][1], pa[0], pl[0]);
      split_f16x2(pp[0][2], pp[0][3], pa[1], pl[1]);
      split_f16x2(pp[1][0], pp[1][1], pa[2], pl[2]);
      split_f16x2(pp[1][2], pp[1][3], pa[3], pl[3]);
      l0 = l0 * a0 + ((pp[0][0] + pp[0][1]) + (pp[1][0] + pp[1][1]));
      l1 = l1 * a1 + ((pp[0][2] + pp[0][3]) + (pp[1][2] + pp[1][3]));
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        o[nt][0] *= a0;
        o[nt][1] *= a0;
        o[nt][2] *= a1;
        o[nt][3] *= a1;
      }
      const int vr = 16 * j + vtok;
#pragma unroll
      for (int nn = 0; nn < HD / 16; ++nn) {
        const int ch = 2 * nn + vchk;
        uint32_t v0, v1, v2, v3;
        ldmatrix_x4_trans(v0, v1, v2, v3, vbase + vr * (HD * 2) + ((ch ^ kv_swz(vr, RC)) << 4));
        const uint32_t h0 = bf16x2_to_f16x2(v0), h1 = bf16x2_to_f16x2(v1);
        const uint32_t h2 = bf16x2_to_f16x2(v2), h3 = bf16x2_to_f16x2(v3);
        mma_f16_16816(o[2 * nn], pa, h0, h1);
        mma_f16_16816(o[2 * nn], pl, h0, h1);
        mma_f16_16816(o[2 * nn + 1], pa, h2, h3);
        mma_f16_16816(o[2 * nn + 1], pl, h2, h3);
      }
    }
    __syncthreads();  // this buffer is refilled by the load issued in iteration kt + 1
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    if (q0 + r0 < P) {
      __nv_bfloat162 x = __floats2bfloat162_rn(o[nt][0] * i0, o[nt][1] * i0);
      *reinterpret_cast<__nv_bfloat162*>(out + ((size_t)(off + q0 + r0) * nq + h) * HD + 8 * nt + cq) = x;
    }
    if (q0 + r1 < P) {
      __nv_bfloat162 x = __floats2bfloat162_rn(o[nt][2] * i1, o[nt][3] * i1);
      *reinterpret_cast<__nv_bfloat162*>(out + ((size_t)(off + q0 + r1) * nq + h) * HD + 8 * nt + cq) = x;
    }
  }
}

template <int HD>
static cudaError_t launch_prefill(const void* q, const void* k, const void* v, const int32_t* offs,
                                  const int32_t* qblocks, int n_qblocks, int nq, int nkv, float sl2, void* out,
                                  cudaStream_t stream) {
  constexpr int smem = 2 * 2 * 64 * HD * 2;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(attn_prefill_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    set = true;
  }
  return launch_pdl(attn_prefill_kernel<HD>, dim3(4 * n_qblocks, nkv), dim3(32 * (nq / nkv)), (size_t)smem, stream,
                    reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k),
                    reinterpret_cast<const __nv_bfloat16*>(v), offs, qblocks, nq, nkv, sl2,
                    reinterpret_cast<__nv_bfloat16*>(out));
}

cudaError_t attn_prefill(const void* q, const void* k, const void* v, const int32_t* offs, const int32_t* qblocks,
                         int n_qblocks, int nq, int nkv, int hd, void* out, cudaStream_t stream) {
  if (n_qblocks <= 0) return cudaSuccess;
  if (nq % nkv != 0 || nq / nkv > 8) return cudaErrorInvalidValue;  // one warp per query head of a group
  const float sl2 = (float)(1.4426950408889634 / std::sqrt((double)hd));
  switch (hd) {
    case 32:
      return launch_prefill<32>(q, k, v, offs, qblocks, n_qblocks, nq, nkv, sl2, out, stream);
    case 64:
      return launch_prefill<64>(q, k, v, offs, qblocks, n_qblocks, nq, nkv, sl2, out, stream);
    case 128:
      return launch_prefill<128>(q, k, v, offs, qblocks, n_qblocks, nq, nkv, sl2, out, stream);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace sgs
