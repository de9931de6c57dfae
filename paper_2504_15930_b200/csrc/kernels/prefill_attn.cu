// a4 / K10: causal prefill attention over each admitted prompt (the prompt
// tokens "establish the KV cache", §2.1).  Flash-style: one CTA =
// (prompt, query head, 64-query block), 4 warps x 16 query rows; key/value
// tiles of 64 tokens staged in shared memory (XOR-swizzled rows), S = Q K^T
// on mma.sync bf16 with fp32 accumulation, online softmax in fp32 (exp2),
// O += P V with P in fp16.  The prompt K/V come from the contiguous copy the
// RoPE/append kernel writes for prefill rows.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace sgs {

template <int HD>
__global__ void __launch_bounds__(128)
    attn_prefill_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                        const __nv_bfloat16* __restrict__ v, const int32_t* __restrict__ offs,
                        const int32_t* __restrict__ qblocks, int nq, int nkv, float scale_log2,
                        __nv_bfloat16* __restrict__ out) {
  constexpr int BQ = 64, BK = 64, RC = HD / 8, NT = HD / 8;
  __shared__ __align__(128) uint8_t sK[BK * HD * 2];
  __shared__ __align__(128) uint8_t sV[BK * HD * 2];
  const int p = qblocks[2 * blockIdx.x], qb = qblocks[2 * blockIdx.x + 1];
  const int h = blockIdx.y, kh = h / (nq / nkv);
  const int off = offs[p], P = offs[p + 1] - off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = qb * BQ + warp * 16;
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
  const int kend = min(P, (qb + 1) * BQ);
  const uint32_t kbase = smem_u32(sK), vbase = smem_u32(sV);

  for (int kt = 0; kt * BK < kend; ++kt) {
    __syncthreads();
    for (int c = threadIdx.x; c < BK * RC; c += blockDim.x) {
      const int r = c / RC, ch = c % RC, key = kt * BK + r;
      uint4 kvv = make_uint4(0, 0, 0, 0), vvv = make_uint4(0, 0, 0, 0);
      if (key < P) {
        const size_t src = ((size_t)(off + key) * nkv + kh) * HD + ch * 8;
        kvv = *reinterpret_cast<const uint4*>(k + src);
        vvv = *reinterpret_cast<const uint4*>(v + src);
      }
      const int dst = r * HD * 2 + ((ch ^ kv_swz(r, RC)) << 4);
      *reinterpret_cast<uint4*>(sK + dst) = kvv;
      *reinterpret_cast<uint4*>(sV + dst) = vvv;
    }
    __syncthreads();
    if (q0 + 15 < kt * BK) continue;  // whole tile is in this warp's future
#pragma unroll
    for (int j = 0; j < BK / 16; ++j) {
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
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = kt * BK + 16 * j + 8 * t + cq + (e & 1);
          const int qry = q0 + (e < 2 ? r0 : r1);
          if (key > qry || key >= P) sc[t][e] = -INFINITY;
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

cudaError_t attn_prefill(const void* q, const void* k, const void* v, const int32_t* offs, const int32_t* qblocks,
                         int n_qblocks, int nq, int nkv, int hd, void* out, cudaStream_t stream) {
  if (n_qblocks <= 0) return cudaSuccess;
  const float sl2 = (float)(1.4426950408889634 / std::sqrt((double)hd));
  dim3 grid(n_qblocks, nq);
  auto Q = reinterpret_cast<const __nv_bfloat16*>(q);
  auto K = reinterpret_cast<const __nv_bfloat16*>(k);
  auto V = reinterpret_cast<const __nv_bfloat16*>(v);
  auto O = reinterpret_cast<__nv_bfloat16*>(out);
  switch (hd) {
    case 32:
      attn_prefill_kernel<32><<<grid, 128, 0, stream>>>(Q, K, V, offs, qblocks, nq, nkv, sl2, O);
      break;
    case 64:
      attn_prefill_kernel<64><<<grid, 128, 0, stream>>>(Q, K, V, offs, qblocks, nq, nkv, sl2, O);
      break;
    case 128:
      attn_prefill_kernel<128><<<grid, 128, 0, stream>>>(Q, K, V, offs, qblocks, nq, nkv, sl2, O);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace sgs
