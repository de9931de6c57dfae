// NEXT-2 tensor-parallel exchange over NVLink peer memory (decode program).
//
// A tensor-parallel instance (DESIGN.md §10 NEXT-2) splits every layer's
// heads / FFN columns / vocabulary rows over tp shards; after the O and down
// projections each shard holds a partial of the residual update and after the
// LM head a partial argmax.  With NCCL the decode step of a 7B model at b=1
// spends more time in 57 all-reduce launches than it saves in weight reads
// (profiles/r02/tp_*.json).  These kernels do the exchange themselves, in the
// consumer: each shard pushes its partial rows straight into every peer's
// receive slot (remote stores over NVLink into memory opened with CUDA IPC),
// raises one flag per CTA in the peer, waits for the peers' flags and reduces
// locally -- fused with the RMSNorm that consumes the sum, so an all-reduce
// costs no extra launch and one NVLink one-way trip.
//
// Exchange memory (one cudaMalloc per shard, opened by the peers):
//   data [2 parity][tp src][rows * d] fp32   partial rows
//   keys [2 parity][tp src][rows]     u64    argmax keys
//   flag [2 parity][tp src][TPX_CTAS] u32    epoch written by src for CTA c
//   seq, done                         u32    local epoch counter (last CTA bumps)
// Exchanges are numbered by a device-side epoch (all shards run the same
// sequence, so the numbers agree); consecutive exchanges alternate parity,
// and a shard can be at most one exchange ahead of a peer (it cannot finish
// exchange e+1 before the peer pushed e+1, i.e. finished reading e), so two
// parities make the slot reuse race-free.  A peer that never arrives (a shard
// that diverged) traps after 10 s instead of hanging the GPU.
#include <cuda_bf16.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace sgs {

__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct XchView {
  float* data;
  unsigned long long* keys;
  unsigned int* flag;
  unsigned int* ctr;  // [0] seq, [1] done
};
__device__ __forceinline__ XchView xch_view(uint8_t* base, int tp, int rows, int d) {
  XchView v;
  v.data = reinterpret_cast<float*>(base);
  v.keys = reinterpret_cast<unsigned long long*>(base + (size_t)2 * tp * rows * d * 4);
  v.flag = reinterpret_cast<unsigned int*>(base + (size_t)2 * tp * rows * d * 4 + (size_t)2 * tp * rows * 8);
  v.ctr = v.flag + 2 * tp * TPX_CTAS;
  return v;
}

size_t tp_xch_bytes(int tp, int rows, int d) {
  return (size_t)2 * tp * rows * d * 4 + (size_t)2 * tp * rows * 8 + (size_t)2 * tp * TPX_CTAS * 4 + 64;
}

// Thread 0 of each CTA: publish this CTA's pushes to every peer, then wait
// until every peer has published its own for the same CTA and epoch.
__device__ void xch_signal_wait(const TpPeers& P, int rows, int d, unsigned int epoch, int cta) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int par = epoch & 1;
    for (int s = 0; s < P.tp; ++s) {
      if (s == P.me) continue;
      XchView pv = xch_view(P.base[s], P.tp, rows, d);
      st_release_sys(pv.flag + ((size_t)par * P.tp + P.me) * TPX_CTAS + cta, epoch);
    }
    XchView mv = xch_view(P.base[P.me], P.tp, rows, d);
    const uint64_t t0 = globaltimer();
    for (int s = 0; s < P.tp; ++s) {
      if (s == P.me) continue;
      const unsigned int* f = mv.flag + ((size_t)par * P.tp + s) * TPX_CTAS + cta;
      while ((int)(ld_acquire_sys(f) - epoch) < 0) {
        if (globaltimer() - t0 > 10000000000ull) __trap();  // a shard left the common exchange sequence
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned int xch_epoch(const TpPeers& P, int rows, int d) {
  __shared__ unsigned int ep;
  if (threadIdx.x == 0) ep = *(volatile unsigned int*)xch_view(P.base[P.me], P.tp, rows, d).ctr + 1u;
  __syncthreads();
  return ep;
}

// the last CTA to finish advances the epoch for the next exchange on this shard
__device__ __forceinline__ void xch_retire(const TpPeers& P, int rows, int d, unsigned int epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    XchView mv = xch_view(P.base[P.me], P.tp, rows, d);
    __threadfence();
    if (atomicAdd(mv.ctr + 1, 1u) == gridDim.x - 1) {
      mv.ctr[1] = 0u;
      *(volatile unsigned int*)mv.ctr = epoch;
    }
  }
}

// h[T, d]: this shard's partial (shard 0's includes the residual).  After the
// call h = sum of all shards' partials in shard order on shard 0 and 0 on the
// others (their next projection accumulates into a zeroed h), and, when w is
// given, y = RMSNorm(sum) * w in bf16 on every shard (same arithmetic as
// rmsnorm_kernel: fp64 sum of squares and scaling).  CTA c owns rows c, c+G, ...
template <int VPT>
__global__ void tp_allreduce_rmsnorm_kernel(float* __restrict__ h, const __nv_bfloat16* __restrict__ w,
                                            __nv_bfloat16* __restrict__ y, int T, int d, float eps, TpPeers P,
                                            int rows_cap) {
  pdl_trigger();
  const int i0 = threadIdx.x * 4 * VPT;
  uint2 wb[VPT];
  if (w) {
#pragma unroll
    for (int k = 0; k < VPT; ++k) wb[k] = *reinterpret_cast<const uint2*>(w + i0 + 4 * k);
  }
  pdl_wait();
  const unsigned int epoch = xch_epoch(P, rows_cap, d);
  const int par = epoch & 1;
  // push this shard's partial rows into slot [par][me] of every peer
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const float* hr = h + (size_t)t * d;
    float4 v[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) v[k] = *reinterpret_cast<const float4*>(hr + i0 + 4 * k);
    for (int s = 0; s < P.tp; ++s) {
      if (s == P.me) continue;
      float* dst = xch_view(P.base[s], P.tp, rows_cap, d).data + (((size_t)par * P.tp + P.me) * rows_cap + t) * d;
#pragma unroll
      for (int k = 0; k < VPT; ++k) *reinterpret_cast<float4*>(dst + i0 + 4 * k) = v[k];
    }
  }
  xch_signal_wait(P, rows_cap, d, epoch, blockIdx.x);
  const float* mine = xch_view(P.base[P.me], P.tp, rows_cap, d).data;
  __shared__ double red[32];
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    float* hr = h + (size_t)t * d;
    float4 v[VPT];
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < P.tp; ++s) {  // shard order: every shard forms the bitwise-same sum
        const float4 b = s == P.me ? *reinterpret_cast<const float4*>(hr + i0 + 4 * k)
                                   : __ldcv(reinterpret_cast<const float4*>(
                                         mine + (((size_t)par * P.tp + s) * rows_cap + t) * d + i0 + 4 * k));
        if (s == 0) {
          a = b;
        } else {
          a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
        }
      }
      v[k] = a;
      ss += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
    }
#pragma unroll
    for (int k = 0; k < VPT; ++k)
      *reinterpret_cast<float4*>(hr + i0 + 4 * k) = P.me == 0 ? v[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    if (!w) continue;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
      double a = threadIdx.x < ((blockDim.x + 31) >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (threadIdx.x == 0) red[0] = a;
    }
    __syncthreads();
    const double r = 1.0 / sqrt(red[0] / (double)d + (double)eps);
    __nv_bfloat16* yr = y + (size_t)t * d;
    auto f = [&](float x, uint32_t wbits) { return (float)((double)x * r * (double)__uint_as_float(wbits)); };
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      uint2 o;
      o.x = pack_bf16x2(f(v[k].x, wb[k].x << 16), f(v[k].y, wb[k].x & 0xffff0000u));
      o.y = pack_bf16x2(f(v[k].z, wb[k].y << 16), f(v[k].w, wb[k].y & 0xffff0000u));
      *reinterpret_cast<uint2*>(yr + i0 + 4 * k) = o;
    }
    __syncthreads();
  }
  xch_retire(P, rows_cap, d, epoch);
}

cudaError_t tp_allreduce_rmsnorm(float* h, const void* w, void* y, int T, int d, float eps, const TpPeers& P,
                                 int rows_cap, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  if (T > rows_cap || P.tp < 2 || P.tp > TPX_MAX) return cudaErrorInvalidValue;
  const int grid = T < TPX_CTAS ? T : TPX_CTAS;
  const __nv_bfloat16* W = reinterpret_cast<const __nv_bfloat16*>(w);
  __nv_bfloat16* Y = reinterpret_cast<__nv_bfloat16*>(y);
  if (d % 8 == 0 && d / 8 <= 1024 && d / 8 >= 32)
    return launch_pdl(tp_allreduce_rmsnorm_kernel<2>, dim3(grid), dim3(d / 8), 0, stream, h, W, Y, T, d, eps, P,
                      rows_cap);
  if (d % 4 == 0 && d / 4 <= 1024 && d / 4 >= 32)
    return launch_pdl(tp_allreduce_rmsnorm_kernel<1>, dim3(grid), dim3(d / 4), 0, stream, h, W, Y, T, d, eps, P,
                      rows_cap);
  return cudaErrorInvalidValue;
}

// Greedy sampling across vocabulary shards: every shard's (max logit, lowest
// index) keys (GEMM mode 4, finalize = 0) are exchanged, the maximum taken,
// and the tokens written exactly as argmax_keys_finalize does; keys are
// re-zeroed for the next launch.
__global__ void tp_argmax_exchange_kernel(unsigned long long* keys, int rows, const int32_t* slot,
                                          const int32_t* tok_idx, int32_t* last_tok, int32_t* hist, int max_gen,
                                          TpPeers P, int rows_cap, int d) {
  pdl_trigger();
  pdl_wait();
  const unsigned int epoch = xch_epoch(P, rows_cap, d);
  const int par = epoch & 1;
  for (int t = threadIdx.x; t < rows; t += blockDim.x) {
    const unsigned long long k = keys[t];
    for (int s = 0; s < P.tp; ++s) {
      if (s == P.me) continue;
      xch_view(P.base[s], P.tp, rows_cap, d).keys[((size_t)par * P.tp + P.me) * rows_cap + t] = k;
    }
  }
  xch_signal_wait(P, rows_cap, d, epoch, 0);
  const unsigned long long* mine = xch_view(P.base[P.me], P.tp, rows_cap, d).keys;
  for (int t = threadIdx.x; t < rows; t += blockDim.x) {
    unsigned long long k = keys[t];
    for (int s = 0; s < P.tp; ++s) {
      if (s == P.me) continue;
      const unsigned long long o = __ldcv(mine + ((size_t)par * P.tp + s) * rows_cap + t);
      k = o > k ? o : k;
    }
    keys[t] = 0ull;
    const int sl = slot[t];
    if (sl >= 0) {
      const int32_t tok = (int32_t)(~(uint32_t)k);
      last_tok[sl] = tok;
      hist[(size_t)sl * max_gen + tok_idx[t]] = tok;
    }
  }
  xch_retire(P, rows_cap, d, epoch);
}

cudaError_t tp_argmax_exchange(unsigned long long* keys, int rows, const int32_t* slot, const int32_t* tok_idx,
                               int32_t* last_tok, int32_t* hist, int max_gen, const TpPeers& P, int rows_cap, int d,
                               cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (rows > rows_cap || P.tp < 2 || P.tp > TPX_MAX) return cudaErrorInvalidValue;
  return launch_pdl(tp_argmax_exchange_kernel, dim3(1), dim3(256), 0, stream, keys, rows, slot, tok_idx, last_tok,
                    hist, max_gen, P, rows_cap, d);
}

}  // namespace sgs
