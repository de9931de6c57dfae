// NEXT-2 tensor-parallel exchange over NVLink peer memory (decode program).
//
// A tensor-parallel instance (DESIGN.md §10 NEXT-2) splits every layer's
// heads / FFN columns / vocabulary rows over tp shards; after the O and down
// projections each shard holds a partial of the residual update and after the
// LM head a partial argmax.  With NCCL the decode step of a 7B model at b=1
// spends more time in 57 all-reduce launches than it saves in weight reads
// (profiles/r02/tp_*.json).  These kernels do the exchange themselves, in the
// consumer: each shard pushes its partial rows straight into every peer's
// receive slot (remote stores over NVLink into memory opened with CUDA IPC)
// and reduces locally -- fused with the RMSNorm that consumes the sum, so an
// all-reduce costs no extra launch and one NVLink one-way trip.
//
// Low-latency protocol: every 16-byte store carries 8 bytes of payload and
// the exchange's epoch twice ({x, E, y, E}); 8-byte halves are single-copy
// atomic, so a receiver that reads both epochs equal to E has the payload --
// no fences, no separate flags, no counters.  Epochs come from the decode
// metadata (launch counter) and the exchange's index in the launch, so every
// shard numbers the exchanges identically; consecutive exchanges alternate
// between two slot parities, and a shard can be at most one exchange ahead
// of a peer (it cannot finish exchange e+1 before the peer pushed e+1, i.e.
// finished reading e), so the parities make slot reuse race-free.  A peer
// that never arrives (a shard that left the common sequence) traps after
// 10 s instead of hanging the GPU.
//
// Exchange memory (one cudaMalloc per shard, opened by the peers):
//   data [2 parity][tp src][rows * d / 2] uint4   {x, E, y, E} per 2 floats
//   keys [2 parity][tp src][rows]         uint4   {lo, E, hi, E} per u64 key
#include <cuda_bf16.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace sgs {

__device__ __forceinline__ void st_ll(uint4* p, uint32_t a, uint32_t b, uint32_t e) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(e), "r"(b), "r"(e)
               : "memory");
}
__device__ __forceinline__ uint4 ld_ll(const uint4* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// spin until both epochs of the unit are e; returns the payload (x, y)
__device__ __forceinline__ uint2 wait_ll(const uint4* p, uint32_t e) {
  uint4 v = ld_ll(p);
  if (v.y == e && v.w == e) return make_uint2(v.x, v.z);
  const uint64_t t0 = globaltimer();
  for (uint32_t n = 1;; ++n) {
    v = ld_ll(p);
    if (v.y == e && v.w == e) return make_uint2(v.x, v.z);
    if ((n & 1023) == 0 && globaltimer() - t0 > 10000000000ull) __trap();  // a shard left the sequence
  }
}

__device__ __forceinline__ uint4* xch_data(uint8_t* base, int tp, int rows, int d, int par, int src) {
  return reinterpret_cast<uint4*>(base) + ((size_t)par * tp + src) * rows * (d / 2);
}
__device__ __forceinline__ uint4* xch_keys(uint8_t* base, int tp, int rows, int d, int par, int src) {
  return reinterpret_cast<uint4*>(base) + (size_t)2 * tp * rows * (d / 2) + ((size_t)par * tp + src) * rows;
}

size_t tp_xch_bytes(int tp, int rows, int d) { return (size_t)2 * tp * rows * ((size_t)d / 2 + 1) * 16 + 256; }

__device__ __forceinline__ uint32_t xch_epoch(const int32_t* launch, int index, int per_launch) {
  return (uint32_t)*launch * (uint32_t)per_launch + (uint32_t)index + 1u;
}

// h[T, d]: this shard's partial (shard 0's includes the residual).  After the
// call h = sum of all shards' partials in shard order on shard 0 and 0 on the
// others (their next projection accumulates into a zeroed h), and, when w is
// given, y = RMSNorm(sum) * w in bf16 on every shard (same arithmetic as
// rmsnorm_kernel: fp64 sum of squares and scaling).  CTA c owns rows c, c+G,
// ...; thread t owns the float pairs t + k * blockDim.x (k < PPT), so a warp's
// loads, LL stores and polls each cover consecutive 8- / 16-byte units.
template <int PPT>
__global__ void tp_allreduce_rmsnorm_kernel(float* __restrict__ h, const __nv_bfloat16* __restrict__ w,
                                            __nv_bfloat16* __restrict__ y, int T, int d, float eps, TpPeers P,
                                            int rows_cap, const int32_t* launch, int index, int per_launch) {
  pdl_trigger();
  const int nt = blockDim.x, half = d / 2;
  uint32_t wb[PPT];
  if (w) {
#pragma unroll
    for (int k = 0; k < PPT; ++k) wb[k] = reinterpret_cast<const uint32_t*>(w)[threadIdx.x + k * nt];
  }
  pdl_wait();
  const uint32_t E = xch_epoch(launch, index, per_launch);
  const int par = E & 1;
  // push this shard's partial rows into slot [par][me] of every peer
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const float2* hr = reinterpret_cast<const float2*>(h + (size_t)t * d);
    float2 v[PPT];
#pragma unroll
    for (int k = 0; k < PPT; ++k) v[k] = hr[threadIdx.x + k * nt];
    for (int s = 0; s < P.tp; ++s) {
      if (s == P.me) continue;
      uint4* dst = xch_data(P.base[s], P.tp, rows_cap, d, par, P.me) + (size_t)t * half;
#pragma unroll
      for (int k = 0; k < PPT; ++k)
        st_ll(dst + threadIdx.x + k * nt, __float_as_uint(v[k].x), __float_as_uint(v[k].y), E);
    }
  }
  __shared__ double red[32];
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    float2* hr = reinterpret_cast<float2*>(h + (size_t)t * d);
    float2 a[PPT];
    for (int s = 0; s < P.tp; ++s) {  // shard order: every shard forms the bitwise-same sum
      float2 b[PPT];
      if (s == P.me) {
#pragma unroll
        for (int k = 0; k < PPT; ++k) b[k] = hr[threadIdx.x + k * nt];
      } else {
        const uint4* src = xch_data(P.base[P.me], P.tp, rows_cap, d, par, s) + (size_t)t * half + threadIdx.x;
        uint4 u[PPT];
        bool ok = true;
#pragma unroll
        for (int k = 0; k < PPT; ++k) {  // all polls in flight at once; re-poll only what is missing
          u[k] = ld_ll(src + k * nt);
          ok = ok && u[k].y == E && u[k].w == E;
        }
        if (!ok) {
#pragma unroll
          for (int k = 0; k < PPT; ++k) {
            const uint2 q = wait_ll(src + k * nt, E);
            u[k].x = q.x, u[k].z = q.y;
          }
        }
#pragma unroll
        for (int k = 0; k < PPT; ++k) b[k] = make_float2(__uint_as_float(u[k].x), __uint_as_float(u[k].z));
      }
      if (s == 0) {
#pragma unroll
        for (int k = 0; k < PPT; ++k) a[k] = b[k];
      } else {
#pragma unroll
        for (int k = 0; k < PPT; ++k) a[k].x += b[k].x, a[k].y += b[k].y;
      }
    }
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      ss += (double)a[k].x * a[k].x + (double)a[k].y * a[k].y;
      hr[threadIdx.x + k * nt] = P.me == 0 ? a[k] : make_float2(0.f, 0.f);
    }
    if (!w) continue;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
      double q = threadIdx.x < ((blockDim.x + 31) >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
      if (threadIdx.x == 0) red[0] = q;
    }
    __syncthreads();
    const double r = 1.0 / sqrt(red[0] / (double)d + (double)eps);
    uint32_t* yr = reinterpret_cast<uint32_t*>(y + (size_t)t * d);
    auto f = [&](float x, uint32_t wbits) { return (float)((double)x * r * (double)__uint_as_float(wbits)); };
#pragma unroll
    for (int k = 0; k < PPT; ++k)
      yr[threadIdx.x + k * nt] = pack_bf16x2(f(a[k].x, wb[k] << 16), f(a[k].y, wb[k] & 0xffff0000u));
    __syncthreads();
  }
}

cudaError_t tp_allreduce_rmsnorm(float* h, const void* w, void* y, int T, int d, float eps, const TpPeers& P,
                                 int rows_cap, const int32_t* launch, int index, int per_launch, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  if (T > rows_cap || P.tp < 2 || P.tp > TPX_MAX || d % 64) return cudaErrorInvalidValue;
  // up to two rows' CTAs per SM, all co-resident (a CTA waits only for its own rows' peers)
  const int grid = T < TPX_CTAS ? T : TPX_CTAS;
  const __nv_bfloat16* W = reinterpret_cast<const __nv_bfloat16*>(w);
  __nv_bfloat16* Y = reinterpret_cast<__nv_bfloat16*>(y);
  const int half = d / 2;
  if (half % (4 * 32) == 0 && half / 4 <= 1024)
    return launch_pdl(tp_allreduce_rmsnorm_kernel<4>, dim3(grid), dim3(half / 4), 0, stream, h, W, Y, T, d, eps, P,
                      rows_cap, launch, index, per_launch);
  if (half % (2 * 32) == 0 && half / 2 <= 1024)
    return launch_pdl(tp_allreduce_rmsnorm_kernel<2>, dim3(grid), dim3(half / 2), 0, stream, h, W, Y, T, d, eps, P,
                      rows_cap, launch, index, per_launch);
  if (half % 32 == 0 && half <= 1024)
    return launch_pdl(tp_allreduce_rmsnorm_kernel<1>, dim3(grid), dim3(half), 0, stream, h, W, Y, T, d, eps, P,
                      rows_cap, launch, index, per_launch);
  return cudaErrorInvalidValue;
}

// Greedy sampling across vocabulary shards: every shard's (max logit, lowest
// index) keys (GEMM mode 4, finalize = 0) are exchanged, the maximum taken,
// and the tokens written exactly as argmax_keys_finalize does; keys are
// re-zeroed for the next launch.
__global__ void tp_argmax_exchange_kernel(unsigned long long* keys, int rows, const int32_t* slot,
                                          const int32_t* tok_idx, int32_t* last_tok, int32_t* hist, int max_gen,
                                          TpPeers P, int rows_cap, int d, const int32_t* launch, int index,
                                          int per_launch) {
  pdl_trigger();
  pdl_wait();
  const uint32_t E = xch_epoch(launch, index, per_launch);
  const int par = E & 1;
  for (int t = threadIdx.x; t < rows; t += blockDim.x) {
    const unsigned long long k = keys[t];
    for (int s = 0; s < P.tp; ++s) {
      if (s == P.me) continue;
      st_ll(xch_keys(P.base[s], P.tp, rows_cap, d, par, P.me) + t, (uint32_t)k, (uint32_t)(k >> 32), E);
    }
  }
  for (int t = threadIdx.x; t < rows; t += blockDim.x) {
    unsigned long long k = keys[t];
    for (int s = 0; s < P.tp; ++s) {
      if (s == P.me) continue;
      const uint2 o = wait_ll(xch_keys(P.base[P.me], P.tp, rows_cap, d, par, s) + t, E);
      const unsigned long long ok = ((unsigned long long)o.y << 32) | o.x;
      k = ok > k ? ok : k;
    }
    keys[t] = 0ull;
    const int sl = slot[t];
    if (sl >= 0) {
      const int32_t tok = (int32_t)(~(uint32_t)k);
      last_tok[sl] = tok;
      hist[(size_t)sl * max_gen + tok_idx[t]] = tok;
    }
  }
}

cudaError_t tp_argmax_exchange(unsigned long long* keys, int rows, const int32_t* slot, const int32_t* tok_idx,
                               int32_t* last_tok, int32_t* hist, int max_gen, const TpPeers& P, int rows_cap, int d,
                               const int32_t* launch, int index, int per_launch, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (rows > rows_cap || P.tp < 2 || P.tp > TPX_MAX) return cudaErrorInvalidValue;
  return launch_pdl(tp_argmax_exchange_kernel, dim3(1), dim3(256), 0, stream, keys, rows, slot, tok_idx, last_tok,
                    hist, max_gen, P, rows_cap, d, launch, index, per_launch);
}

}  // namespace sgs
