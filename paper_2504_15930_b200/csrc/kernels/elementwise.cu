// Small HBM/latency-bound kernels of the iteration (SURVEY §8a rows a5, a6,
// a7, a10 epilogue, a13, K11):
//   rmsnorm      y = bf16(x / sqrt(mean(x^2) + eps) * w)          (fp32 math)
//   rope_append  NeoX rotate-half RoPE on q,k (+bias) at each row's position,
//                q -> bf16 buffer, k/v -> paged KV pool (XOR-swizzled rows)
//   embed        h = float(E[token])
//   silu_mul     m = bf16(SiLU(g) * u)
//   argmax_rows  greedy sampling, lowest index on ties
//   hash_init    counter-based bf16 weight generator
//   checksum     sum_i bits16(w_i) * (2i+1) mod 2^64
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace sgs {

// ------------------------------------------------------------------ RMSNorm
// One block per row, d/8 threads, 8 elements per thread held in registers
// (single pass over x).  The weight row is loaded before griddepcontrol.wait
// (weights never change inside a launch sequence).
template <int VPT>
__global__ void rmsnorm_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                               __nv_bfloat16* __restrict__ y, const int32_t* __restrict__ rows, int T, int d,
                               float eps) {
  pdl_trigger();
  const int i0 = threadIdx.x * 4 * VPT;
  uint2 wb[VPT];
#pragma unroll
  for (int k = 0; k < VPT; ++k) wb[k] = *reinterpret_cast<const uint2*>(w + i0 + 4 * k);
  pdl_wait();
  __shared__ double red[32];
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
  const int src = rows ? rows[t] : t;
  const float* xr = x + (size_t)src * d;
  // fp64 sum of squares and scaling (latency-bound kernel: the arithmetic is
  // free), so the bf16 rounding of x sees the fp32 residual exactly scaled
  float4 v[VPT];
  double ss = 0.0;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    v[k] = *reinterpret_cast<const float4*>(xr + i0 + 4 * k);
    ss += (double)v[k].x * v[k].x + (double)v[k].y * v[k].y + (double)v[k].z * v[k].z + (double)v[k].w * v[k].w;
  }
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
  __syncthreads();  // red[] is reused by the next row
  }
}

cudaError_t rmsnorm(const float* x, const void* w, void* y, const int32_t* rows, int T, int d, float eps,
                    cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  auto W = reinterpret_cast<const __nv_bfloat16*>(w);
  auto Y = reinterpret_cast<__nv_bfloat16*>(y);
  // the sum of squares is a warp/block reduction whose order depends on the
  // thread count; every row uses the same configuration for a given d
  const int grid = T < 1184 ? T : 1184;  // grid-stride over rows beyond 8 CTAs per SM
  if (d % 8 == 0 && d / 8 <= 1024 && d / 8 >= 32)
    return launch_pdl(rmsnorm_kernel<2>, dim3(grid), dim3(d / 8), 0, stream, x, W, Y, rows, T, d, eps);
  if (d % 4 == 0 && d / 4 <= 1024 && d / 4 >= 32)
    return launch_pdl(rmsnorm_kernel<1>, dim3(grid), dim3(d / 4), 0, stream, x, W, Y, rows, T, d, eps);
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ RoPE + KV append
// Work unit = a "duo" of adjacent rotation pairs (i, i+1), i even, of one head:
// duo j of a row -> head = 2j / half, i = 2j % half; q/k heads rotate
// (x_i, x_{i+half}), v heads copy; all loads/stores are 2-wide.  Grid
// (row block, duo group): small batches spread a row over up to 9 CTAs so
// the store issue of a row is not serialised on one SM; large batches use
// few fat CTAs that stride over rows (the CTA launch rate bounds thousands of
// tiny CTAs).  Position, slot, block-table entry, bias and cos/sin are read
// before griddepcontrol.wait; after it every qkv load of the unit is issued
// before any store.  The fp32 qkv row is zeroed after it is read, so the next
// split-K QKV GEMM (fp32 red.add) finds a zeroed accumulator without a memset.
constexpr int ROPE_THREADS = 128, ROPE_U = 4;  // small unroll: the kernel stays far below the I-cache knee
__global__ void __launch_bounds__(ROPE_THREADS)
    rope_append_kernel(float* __restrict__ qkv, const __nv_bfloat16* __restrict__ bias,
                       const int32_t* __restrict__ pos, const int32_t* __restrict__ slot,
                       const int32_t* __restrict__ bt, int max_pages, const float* __restrict__ cs,
                       __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ kv,
                       __nv_bfloat16* __restrict__ k_out, __nv_bfloat16* __restrict__ v_out, int T, int nq, int nkv,
                       int hd, int page, int per, int v_f16) {
  pdl_trigger();
  const int half = hd >> 1;
  const int nh = nq + 2 * nkv;
  const int nduo = nh * half / 2;
  const int rc = hd / 8;
  const int j0 = blockIdx.y * per, j1 = min(j0 + per, nduo);
  bool waited = false;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const int ps = pos[t];
    const int r = ps % page;
    const int sl = slot ? slot[t] : -1;
    const int pg = (kv && sl >= 0) ? bt[(size_t)sl * max_pages + ps / page] : -1;
    float2 b1[ROPE_U], b2[ROPE_U], x1[ROPE_U], x2[ROPE_U];
    float4 c[ROPE_U];
#pragma unroll
    for (int u = 0; u < ROPE_U; ++u) {
      const int j = j0 + threadIdx.x + ROPE_THREADS * u;
      b1[u] = b2[u] = make_float2(0.f, 0.f);
      c[u] = make_float4(1.f, 0.f, 1.f, 0.f);  // (cos, sin) of pairs i and i+1; identity for v heads
      if (j < j1) {
        const int hh = (2 * j) / half, i = 2 * j - hh * half;
        if (bias) {
          b1[u] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(bias + hh * hd + i));
          b2[u] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(bias + hh * hd + i + half));
        }
        if (hh < nq + nkv) c[u] = *reinterpret_cast<const float4*>(cs + ((size_t)ps * half + i) * 2);
      }
    }
    if (!waited) pdl_wait(), waited = true;
    float* row = qkv + (size_t)t * nh * hd;
#pragma unroll
    for (int u = 0; u < ROPE_U; ++u) {
      const int j = j0 + threadIdx.x + ROPE_THREADS * u;
      if (j < j1) {
        const int hh = (2 * j) / half, i = 2 * j - hh * half;
        x1[u] = *reinterpret_cast<const float2*>(row + hh * hd + i);
        x2[u] = *reinterpret_cast<const float2*>(row + hh * hd + i + half);
      }
    }
#pragma unroll
    for (int u = 0; u < ROPE_U; ++u) {
      const int j = j0 + threadIdx.x + ROPE_THREADS * u;
      if (j >= j1) continue;
      const int hh = (2 * j) / half, i = 2 * j - hh * half;
      *reinterpret_cast<float2*>(row + hh * hd + i) = make_float2(0.f, 0.f);
      *reinterpret_cast<float2*>(row + hh * hd + i + half) = make_float2(0.f, 0.f);
      const float a0 = x1[u].x + b1[u].x, a1 = x1[u].y + b1[u].y;  // x_i, x_{i+1}
      const float e0 = x2[u].x + b2[u].x, e1 = x2[u].y + b2[u].y;  // x_{i+half}, x_{i+1+half}
      const float y10 = a0 * c[u].x - e0 * c[u].y, y20 = e0 * c[u].x + a0 * c[u].y;
      const float y11 = a1 * c[u].z - e1 * c[u].w, y21 = e1 * c[u].z + a1 * c[u].w;
      const __nv_bfloat162 o1 = __floats2bfloat162_rn(y10, y11), o2 = __floats2bfloat162_rn(y20, y21);
      if (hh < nq) {
        *reinterpret_cast<__nv_bfloat162*>(q_out + ((size_t)t * nq + hh) * hd + i) = o1;
        *reinterpret_cast<__nv_bfloat162*>(q_out + ((size_t)t * nq + hh) * hd + i + half) = o2;
        continue;
      }
      const int isv = hh >= nq + nkv;
      const int kvh = isv ? hh - nq - nkv : hh - nq;
      if (pg >= 0) {
        __nv_bfloat16* base = kv + (((size_t)pg * nkv + kvh) * 2 + isv) * (size_t)page * hd + (size_t)r * hd;
        const int e1i = i, e2i = i + half;  // even: both elements stay in one 8-element chunk
        *reinterpret_cast<__nv_bfloat162*>(base + ((((e1i >> 3) ^ kv_swz(r, rc)) << 3) + (e1i & 7))) = o1;
        *reinterpret_cast<__nv_bfloat162*>(base + ((((e2i >> 3) ^ kv_swz(r, rc)) << 3) + (e2i & 7))) = o2;
      }
      __nv_bfloat16* cont = isv ? v_out : k_out;
      if (cont) {
        if (isv && v_f16) {  // fp16(bf16 v): exact, the tcgen05 prefill attention's P.V operand
          const __half2 h1 = __floats2half2_rn(__low2float(o1), __high2float(o1));
          const __half2 h2 = __floats2half2_rn(__low2float(o2), __high2float(o2));
          *reinterpret_cast<__half2*>(cont + ((size_t)t * nkv + kvh) * hd + i) = h1;
          *reinterpret_cast<__half2*>(cont + ((size_t)t * nkv + kvh) * hd + i + half) = h2;
        } else {
          *reinterpret_cast<__nv_bfloat162*>(cont + ((size_t)t * nkv + kvh) * hd + i) = o1;
          *reinterpret_cast<__nv_bfloat162*>(cont + ((size_t)t * nkv + kvh) * hd + i + half) = o2;
        }
      }
    }
  }
  if (!waited) pdl_wait();
}

cudaError_t rope_append(const float* qkv, const void* bias, const int32_t* pos, const int32_t* slot,
                        const int32_t* block_table, int max_pages, const float* cos_sin, void* q_out, void* kv,
                        void* k_out, void* v_out, int T, int nq, int nkv, int hd, int page, cudaStream_t stream,
                        int v_f16) {
  if (T <= 0) return cudaSuccess;
  if (hd % 4) return cudaErrorInvalidValue;
  const int nduo = (nq + 2 * nkv) * (hd / 2) / 2;
  const int gmin = (nduo + ROPE_THREADS * ROPE_U - 1) / (ROPE_THREADS * ROPE_U);
  const int gmax = (nduo + ROPE_THREADS - 1) / ROPE_THREADS;
  int G = (4 * 148 + T - 1) / T;  // about 4 CTAs per SM
  G = G < gmin ? gmin : (G > gmax ? gmax : G);
  const int per = (nduo + G - 1) / G;
  int rows = (1184 + G - 1) / G;  // beyond 8 CTAs per SM the CTAs stride over rows
  rows = T < rows ? T : rows;
  return launch_pdl(rope_append_kernel, dim3(rows, G), dim3(ROPE_THREADS), 0, stream, const_cast<float*>(qkv),
                    reinterpret_cast<const __nv_bfloat16*>(bias), pos, slot, block_table, max_pages, cos_sin,
                    reinterpret_cast<__nv_bfloat16*>(q_out), reinterpret_cast<__nv_bfloat16*>(kv),
                    reinterpret_cast<__nv_bfloat16*>(k_out), reinterpret_cast<__nv_bfloat16*>(v_out), T, nq, nkv, hd,
                    page, per, v_f16);
}

// ------------------------------------------------------------------ tensor-parallel greedy sampling
// after the all-reduce (max) of the shards' packed (logit, ~vocab index) keys:
// the token of each row, the keys re-zeroed for the next launch
__global__ void argmax_keys_finalize_kernel(unsigned long long* keys, int rows, const int32_t* slot,
                                            const int32_t* tok_idx, int32_t* last_tok, int32_t* hist, int max_gen) {
  pdl_trigger();
  pdl_wait();
  for (int t = threadIdx.x; t < rows; t += blockDim.x) {
    const unsigned long long k = keys[t];
    keys[t] = 0ull;
    const int s = slot[t];
    if (s >= 0) {
      const int32_t tok = (int32_t)(~(uint32_t)k);
      last_tok[s] = tok;
      hist[(size_t)s * max_gen + tok_idx[t]] = tok;
    }
  }
}

cudaError_t argmax_keys_finalize(unsigned long long* keys, int rows, const int32_t* slot, const int32_t* tok_idx,
                                 int32_t* last_tok, int32_t* hist, int max_gen, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  return launch_pdl(argmax_keys_finalize_kernel, dim3(1), dim3(256), 0, stream, keys, rows, slot, tok_idx, last_tok,
                    hist, max_gen);
}

// ------------------------------------------------------------------ bf16 -> fp16 (exact for the normal fp16 range)
__global__ void bf16_to_f16_kernel(const __nv_bfloat16* __restrict__ src, __half* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2half_rn(__bfloat162float(src[i]));
}

cudaError_t bf16_to_f16(const void* src, void* dst, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  bf16_to_f16_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(src),
                                                 reinterpret_cast<__half*>(dst), n);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ embedding gather
// The table row is gathered before griddepcontrol.wait (the token ids come
// from the host metadata or the previous iteration's sampler, both complete
// before a decode/prefill launch sequence starts); h is written after it.
__global__ void embed_kernel(const __nv_bfloat16* __restrict__ E, const int32_t* __restrict__ tokens,
                             const int32_t* __restrict__ slots, const int32_t* __restrict__ last_tok,
                             float* __restrict__ h, int T, int d) {
  pdl_trigger();
  bool waited = false;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const int sl = slots ? slots[t] : 0;
    const int tok = slots ? (sl >= 0 ? last_tok[sl] : 0) : tokens[t];  // slot -1: padding row
    const __nv_bfloat16* e = E + (size_t)tok * d;
    const int i = threadIdx.x * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (i < d) v = *reinterpret_cast<const uint4*>(e + i);
    if (!waited) pdl_wait(), waited = true;
    if (i >= d) continue;
    float* o = h + (size_t)t * d + i;
    *reinterpret_cast<float4*>(o) = make_float4(__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u),
                                                __uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u));
    *reinterpret_cast<float4*>(o + 4) = make_float4(__uint_as_float(v.z << 16), __uint_as_float(v.z & 0xffff0000u),
                                                    __uint_as_float(v.w << 16), __uint_as_float(v.w & 0xffff0000u));
  }
  if (!waited) pdl_wait();
}

cudaError_t embed(const void* E, const int32_t* tokens, const int32_t* slots, const int32_t* last_tok, float* h,
                  int T, int d, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  if (d % 8 || d / 8 > 1024) return cudaErrorInvalidValue;
  const int threads = (d / 8 + 31) / 32 * 32;
  const int grid = T < 1184 ? T : 1184;
  return launch_pdl(embed_kernel, dim3(grid), dim3(threads), 0, stream, reinterpret_cast<const __nv_bfloat16*>(E),
                    tokens, slots, last_tok, h, T, d);
}

// ------------------------------------------------------------------ SwiGLU
// gu rows use the interleaved gate/up layout: feature i has its gate value at
// column (i/64)*128 + i%64 and its up value 64 columns later.
__global__ void silu_mul_kernel(float* __restrict__ gu, __nv_bfloat16* __restrict__ m, int f) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.y;
  float* row = gu + (size_t)t * 2 * f;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * 2; i < f; i += gridDim.x * blockDim.x * 2) {
    float* g = row + (i / 64) * 128 + (i % 64);
    float* u = g + 64;
    const float2 gv = *reinterpret_cast<const float2*>(g);
    const float2 uv = *reinterpret_cast<const float2*>(u);
    *reinterpret_cast<float2*>(g) = make_float2(0.f, 0.f);  // zeroed for a split-K successor
    *reinterpret_cast<float2*>(u) = make_float2(0.f, 0.f);
    const float s0 = gv.x / (1.f + expf(-gv.x)), s1 = gv.y / (1.f + expf(-gv.y));
    *reinterpret_cast<uint32_t*>(m + (size_t)t * f + i) = pack_bf16x2(s0 * uv.x, s1 * uv.y);
  }
}

cudaError_t silu_mul(const float* gu, void* m, int T, int f, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  int bx = (f / 2 + 255) / 256;
  if (bx > 16) bx = 16;
  return launch_pdl(silu_mul_kernel, dim3(bx, T), dim3(256), 0, stream, const_cast<float*>(gu),
                    reinterpret_cast<__nv_bfloat16*>(m), f);
}

// ------------------------------------------------------------------ greedy sampler
__global__ void __launch_bounds__(1024) argmax_kernel(const float* __restrict__ logits, int V, int32_t* ids,
                                                      const int32_t* __restrict__ slot,
                                                      const int32_t* __restrict__ tok_idx, int32_t* last_tok,
                                                      int32_t* out_hist, int max_gen) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const float* x = logits + (size_t)r * V;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x * 4; i < V; i += blockDim.x * 4) {
    if (i + 3 < V) {
      const float4 v = *reinterpret_cast<const float4*>(x + i);
      if (v.x > bv) bv = v.x, bi = i;
      if (v.y > bv) bv = v.y, bi = i + 1;
      if (v.z > bv) bv = v.z, bi = i + 2;
      if (v.w > bv) bv = v.w, bi = i + 3;
    } else {
      for (int j = i; j < V; ++j)
        if (x[j] > bv) bv = x[j], bi = j;
    }
  }
  // (value desc, index asc) reduction
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) bv = ov, bi = oi;
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = bv, si[threadIdx.x >> 5] = bi;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    bv = threadIdx.x < nw ? sv[threadIdx.x] : -INFINITY;
    bi = threadIdx.x < nw ? si[threadIdx.x] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) bv = ov, bi = oi;
    }
    if (threadIdx.x == 0) {
      if (bi == 0x7fffffff) bi = 0;
      if (ids) ids[r] = bi;
      if (slot && slot[r] >= 0) {  // slot -1: padding row of a CUDA-graph bucket
        const int s = slot[r];
        last_tok[s] = bi;
        out_hist[(size_t)s * max_gen + tok_idx[r]] = bi;
      }
    }
  }
}

cudaError_t argmax_rows(const float* logits, int rows, int V, int32_t* ids, const int32_t* slot,
                        const int32_t* tok_idx, int32_t* last_tok, int32_t* out_hist, int max_gen,
                        cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (V % 4) return cudaErrorInvalidValue;
  return launch_pdl(argmax_kernel, dim3(rows), dim3(1024), 0, stream, logits, V, ids, slot, tok_idx, last_tok,
                    out_hist, max_gen);
}

// ------------------------------------------------------------------ top-p sampler
// DESIGN.md R18: p = softmax(logits / tau) (fp32); nucleus = shortest prefix of
// the tokens ordered by (p desc, id asc) whose mass reaches top_p; u = 24-bit
// uniform from Philox4x32-10(key = seed, ctr = (sample id, step)) scaled by the
// nucleus mass; the sample is the token at which the cumulative mass in that
// order first exceeds u.  No sort: the ordered cumulative mass is located by a
// radix select over the bits of p (positive floats order like their bits), 8
// bits per pass, with a block-wide 256-bin mass histogram.
__device__ __forceinline__ void philox_dev(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                           uint32_t k1, uint32_t* out) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0, c1 = lo1, c2 = n2, c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0, out[1] = c1, out[2] = c2, out[3] = c3;
}

// Largest bit pattern P such that mass(p >= P) >= target (the p value of the
// token at which the ordered cumulative mass reaches target); *above = mass(p > P).
__device__ float radix_mass_select(const float* __restrict__ x, int V, float m, float inv_tau, float target,
                                   uint32_t* P_out, float* above_out, float* hist) {
  uint32_t prefix = 0, mask = 0;
  float above = 0.f;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0.f;
    __syncthreads();
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
      const float p = __expf((x[i] - m) * inv_tau);
      const uint32_t bits = __float_as_uint(p);
      if ((bits & mask) == prefix) atomicAdd(&hist[(bits >> shift) & 255], p);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // first non-empty bucket (descending p) at which the mass reaches the
      // target; if fp32 re-summation at this level falls short of a target
      // that the parent bucket reached, the last non-empty bucket is taken
      float c = above, c_last = above;
      int k = 255, k_last = -1;
      bool found = false;
      for (; k >= 0; --k) {
        const float hk = hist[k];
        if (hk > 0.f) {
          k_last = k, c_last = c;
          if (c + hk >= target) {
            found = true;
            break;
          }
        }
        c += hk;
      }
      if (!found) k = k_last >= 0 ? k_last : 0, c = c_last;
      above = c;
      prefix |= (uint32_t)k << shift;
      mask |= 255u << shift;
      hist[256] = above, reinterpret_cast<uint32_t*>(hist)[257] = prefix;
    }
    __syncthreads();
    above = hist[256];
    prefix = reinterpret_cast<uint32_t*>(hist)[257];
    mask |= 255u << shift;
    __syncthreads();
  }
  *P_out = prefix;
  *above_out = above;
  return __uint_as_float(prefix);
}

__global__ void __launch_bounds__(1024) top_p_kernel(const float* __restrict__ logits, int V, float inv_tau,
                                                     float top_p, uint64_t seed, const uint32_t* __restrict__ sid,
                                                     const int32_t* __restrict__ slot,
                                                     const int32_t* __restrict__ tok_idx, int32_t* ids,
                                                     int32_t* last_tok, int32_t* out_hist, int max_gen) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (slot && slot[r] < 0) return;
  const float* x = logits + (size_t)r * V;
  __shared__ float hist[258];
  __shared__ float red[32];
  __shared__ int cnt[32];
  // max and normaliser
  float mx = -INFINITY;
  for (int i = threadIdx.x; i < V; i += blockDim.x) mx = fmaxf(mx, x[i]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    v = warp_max(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float m = red[0];
  __syncthreads();
  float z = 0.f;
  for (int i = threadIdx.x; i < V; i += blockDim.x) z += __expf((x[i] - m) * inv_tau);
  z = warp_sum(z);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = z;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float Z = red[0];
  __syncthreads();
  // nucleus: tokens with p > theta plus the first k_eq (by id) with p == theta
  uint32_t tb;
  float above;
  const float theta = radix_mass_select(x, V, m, inv_tau, fminf(top_p, 1.f) * Z, &tb, &above, hist);
  const int k_eq = max(1, (int)ceilf((fminf(top_p, 1.f) * Z - above) / theta));
  const float mass = above + (float)k_eq * theta;
  // u in [0, mass)
  const uint64_t sidv = sid ? ((uint64_t)sid[2 * r] | ((uint64_t)sid[2 * r + 1] << 32)) : (uint64_t)r;
  const uint64_t step = tok_idx ? (uint64_t)tok_idx[r] : 0;
  uint32_t rnd[4];
  philox_dev((uint32_t)sidv, (uint32_t)(sidv >> 32), (uint32_t)step, (uint32_t)(step >> 32), (uint32_t)seed,
             (uint32_t)(seed >> 32), rnd);
  const float u = (float)(rnd[0] >> 8) * (1.0f / 16777216.0f) * mass;
  // the token where the ordered cumulative mass first exceeds u
  uint32_t ub;
  float above_u;
  // nextafter: the cumulative mass must strictly exceed u
  const float theta_u = radix_mass_select(x, V, m, inv_tau, __uint_as_float(__float_as_uint(u) + 1), &ub, &above_u,
                                          hist);
  int j = (int)floorf((u - above_u) / theta_u);
  if (ub == tb) j = min(j, k_eq - 1);
  j = max(j, 0);
  // j-th token (ascending id) with p == theta_u
  // (fp32 histogram sums can put j one past the last tied token: then the
  // last token with p == theta_u, the end of that mass interval, is taken)
  __shared__ int chosen, last_eq;
  if (threadIdx.x == 0) chosen = -1, last_eq = 0;
  __syncthreads();
  int base = 0;
  for (int i0 = 0; i0 < V && chosen < 0; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const bool eq = i < V && __float_as_uint(__expf((x[i] - m) * inv_tau)) == ub;
    const unsigned bal = __ballot_sync(0xffffffffu, eq);
    const int wpre = __popc(bal & ((1u << (threadIdx.x & 31)) - 1));
    if ((threadIdx.x & 31) == 0) cnt[threadIdx.x >> 5] = __popc(bal);
    __syncthreads();
    int before = base;
    for (int w = 0; w < (threadIdx.x >> 5); ++w) before += cnt[w];
    int tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += cnt[w];
    if (eq && before + wpre == j) chosen = i;
    if (eq) atomicMax(&last_eq, i);
    __syncthreads();
    base += tot;
  }
  if (threadIdx.x == 0) {
    const int tok = chosen >= 0 ? chosen : last_eq;
    if (ids) ids[r] = tok;
    if (slot) {
      last_tok[slot[r]] = tok;
      out_hist[(size_t)slot[r] * max_gen + tok_idx[r]] = tok;
    }
  }
}

cudaError_t sample_top_p(const float* logits, int rows, int V, float temperature, float top_p, uint64_t seed,
                         const uint32_t* sample_ids, int32_t* ids, const int32_t* slot, const int32_t* tok_idx,
                         int32_t* last_tok, int32_t* out_hist, int max_gen, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (temperature <= 0.f) return argmax_rows(logits, rows, V, ids, slot, tok_idx, last_tok, out_hist, max_gen, stream);
  return launch_pdl(top_p_kernel, dim3(rows), dim3(1024), 0, stream, logits, V, 1.f / temperature, top_p, seed,
                    sample_ids, slot, tok_idx, ids, last_tok, out_hist, max_gen);
}

// ------------------------------------------------------------------ weights
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Physical index of logical element i of a [rows x cols] tensor stored with
// row blocks of `blk` rows every `stride` rows starting at `off` (blk 0:
// contiguous).  The gate/up weights interleave 64-row blocks so
// one 128-row GEMM tile holds the gate and up rows of the same 64 features.
__device__ __forceinline__ int64_t phys_index(int64_t i, int64_t cols, int blk, int stride, int off, int tiled) {
  if (blk == 0 && !tiled) return i;
  const int64_t r = i / cols, c = i - r * cols;
  const int64_t R = blk ? (r / blk) * stride + off + r % blk : r;
  if (!tiled) return R * cols + c;
  return (((R >> 7) * (cols >> 6) + (c >> 6)) << 13) + ((R & 127) << 6) + (c & 63);
}

__global__ void hash_init_kernel(__nv_bfloat16* __restrict__ dst, uint64_t key, int64_t n, int is_norm, int64_t cols,
                                 int blk, int stride, int off, ShardMap sm, int tiled) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    // a tensor-parallel shard holds a window of the full tensor: element i of
    // the shard is element (row0 + i / lcols, col0 + i % lcols) of the full one
    const int64_t g = sm.src_cols ? (sm.row0 + i / sm.lcols) * sm.src_cols + sm.col0 + i % sm.lcols : i;
    const uint64_t h = splitmix64(key + (uint64_t)g);
    const int32_t m = (int32_t)(h >> 40) - (1 << 23);
    const float u = (float)m * (1.0f / 8388608.0f);
    const float v = is_norm ? __fadd_rn(1.0f, __fmul_rn(u, 0.125f)) : __fmul_rn(u, 0.034641016f);
    dst[phys_index(i, cols, blk, stride, off, tiled)] = __float2bfloat16_rn(v);
  }
}

cudaError_t hash_init(void* dst, uint64_t seed, uint64_t tensor_id, int64_t n, int is_norm, cudaStream_t stream,
                      int64_t cols, int blk, int stride, int off, ShardMap sm, int tiled) {
  // key = splitmix64(seed ^ tensor_id * C): computed on the host, same constant as DESIGN.md §3
  uint64_t z = seed ^ (tensor_id * 0xD1B54A32D192ED03ull);
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  const uint64_t key = z ^ (z >> 31);
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  hash_init_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<__nv_bfloat16*>(dst), key, n, is_norm, cols, blk,
                                               stride, off, sm, tiled);
  return cudaGetLastError();
}

__global__ void checksum_kernel(const uint16_t* __restrict__ src, int64_t n, unsigned long long* out, int64_t cols,
                                int blk, int stride, int off, int tiled) {
  unsigned long long acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += (unsigned long long)src[phys_index(i, cols, blk, stride, off, tiled)] * (unsigned long long)(2 * i + 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

cudaError_t checksum_bf16(const void* src, int64_t n, unsigned long long* out_dev, cudaStream_t stream, int64_t cols,
                          int blk, int stride, int off, int tiled) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  checksum_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const uint16_t*>(src), n, out_dev, cols, blk, stride,
                                              off, tiled);
  return cudaGetLastError();
}

// canonical row-major tensor -> its placement (interleaved rows, tiled blocks);
// reads are coalesced, writes land in 128-byte runs
__global__ void relayout_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst, int64_t n, int64_t cols,
                                int blk, int stride, int off, int tiled) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[phys_index(i, cols, blk, stride, off, tiled)] = src[i];
}
// 8 elements (16 bytes) per thread: 8 consecutive columns stay consecutive in
// every placement when cols % 8 == 0 (a 64-column block holds whole groups)
__global__ void relayout8_kernel(const uint4* __restrict__ src, uint16_t* __restrict__ dst, int64_t n8, int64_t cols,
                                 int blk, int stride, int off, int tiled) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n8; j += (int64_t)gridDim.x * blockDim.x)
    *reinterpret_cast<uint4*>(dst + phys_index(8 * j, cols, blk, stride, off, tiled)) = src[j];
}

cudaError_t relayout_bf16(const void* src, void* dst, int64_t n, int64_t cols, int blk, int stride, int off, int tiled,
                          cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const bool vec = n % 8 == 0 && cols % 8 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  const int64_t work = vec ? n / 8 : n;
  int blocks = (int)((work + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (vec)
    relayout8_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint16_t*>(dst),
                                                 n / 8, cols, blk, stride, off, tiled);
  else
    relayout_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const uint16_t*>(src),
                                                reinterpret_cast<uint16_t*>(dst), n, cols, blk, stride, off, tiled);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ block-table deltas
// (slot, index, value) triples: index >= 0 sets block-table entry bt[slot][index];
// index -1 sets the slot's next input token (prefix sharing: a group member's
// first decode row re-feeds the prompt's last token, R26)
__global__ void bt_delta_kernel(int32_t* bt, int max_pages, const int32_t* __restrict__ d, int n,
                                int32_t* last_tok) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (d[3 * i + 1] >= 0)
    bt[(size_t)d[3 * i] * max_pages + d[3 * i + 1]] = d[3 * i + 2];
  else if (last_tok)
    last_tok[d[3 * i]] = d[3 * i + 2];
}

cudaError_t apply_bt_deltas(int32_t* block_table, int max_pages, const int32_t* deltas, int n, cudaStream_t stream,
                            int32_t* last_tok) {
  if (n <= 0) return cudaSuccess;
  bt_delta_kernel<<<(n + 255) / 256, 256, 0, stream>>>(block_table, max_pages, deltas, n, last_tok);
  return cudaGetLastError();
}

// KV page copies (src, dst) in every layer's pool (prefix sharing, R26)
__global__ void copy_kv_pages_kernel(uint8_t* __restrict__ pool, int64_t layer_stride, int64_t page_bytes,
                                     const int32_t* __restrict__ pairs) {
  const int k = blockIdx.x, l = blockIdx.y;
  const uint4* src = reinterpret_cast<const uint4*>(pool + l * layer_stride + (int64_t)pairs[2 * k] * page_bytes);
  uint4* dst = reinterpret_cast<uint4*>(pool + l * layer_stride + (int64_t)pairs[2 * k + 1] * page_bytes);
  for (int64_t i = threadIdx.x; i < page_bytes / 16; i += blockDim.x) dst[i] = src[i];
}

cudaError_t copy_kv_pages(void* pool, int64_t layer_stride, int64_t page_bytes, int n_layers, const int32_t* pairs,
                          int n_pairs, cudaStream_t stream) {
  if (n_pairs <= 0) return cudaSuccess;
  copy_kv_pages_kernel<<<dim3(n_pairs, n_layers), 256, 0, stream>>>(reinterpret_cast<uint8_t*>(pool), layer_stride,
                                                                    page_bytes, pairs);
  return cudaGetLastError();
}

}  // namespace sgs
