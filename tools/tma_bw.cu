// TMA load-bandwidth microbenchmark (design study for the GEMM pipeline):
// every CTA streams `iters` 2-D tiles (box 64 bf16 x ROWS, 128-byte swizzle)
// through an S-stage shared-memory ring; a consumer warp only waits on the
// full barrier and releases the slot.  Modes: 0 = each CTA reads its own
// rows of a buffer larger than L2 (HBM stream), 1 = all CTAs read the same
// 2 MB region (L2-resident), 2 = the HBM stream of mode 0 over a tiled copy
// of the matrix in which every (ROWS x 64) box is one contiguous block (a
// 4-D tensor map; the shared-memory image is the same).  Prints GB/s per
// configuration.  `tma_bw tiled` runs only modes 0 and 2.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tools/tma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <string>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(96) tma_stream(const __grid_constant__ CUtensorMap tm, int stages, int iters,
                                                 int box_rows, int mode, int rows_total, unsigned long long* sink,
                                                 int kc, int producers, const void* gbase) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int box_bytes = box_rows * 128 * kc;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * box_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int row_tiles = rows_total / box_rows;
  const int pid = threadIdx.x == 0 ? 0 : (threadIdx.x == 64 ? 1 : -1);
  if (pid >= 0 && pid < producers) {
    for (int i = pid; i < iters; i += producers) {
      const int s = i % stages;
      if (i >= stages) {
        const uint32_t par = ((i / stages) - 1) & 1;
        asm volatile(
            "{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}\n" ::"r"(
                su32(&empty[s])),
            "r"(par)
            : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(box_bytes)
                   : "memory");
      // mode 0: CTA-private row bands (distinct data, HBM); mode 1: 2 MB shared window (L2)
      const int kt = 64 / kc;  // boxes per row band (K = 4096 = 64 chunks)
      int x, y;
      if (mode == 0 || mode >= 2) {
        const int band = (blockIdx.x * 3 + i / kt) % row_tiles;
        x = (i % kt) * kc, y = band * box_rows;
      } else {
        const int win = (2 << 20) / box_bytes;
        const int t = (blockIdx.x * 7 + i) % win;
        x = (t % kt) * kc, y = (t / kt) * box_rows;
      }
      if (mode == 3) {  // 1-D bulk copy of the same contiguous block (no tensor map, no swizzle)
        const uint8_t* g = reinterpret_cast<const uint8_t*>(gbase) +
                           ((size_t)(y / box_rows) * (4096 / 64) + x) * (size_t)(box_rows * 128);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(smem + (size_t)s * box_bytes)),
            "l"(g), "r"(box_bytes), "r"(su32(&full[s]))
            : "memory");
      } else if (mode == 2)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
            "[%2];" ::"r"(su32(smem + (size_t)s * box_bytes)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&full[s])), "r"(0), "r"(0), "r"(x), "r"(y / box_rows)
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
            "[%2];" ::"r"(su32(smem + (size_t)s * box_bytes)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&full[s])), "r"(0), "r"(y), "r"(x)
            : "memory");
    }
  } else if (threadIdx.x == 32) {
    unsigned long long acc = 0;
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      const uint32_t par = (i / stages) & 1;
      asm volatile(
          "{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(
              su32(&full[s])),
          "r"(par)
          : "memory");
      acc += smem[(size_t)s * box_bytes + (i & 127)];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    if (acc == 0xFFFFFFFFFFFFull) *sink = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const bool tiled_only = argc > 1 && std::string(argv[1]) == "tiled";
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fnp);
  const int K = 4096;
  const int rows = 65536;  // 512 MB of bf16 >> L2
  void* buf = nullptr;
  cudaMalloc(&buf, (size_t)rows * K * 2);
  cudaMemset(buf, 1, (size_t)rows * K * 2);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Cfg { int mode, box_rows, kc, per_sm, stages, producers; };
  std::vector<Cfg> cfgs;
  for (int mode : {0, 1, 2, 3})
    for (int box_rows : {128, 256})
      for (int kc : {1, 2, 4})
        for (int per_sm : {1, 2})
          for (int producers : {1, 2})
            for (int stages : {3, 6}) cfgs.push_back({mode, box_rows, kc, per_sm, stages, producers});
  for (const Cfg& c : cfgs) {
    const int box_bytes = c.box_rows * 128 * c.kc;
    const size_t smem = 1024 + (size_t)c.stages * box_bytes + 2 * c.stages * 8;
    if (smem * c.per_sm > 226 * 1024 || c.box_rows * c.kc > 256 * 2 + 0 && c.kc * c.box_rows > 512) continue;
    if (tiled_only && c.mode == 1) continue;
    CUtensorMap tm;
    CUresult er;
    if (c.mode >= 2) {  // [rows / R][K / 64][R][64]: one contiguous block per box
      const cuuint64_t R = (cuuint64_t)c.box_rows;
      cuuint64_t dims[4] = {64, R, (cuuint64_t)(K / 64), (cuuint64_t)rows / R};
      cuuint64_t strides[3] = {128, R * 128, (cuuint64_t)(K / 64) * R * 128};
      cuuint32_t box[4] = {64, (cuuint32_t)c.box_rows, (cuuint32_t)c.kc, 1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      er = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(K / 64)};
      cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
      cuuint32_t box[3] = {64, (cuuint32_t)c.box_rows, (cuuint32_t)c.kc};
      cuuint32_t es[3] = {1, 1, 1};
      er = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (er != CUDA_SUCCESS) {
      printf("encode failed kc=%d rows=%d\n", c.kc, c.box_rows);
      continue;
    }
    const int grid = sms * c.per_sm;
    const int iters = (int)((256LL << 20) * (c.mode == 1 ? 2 : 1) / ((long long)grid * box_bytes));
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      tma_stream<<<grid, 96, smem>>>(tm, c.stages, iters, c.box_rows, c.mode, rows, sink, c.kc, c.producers, buf);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best) best = ms;
    }
    const double bytes = (double)grid * iters * box_bytes;
    printf("{\"mode\": \"%s\", \"box_KB\": %d, \"box_rows\": %d, \"kc\": %d, \"ctas_per_sm\": %d, \"producers\": %d, "
           "\"stages\": %d, \"GBs\": %.1f, \"GBs_per_sm\": %.1f}\n",
           c.mode == 0 ? "hbm" : c.mode == 1 ? "l2" : c.mode == 2 ? "hbm_tiled" : "hbm_bulk1d", box_bytes / 1024, c.box_rows, c.kc, c.per_sm, c.producers, c.stages,
           bytes / best / 1e6, bytes / best / 1e6 / sms);
    fflush(stdout);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
