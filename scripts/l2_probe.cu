// L2 -> SM delivery ceiling on B200 for the wide tile's stage pattern.  Test instrument
// only (not part of the library): how many bytes per SM clock can 148 SMs pull out of L2 into shared memory
// with TMA when the data is L2-resident, as a function of the ring (stages x bytes per stage)?  The wide
// 256 x 512 pair tile moves one 16 KB token-row box + one 32 KB W box per CTA per K block; here the same two
// boxes (SW128, same tensor-map shapes) are loaded into a ring and released by a consumer warp with no
// MMA, so the loop runs at the memory system's rate.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o build/l2_probe scripts/l2_probe.cu -lcuda
//   build/l2_probe            (one JSON line per (a_kb, b_kb, stages, ctas))
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e = (x);                                                                         \
    if (e != cudaSuccess) {                                                                      \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));                  \
      exit(1);                                                                                   \
    }                                                                                            \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_expect(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(b), "r"(par)
        : "memory");
  }
}

constexpr int kMaxStages = 12;
constexpr int kH = 4096;          // K
constexpr int kRows = 2048;       // token rows of X (16 MB)
constexpr int kN = 2048;          // W columns (16 MB)

// CTA c walks "tiles" (row tile rt, column block cb) like the persistent kernel: for each tile, the K blocks
// kb = 0..63; per K block one A box (128 rows x 64 K, 16 KB) and one B box (64 K x 256 cols, 32 KB).
__global__ void __launch_bounds__(64, 1) ring_kernel(const __grid_constant__ CUtensorMap tmA,
                                                    const __grid_constant__ CUtensorMap tmB, int stages, int use_a,
                                                    int use_b, int tiles, long long* cycles) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  const int tid = threadIdx.x;
  const uint32_t a_bytes = use_a ? 16384u : 0u, b_bytes = use_b ? 32768u : 0u;
  const uint32_t slot = 49152u;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      bar_init(su32(&full[s]), 1);
      bar_init(su32(&empty[s]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long t0 = clock64();
  const int nkb = kH / 64;
  if (tid == 0) {
    int g = 0;
    for (int t = 0; t < tiles; ++t) {
      const int v = blockIdx.x + t * gridDim.x;
      const int rt = v % (kRows / 128), cb = (v / (kRows / 128)) % (kN / 256);
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % stages;
        bar_wait(su32(&empty[s]), ((g / stages) & 1) ^ 1);
        const uint32_t fb = su32(&full[s]);
        bar_expect(fb, a_bytes + b_bytes);
        const uint32_t dst = su32(smem) + s * slot;
        if (use_a)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
                  "r"(dst), "l"((uint64_t)&tmA), "r"(fb), "r"(kb * 64), "r"(rt * 128)
              : "memory");
        if (use_b)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
                  "r"(dst + 16384u), "l"((uint64_t)&tmB), "r"(fb), "r"(0), "r"(kb * 64), "r"(cb * 4)
              : "memory");
      }
    }
  } else if (tid == 32) {
    int g = 0;
    for (int t = 0; t < tiles; ++t)
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % stages;
        bar_wait(su32(&full[s]), (g / stages) & 1);
        bar_arrive(su32(&empty[s]));
      }
  }
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
}

int main() {
  int nsm = 0;
  CK(cudaSetDevice(0));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  char *X, *W;
  CK(cudaMalloc(&X, (size_t)kRows * kH * 2));
  CK(cudaMalloc(&W, (size_t)kH * kN * 2));
  CK(cudaMemset(X, 1, (size_t)kRows * kH * 2));
  CK(cudaMemset(W, 1, (size_t)kH * kN * 2));
  long long* cyc;
  CK(cudaMalloc(&cyc, 1024 * sizeof(long long)));
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap tmA, tmB;
  {
    const cuuint64_t d[2] = {(cuuint64_t)kH, (cuuint64_t)kRows};
    const cuuint64_t st[1] = {(cuuint64_t)kH * 2};
    const cuuint32_t box[2] = {64, 128};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 1;
  }
  {
    // W [K, N] row-major as {64 columns, K, N / 64}: a box = 64 K rows x 4 chunks of 64 columns (32 KB)
    const cuuint64_t d[3] = {64, (cuuint64_t)kH, (cuuint64_t)(kN / 64)};
    const cuuint64_t st[2] = {(cuuint64_t)kN * 2, 128};
    const cuuint32_t box[3] = {64, 64, 4};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, W, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 1;
  }
  CK(cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 49152 + 1024));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int tiles = 12;   // per CTA: 12 x 64 K blocks
  auto run = [&](int use_a, int use_b, int stages, int ctas) {
    const size_t sm = (size_t)stages * 49152 + 1024;
    float best = 1e9f;
    long long cmax = 0;
    for (int rep = 0; rep < 6; ++rep) {    // rep 0 warms L2 (the 32 MB working set stays resident)
      CK(cudaEventRecord(e0));
      ring_kernel<<<ctas, 64, sm>>>(tmA, tmB, stages, use_a, use_b, tiles, cyc);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0 && ms < best) {
        best = ms;
        long long h[1024];
        CK(cudaMemcpy(h, cyc, ctas * sizeof(long long), cudaMemcpyDeviceToHost));
        cmax = 0;
        for (int i = 0; i < ctas; ++i) cmax = h[i] > cmax ? h[i] : cmax;
      }
    }
    CK(cudaGetLastError());
    const double bytes = (double)ctas * tiles * (kH / 64) * ((use_a ? 16384.0 : 0.0) + (use_b ? 32768.0 : 0.0));
    printf("{\"a_kb\": %d, \"b_kb\": %d, \"stages\": %d, \"ctas\": %d, \"us\": %.2f, \"tbs\": %.3f, "
           "\"bytes_per_sm_clk\": %.2f, \"chip_bytes_per_clk\": %.0f, \"sm_mhz_implied\": %.0f}\n",
           use_a ? 16 : 0, use_b ? 32 : 0, stages, ctas, best * 1e3, bytes / (best * 1e-3) / 1e12,
           bytes / ctas / (double)cmax, bytes / (double)cmax, (double)cmax / (best * 1e3));
    fflush(stdout);
  };
  for (int ctas : {148, 74, 16})
    for (int st : {2, 3, 4}) run(1, 1, st, ctas);
  for (int st : {2, 4}) {
    run(1, 0, st, 148);
    run(0, 1, st, 148);
  }
  return 0;
}
