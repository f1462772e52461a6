// Per-SM HBM streaming rate on B200: how many bytes per second one SM can pull from
// HBM as a function of the bytes it keeps in flight and of the number of SMs streaming at once.
// Test instrument only (not part of the library): answers whether memory-bound MoE tiles (one-token
// experts, decode steps) are limited by the ring depth (latency x bytes in flight), by the TMA path,
// or by a per-SM ceiling.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o build/stream_probe scripts/stream_probe.cu -lcuda
//   build/stream_probe            (prints one JSON line per (mode, ctas, stages))
//
// Modes: tma  — one thread issues 2-D TMA box loads (64 rows x 128 B = 8 KB, W-like strided rows) into a
//               ring of `stages` slots (slot = `boxes` boxes), a consumer warp waits and frees;
//        pf   — the same plus cp.async.bulk.prefetch.tensor (L2) of the next `pf` slots;
//        bulk — 1-D cp.async.bulk of contiguous 8 KB chunks into the same ring;
//        ldg  — 512 threads, LDG.128 with 8 loads in flight per thread (no shared memory).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

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
__device__ __forceinline__ void tma2d(const CUtensorMap* m, uint32_t bar, uint32_t dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(dst),
      "l"((uint64_t)m), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void pf2d(const CUtensorMap* m, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"((uint64_t)m), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

constexpr int kBox = 8192;     // 64 rows x 128 B
constexpr int kMaxStages = 24;

// Each CTA streams `iters` slots of `boxes` boxes from its own region: rows [cta * rows_per_cta, ...),
// 64-row boxes walking down a column band of 64 bf16 (128 B) in a matrix of row stride `ld` elements.
__global__ void __launch_bounds__(64, 1) ring_kernel(const __grid_constant__ CUtensorMap tm, const char* base, int mode,
                                                    int stages, int boxes, int iters, int pf, int rows_per_cta,
                                                    long long per_cta) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      bar_init(su32(&full[s]), 1);
      bar_init(su32(&empty[s]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // CTA c streams a 1 KB wide strip (like a 512-column W tile): strip c % 16 of the 16 KB rows,
  // row block c / 16.
  const int row0 = (blockIdx.x / 16) * rows_per_cta;
  const int colb = (blockIdx.x % 16) * 512;
  const int col_bands = 8;                        // 8 bands of 128 B = the 1 KB strip
  auto coords = [&](int it, int b, int& c0, int& c1) {
    const int idx = it * boxes + b;               // box index: band fastest, then 64-row groups
    c0 = colb + (idx % col_bands) * 64;
    c1 = row0 + (idx / col_bands) * 64;
  };
  if (tid == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      if (mode == 1 && pf > 0) {
        const int pk = it == 0 ? 0 : it + pf - 1;
        for (int q = it == 0 ? 0 : pk; q <= it + pf - 1 && q < iters; ++q)
          for (int b = 0; b < boxes; ++b) {
            int c0, c1;
            coords(q, b, c0, c1);
            pf2d(&tm, c0, c1);
          }
      }
      bar_wait(su32(&empty[s]), ((it / stages) & 1) ^ 1);
      const uint32_t fb = su32(&full[s]);
      bar_expect(fb, boxes * kBox);
      for (int b = 0; b < boxes; ++b) {
        const uint32_t dst = su32(smem) + (s * boxes + b) * kBox;
        int c0, c1;
        coords(it, b, c0, c1);
        if (mode == 2) {                          // contiguous 8 KB chunks of the CTA's own 4 MB
          bulk1d(dst, base + blockIdx.x * per_cta + (long long)(it * boxes + b) * kBox, kBox, fb);
        } else {
          tma2d(&tm, fb, dst, c0, c1);
        }
      }
    }
  } else if (tid == 32) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      bar_wait(su32(&full[s]), (it / stages) & 1);
      bar_arrive(su32(&empty[s]));
    }
  }
}

__global__ void __launch_bounds__(512, 1) ldg_kernel(const int4* __restrict__ src, long long per_cta_vec, int4* sink) {
  const int4* p = src + blockIdx.x * per_cta_vec;
  int4 acc = make_int4(0, 0, 0, 0);
  for (long long i = threadIdx.x; i < per_cta_vec; i += 512 * 8) {
    int4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long j = i + u * 512;
      v[u] = j < per_cta_vec ? __ldcs(p + j) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc.x ^= v[u].x ^ v[u].w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

// Mode 4 ("big"): one 3-D TMA op per box of `chunks` x 8 KB (64 columns x 64 rows x chunks, like the
// library's 4-D W view), `boxes` ops per slot.
__global__ void __launch_bounds__(64, 1) big_kernel(const __grid_constant__ CUtensorMap tm3, int stages, int boxes,
                                                   int chunks, int iters, int rows_per_cta) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      bar_init(su32(&full[s]), 1);
      bar_init(su32(&empty[s]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int row0 = (blockIdx.x / 16) * rows_per_cta;
  const int chunk0 = (blockIdx.x % 16) * 8;           // the CTA's 1 KB strip = 8 chunks of 64 columns
  const int per_row_group = 8 / chunks;                // ops per 64-row group
  const int slot_bytes = boxes * chunks * kBox;
  if (tid == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      bar_wait(su32(&empty[s]), ((it / stages) & 1) ^ 1);
      const uint32_t fb = su32(&full[s]);
      bar_expect(fb, slot_bytes);
      for (int b = 0; b < boxes; ++b) {
        const int idx = it * boxes + b;
        const int c2 = chunk0 + (idx % per_row_group) * chunks;
        const int c1 = row0 + (idx / per_row_group) * 64;
        const uint32_t dst = su32(smem) + s * slot_bytes + b * chunks * kBox;
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
                "r"(dst), "l"((uint64_t)&tm3), "r"(fb), "r"(0), "r"(c1), "r"(c2)
            : "memory");
      }
    }
  } else if (tid == 32) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      bar_wait(su32(&full[s]), (it / stages) & 1);
      bar_arrive(su32(&empty[s]));
    }
  }
}

__global__ void __launch_bounds__(512, 1) ldg16_kernel(const int4* __restrict__ src, long long per_cta_vec, int4* sink) {
  const int4* p = src + blockIdx.x * per_cta_vec;
  int4 acc = make_int4(0, 0, 0, 0);
  for (long long i = threadIdx.x; i < per_cta_vec; i += 512 * 16) {
    int4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const long long j = i + u * 512;
      v[u] = j < per_cta_vec ? __ldcs(p + j) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) acc.x ^= v[u].x ^ v[u].w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

int main() {
  int dev = 0, nsm = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  // matrix: rows x 8192 bf16 (16 KB per row, like W's N-contiguous rows), 2 GB
  const long long cols = 8192, rows = 10 * 4096;   // 16 strips x 10 row blocks of 4096 rows: 148 CTAs x 4 MB
  const long long ld_bytes = cols * 2;
  char* buf;
  CK(cudaMalloc(&buf, rows * ld_bytes));
  CK(cudaMemset(buf, 1, rows * ld_bytes));
  char* flush;
  CK(cudaMalloc(&flush, 512 << 20));
  int4* sink;
  CK(cudaMalloc(&sink, 64));
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
  const cuuint32_t box[2] = {64, 64};
  const cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    fprintf(stderr, "encode failed\n");
    return 1;
  }
  CK(cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CUtensorMap tm3;
  {
    const cuuint64_t d3[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
    const cuuint64_t s3[2] = {(cuuint64_t)ld_bytes, 128};
    const cuuint32_t b3[3] = {64, 64, 1};
    const cuuint32_t e3[3] = {1, 1, 1};
    for (int ch : {1}) (void)ch;
    if (enc(&tm3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      fprintf(stderr, "encode3 failed\n");
      return 1;
    }
  }
  auto make3 = [&](int chunks) {
    CUtensorMap m;
    const cuuint64_t d3[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
    const cuuint64_t s3[2] = {(cuuint64_t)ld_bytes, 128};
    const cuuint32_t b3[3] = {64, 64, (cuuint32_t)chunks};
    const cuuint32_t e3[3] = {1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return m;
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&](const char* name, int mode, int ctas, int stages, int boxes, int pf) {
    // each CTA streams 4 MB
    const long long per_cta = 4ll << 20;
    const int iters = (int)(per_cta / ((long long)boxes * kBox));
    const int rows_per_cta = (int)(per_cta / (8 * 128));   // 1 KB wide strip
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemsetAsync(flush, rep, 512 << 20));        // evict, then read so no dirty line is left
      ldg_kernel<<<128, 512>>>(reinterpret_cast<const int4*>(flush), (512ll << 20) / 128 / 16, sink);
      CK(cudaEventRecord(e0));
      if (mode == 3)
        ldg_kernel<<<ctas, 512>>>(reinterpret_cast<const int4*>(buf), per_cta / 16, sink);
      else if (mode == 5)
        ldg16_kernel<<<ctas, 512>>>(reinterpret_cast<const int4*>(buf), per_cta / 16, sink);
      else if (mode == 4) {
        const int chunks = pf;                          // reused argument: chunks per op
        CUtensorMap m = make3(chunks);
        big_kernel<<<ctas, 64, stages * boxes * chunks * kBox>>>(m, stages, boxes, chunks,
                                                                  (int)(per_cta / ((long long)boxes * chunks * kBox)),
                                                                  rows_per_cta);
      }
      else
        ring_kernel<<<ctas, 64, stages * boxes * kBox>>>(tm, buf, mode, stages, boxes, iters, pf, rows_per_cta, per_cta);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    const double gbs = (double)per_cta * ctas / (best * 1e-3) / 1e9;
    printf("{\"mode\": \"%s\", \"ctas\": %d, \"stages\": %d, \"slot_kb\": %d, \"in_flight_kb\": %d, \"pf\": %d, "
           "\"us\": %.2f, \"total_gbs\": %.1f, \"per_sm_gbs\": %.1f}\n",
           name, ctas, stages, boxes * 8 * (mode == 4 ? pf : 1), stages * boxes * 8 * (mode == 4 ? pf : 1), pf,
           best * 1e3, gbs, gbs / ctas);
    fflush(stdout);
  };
  const char* which = getenv("PROBE_SET");
  if (which && which[0] == '2') {
    for (int ctas : {8, 74, 148}) {
      // (stages, ops per slot, chunks per op): bytes per op, per barrier phase, in flight
      const int cfgs[][3] = {{4, 1, 4}, {4, 4, 1}, {6, 1, 4}, {2, 2, 4}, {3, 2, 4}, {2, 1, 8}, {3, 1, 8},
                             {2, 8, 1}, {12, 1, 2}, {6, 2, 2}, {24, 1, 1}, {3, 3, 2}, {2, 3, 4}};
      for (auto& c : cfgs) {
        char name[64];
        snprintf(name, sizeof(name), "big_op%dkb_x%d", c[2] * 8, c[1]);
        run(name, 4, ctas, c[0], c[1], c[2]);
      }
      run("ldg", 3, ctas, 0, 1, 0);
      run("ldg16", 5, ctas, 0, 1, 0);
    }
    return 0;
  }
  for (int ctas : {8, 40, 74, 112, 148}) {
    for (int st : {2, 4, 8, 12, 16, 24}) run("tma", 0, ctas, st, 1, 0);
    for (int st : {2, 4, 6}) run("tma_slot32k", 0, ctas, st, 4, 0);
    for (int pf : {8, 32}) run("tma_pf", 1, ctas, 4, 1, pf);
    for (int st : {4, 12, 24}) run("bulk", 2, ctas, st, 1, 0);
    run("ldg", 3, ctas, 0, 1, 0);
  }
  return 0;
}
