// How fast the chip streams W the way a decode step reads it: W = [rows, 14336] bf16
// (Mixtral's N; 8192 rows = two experts of H = 4096, 235 MB), each CTA reads column strips of `cols`
// columns over a range of rows through a 4-stage ring of 3-D TMA boxes (64 columns x 64 rows x cols/64
// chunks per op, the GEMM kernel's one-box-per-stage W load).  Work assignments compared on the same bytes:
//   whole  — one strip of all 4096 rows of one expert per CTA (the 112 whole 128 x 256 tiles of dec1);
//   split  — every strip's rows cut into S parts, units spread over all CTAs (split-K's layout);
//   narrow — narrower strips (fewer columns per CTA) so ~148 CTAs each own whole rows.
// Test instrument only (not part of the library).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o build/strip_probe scripts/strip_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));   \
      exit(1);                                                                    \
    }                                                                             \
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

constexpr int kStages = 4;
constexpr int kN = 14336;

// A unit = (strip, first row, rows); CTA c takes units c, c + G, c + 2G, ... (static stride).
struct Unit { int strip, row0, rows; };

__global__ void __launch_bounds__(64, 1) strip_kernel(const __grid_constant__ CUtensorMap tm, const Unit* units,
                                                     int n_units, int chunks) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      bar_init(su32(&full[s]), 1);
      bar_init(su32(&empty[s]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int slot = chunks * 8192;
  uint32_t g = 0;
  if (tid == 0) {
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const Unit un = units[u];
      for (int r = un.row0; r < un.row0 + un.rows; r += 64, ++g) {
        const int s = g % kStages;
        bar_wait(su32(&empty[s]), ((g / kStages) & 1) ^ 1);
        bar_expect(su32(&full[s]), slot);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
                "r"(su32(smem) + s * slot), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(0), "r"(r), "r"(un.strip * chunks)
            : "memory");
      }
    }
  } else if (tid == 32) {
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const Unit un = units[u];
      for (int r = un.row0; r < un.row0 + un.rows; r += 64, ++g) {
        const int s = g % kStages;
        bar_wait(su32(&full[s]), (g / kStages) & 1);
        bar_arrive(su32(&empty[s]));
      }
    }
  }
}

// Packed W: each 256-column block of an expert stored contiguously ([E][N/256][H][256]); unit = a contiguous
// byte range streamed with 1-D bulk copies of `op_kb` KB per ring slot.
__global__ void __launch_bounds__(64, 1) packed_kernel(const char* base, long long unit_bytes, int n_units, int op_bytes) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      bar_init(su32(&full[s]), 1);
      bar_init(su32(&empty[s]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t g = 0;
  if (tid == 0) {
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      for (long long off = 0; off < unit_bytes; off += op_bytes, ++g) {
        const int s = g % kStages;
        bar_wait(su32(&empty[s]), ((g / kStages) & 1) ^ 1);
        bar_expect(su32(&full[s]), op_bytes);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(smem) + s * op_bytes),
                     "l"(base + (long long)u * unit_bytes + off), "r"(op_bytes), "r"(su32(&full[s]))
                     : "memory");
      }
    }
  } else if (tid == 32) {
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      for (long long off = 0; off < unit_bytes; off += op_bytes, ++g) {
        const int s = g % kStages;
        bar_wait(su32(&full[s]), (g / kStages) & 1);
        bar_arrive(su32(&empty[s]));
      }
    }
  }
}

int main() {
  const long long rows = 8192;                          // two experts of H = 4096
  char* buf;
  CK(cudaMalloc(&buf, rows * kN * 2));
  CK(cudaMemset(buf, 1, rows * kN * 2));
  char* flush;
  CK(cudaMalloc(&flush, 512 << 20));
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  Unit* d_units;
  CK(cudaMalloc(&d_units, sizeof(Unit) * 65536));
  static Unit h_units[65536];
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&](const char* name, int chunks, int parts, int grid) {
    CUtensorMap tm;
    const cuuint64_t d3[3] = {64, (cuuint64_t)rows, (cuuint64_t)(kN / 64)};
    const cuuint64_t s3[2] = {(cuuint64_t)kN * 2, 128};
    const cuuint32_t b3[3] = {64, 64, (cuuint32_t)chunks};
    const cuuint32_t e3[3] = {1, 1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      fprintf(stderr, "encode failed\n");
      exit(1);
    }
    // units: part-major over (expert, strip): unit = part p of strip s of expert x
    const int strips = kN / (64 * chunks);
    int n = 0;
    const int prow = 4096 / parts;
    for (int p = 0; p < parts; ++p)
      for (int x = 0; x < 2; ++x)
        for (int s = 0; s < strips; ++s) h_units[n++] = {s, x * 4096 + p * prow, prow};
    CK(cudaMemcpy(d_units, h_units, sizeof(Unit) * n, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(strip_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * chunks * 8192));
    float best = 1e9f;
    for (int rep = 0; rep < 7; ++rep) {
      CK(cudaMemsetAsync(flush, rep, 512 << 20));
      CK(cudaEventRecord(e0));
      strip_kernel<<<grid, 64, kStages * chunks * 8192>>>(tm, d_units, n, chunks);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0 && ms < best) best = ms;
    }
    CK(cudaGetLastError());
    const double bytes = (double)rows * kN * 2;
    printf("{\"layout\": \"%s\", \"strip_cols\": %d, \"parts\": %d, \"units\": %d, \"ctas\": %d, \"us\": %.2f, "
           "\"tb_s\": %.3f}\n", name, 64 * chunks, parts, n, grid, best * 1e3, bytes / (best * 1e-3) / 1e12);
    fflush(stdout);
  };
  run("whole", 4, 1, 112);                   // dec1's 112 whole 128 x 256 tiles
  run("whole_on_148", 4, 1, nsm);            // same units, 148 CTAs launched (36 idle)
  run("split_S2", 4, 2, nsm);
  run("split_S4", 4, 4, nsm);
  run("split_S5", 4, 5, nsm);
  run("narrow_192", 3, 1, nsm);              // 74 strips per expert (+ remainder: 14336/192 not integral)
  run("narrow_128", 2, 1, nsm);              // 224 strips: 1.51 per CTA
  // packed layout: the same 235 MB as 112 contiguous 2 MB blocks (or 560 / 148-way row splits of them)
  auto runp = [&](const char* name, int n_units, int grid, int op_kb) {
    const long long total = rows * kN * 2;
    const long long ub = total / n_units / (op_kb * 1024) * (op_kb * 1024);
    CK(cudaFuncSetAttribute(packed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * op_kb * 1024));
    float best = 1e9f;
    for (int rep = 0; rep < 7; ++rep) {
      CK(cudaMemsetAsync(flush, rep, 512 << 20));
      CK(cudaEventRecord(e0));
      packed_kernel<<<grid, 64, kStages * op_kb * 1024>>>(buf, ub, n_units, op_kb * 1024);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0 && ms < best) best = ms;
    }
    CK(cudaGetLastError());
    printf("{\"layout\": \"%s\", \"units\": %d, \"ctas\": %d, \"op_kb\": %d, \"us\": %.2f, \"tb_s\": %.3f}\n", name,
           n_units, grid, op_kb, best * 1e3, (double)ub * n_units / (best * 1e-3) / 1e12);
    fflush(stdout);
  };
  runp("packed_whole", 112, 112, 32);
  runp("packed_whole", 112, 112, 48);
  runp("packed_148", 148, nsm, 32);
  runp("packed_148", 148, nsm, 48);
  runp("packed_split5", 560, nsm, 32);
  return 0;
}
