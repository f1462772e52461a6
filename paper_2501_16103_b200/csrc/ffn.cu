// Weighted combine of the MoE FFN layer ("finally sums them up as the output"; DESIGN.md
// R14).  Two small kernels: (1) the inverse of the route's CSR (token, slot) -> row, (2) one
// block row per token: each thread owns 8 output columns (16-byte loads of bf16 / 2 x 16 bytes of
// fp32), accumulates its token's k rows in fp32 in ascending slot order, and stores once.
// HBM-bound: reads sum_e m_e rows of Y once, writes T rows.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <climits>

#include "common.h"
#include "moe_sm100_ffn.h"

namespace {

constexpr int kCombineThreads = 128;

__global__ void combine_inverse_kernel(const int32_t* __restrict__ token_idx, const int32_t* __restrict__ slot,
                                       const int32_t* __restrict__ row_off, int E, int k, int64_t Tk,
                                       int32_t* __restrict__ inv) {
  const int64_t R = __ldg(row_off + E);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < min(R, Tk); r += (int64_t)gridDim.x * blockDim.x)
    inv[(int64_t)__ldg(token_idx + r) * k + __ldg(slot + r)] = (int32_t)r;
}

__device__ __forceinline__ void load8(const void* Y, bool f32, int64_t r, int64_t N, int64_t c, float (&v)[8]) {
  if (f32) {
    const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(Y) + r * N + c);
    const float4 a = __ldg(p), b = __ldg(p + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(Y) + r * N + c));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
}

__global__ void __launch_bounds__(kCombineThreads)
    combine_kernel(const void* __restrict__ Y, int y_f32, int64_t N, int k, const int32_t* __restrict__ inv,
                   const float* __restrict__ w, void* __restrict__ out, int out_f32) {
  const int64_t t = blockIdx.x;
  const int64_t c = ((int64_t)blockIdx.y * kCombineThreads + threadIdx.x) * 8;
  if (c >= N) return;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int j = 0; j < k; ++j) {
    const int r = __ldg(inv + t * k + j);
    if (r < 0) continue;
    const float wj = __ldg(w + t * k + j);
    float v[8];
    load8(Y, y_f32 != 0, r, N, c, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fmaf(wj, v[i], acc[i]);
  }
  if (out_f32) {
    float4* p = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + t * N + c);
    p[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    p[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  } else {
    uint4 q;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + t * N + c) = q;
  }
}

}  // namespace

extern "C" moe_status moe_combine(const void* Y, int32_t y_dtype, int64_t T, int32_t k, int64_t N,
                                  const int32_t* token_idx, const int32_t* slot, const int32_t* row_off, int32_t E,
                                  const float* topk_w, void* out, int32_t out_dtype, void* stream) {
  moe::NvtxRange nvtx("moe_combine");
  moe::clear_error();
  if (T < 0 || k < 1 || k > 32 || E < 1) MOE_FAIL(MOE_ERR_INVALID, "moe_combine: T=%lld k=%d E=%d", (long long)T, k, E);
  if (N <= 0 || N % 8) MOE_FAIL(MOE_ERR_INVALID, "moe_combine: N=%lld must be a positive multiple of 8", (long long)N);
  if (T * k >= INT_MAX) MOE_FAIL(MOE_ERR_CAPACITY, "moe_combine: T*k >= 2^31");
  if ((y_dtype != MOE_DTYPE_BF16 && y_dtype != MOE_DTYPE_F32) || (out_dtype != MOE_DTYPE_BF16 && out_dtype != MOE_DTYPE_F32))
    MOE_FAIL(MOE_ERR_INVALID, "moe_combine: dtype");
  if (T == 0) return MOE_OK;
  if (!Y || !token_idx || !slot || !row_off || !topk_w || !out) MOE_FAIL(MOE_ERR_INVALID, "moe_combine: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t Tk = T * k;
  int32_t* inv = nullptr;
  cudaError_t err = cudaMallocAsync((void**)&inv, sizeof(int32_t) * (size_t)Tk, s);
  if (err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_combine scratch: %s", cudaGetErrorString(err));
  cudaMemsetAsync(inv, 0xff, sizeof(int32_t) * (size_t)Tk, s);
  const int ib = (int)std::min<int64_t>((Tk + 255) / 256, 4 * 148);
  combine_inverse_kernel<<<ib, 256, 0, s>>>(token_idx, slot, row_off, E, k, Tk, inv);
  const dim3 grid((unsigned)T, (unsigned)((N / 8 + kCombineThreads - 1) / kCombineThreads));
  combine_kernel<<<grid, kCombineThreads, 0, s>>>(Y, y_dtype == MOE_DTYPE_F32, N, k, inv, topk_w, out,
                                                  out_dtype == MOE_DTYPE_F32);
  cudaFreeAsync(inv, s);
  err = cudaGetLastError();
  if (err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_combine launch: %s", cudaGetErrorString(err));
  return MOE_OK;
}
