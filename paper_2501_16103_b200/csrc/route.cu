// Token-index buckets on device (arXiv 2501.16103 §4.3).
//
// The paper scatters tokens into per-expert buckets with atomics, which
// leaves the order inside a bucket to the hardware.  This build produces the
// same buckets in a canonical, deterministic order — ascending token id
// (reading R3) — so Y rows are reproducible run to run:
//   kernel 1 (grid E): counts[e] = #{(t, j) : topk[t, j] == e}
//   kernel 2 (grid E): row_off[e] = sum_{e' < e} counts[e'];
//                      token_idx[row_off[e] + r] = r-th token routed to e,
//                      ranks from a block-wide ballot/popcount scan over t.
// Negative ids are masked slots (e.g. slots owned by another rank in expert parallelism)
// and are skipped silently.  Invalid entries (id >= E, or an id repeated later in the same
// token's list) are dropped by both kernels and reported in *status.
#include <cuda_runtime.h>

#include <climits>

#include "common.h"

namespace {

constexpr int kCountThreads = 512;
constexpr int kScatterThreads = 1024;

// 1: a valid slot; 0: a masked slot (negative id); -1: invalid (id >= E or a duplicate).
__device__ __forceinline__ int classify(const int32_t* row, int j, int E) {
  const int x = row[j];
  if (x < 0) return 0;
  if (x >= E) return -1;
  for (int i = 0; i < j; ++i)
    if (row[i] == x) return -1;
  return 1;
}
__device__ __forceinline__ bool entry_valid(const int32_t* row, int j, int E) { return classify(row, j, E) == 1; }

__global__ void __launch_bounds__(kCountThreads) route_count_kernel(const int32_t* __restrict__ topk, int T, int k,
                                                                    int E, int32_t* __restrict__ counts,
                                                                    int32_t* __restrict__ status) {
  const int e = blockIdx.x;
  int c = 0;
  int bad = 0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int32_t* row = topk + (int64_t)t * k;
    for (int j = 0; j < k; ++j) {
      const int cl = classify(row, j, E);
      c += cl == 1 && row[j] == e;
      bad |= cl < 0;
    }
  }
  // block reduction
  __shared__ int s[kCountThreads / 32];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  const int any_bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += s[w];
    counts[e] = tot;
    if (e == 0 && status) *status = any_bad ? 1 : 0;
  }
}

__global__ void __launch_bounds__(kScatterThreads) route_scatter_kernel(
    const int32_t* __restrict__ topk, int T, int k, int E, const int32_t* __restrict__ counts,
    int32_t* __restrict__ row_off, int32_t* __restrict__ token_idx, int32_t* __restrict__ slot) {
  const int e = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  __shared__ int s_base;
  __shared__ int s_warp[32];
  if (threadIdx.x == 0) {
    int b = 0;
    for (int i = 0; i < e; ++i) b += counts[i];
    s_base = b;
    row_off[e] = b;
    if (e == E - 1) row_off[E] = b + counts[e];
  }
  __syncthreads();
  int base = s_base;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int t0 = 0; t0 < T; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    int hit = -1;
    if (t < T) {
      const int32_t* row = topk + (int64_t)t * k;
      for (int j = 0; j < k; ++j)
        if (row[j] == e && entry_valid(row, j, E)) hit = j;
    }
    const unsigned m = __ballot_sync(0xffffffffu, hit >= 0);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    int woff = 0, tot = 0;
    for (int w = 0; w < nwarps; ++w) {
      const int c = s_warp[w];
      woff += w < warp ? c : 0;
      tot += c;
    }
    if (hit >= 0) {
      const int pos = base + woff + __popc(m & lt_mask);
      token_idx[pos] = t;
      if (slot) slot[pos] = hit;
    }
    base += tot;
    __syncthreads();
  }
}

}  // namespace

extern "C" moe_status moe_route(const int32_t* topk, int64_t T, int32_t k, int32_t E, int32_t* counts,
                                int32_t* row_off, int32_t* token_idx, int32_t* slot, int32_t* status,
                                void* stream) {
  moe::clear_error();
  if (T < 0 || k < 1 || k > 32 || E < 1 || E > 1024)
    MOE_FAIL(MOE_ERR_INVALID, "moe_route: T=%lld k=%d E=%d outside T>=0, 1<=k<=32, 1<=E<=1024", (long long)T, k, E);
  if (T * k >= INT_MAX) MOE_FAIL(MOE_ERR_CAPACITY, "moe_route: T*k >= 2^31");
  if (!counts || !row_off || (T > 0 && (!topk || !token_idx)))
    MOE_FAIL(MOE_ERR_INVALID, "moe_route: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  route_count_kernel<<<E, kCountThreads, 0, s>>>(topk, (int)T, k, E, counts, status);
  route_scatter_kernel<<<E, kScatterThreads, 0, s>>>(topk, (int)T, k, E, counts, row_off, token_idx, slot);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_route launch: %s", cudaGetErrorString(err));
  return MOE_OK;
}
