// Token-index buckets on device (arXiv 2501.16103 §4.3), optionally fused with
// the device-side planner.
//
// The paper scatters tokens into per-expert buckets with atomics, which leaves the
// order inside a bucket to the hardware.  This build produces the same buckets in a
// canonical, deterministic order — ascending token id (reading R3) — so Y rows are
// reproducible run to run.
//
// Up to kOneBlockMaxEntries (T*k) routing entries: ONE single-block launch (route_one_block_kernel).
// Warp w owns a contiguous range of the (token, slot) entries; per 32-entry round,
// __match_any_sync groups the lanes routed to the same expert, so each group costs one
// shared-memory add (no atomics contention however skewed the routing); pass 1 counts per
// (warp, expert), one scan gives every (warp, expert) its first CSR row (and the plan, with
// plan_body), pass 2 replays the rounds and writes each entry at base + its rank in the group.
//
// Larger batches, over 1024-token chunks (three launches):
//   A (grid = chunks):            per-chunk expert histogram (shared-memory counters) and input
//                                 validation;
//   B (one block, thread = expert): counts[e], row_off = exclusive scan, per-(chunk, expert)
//                                 start offsets; with a plan, the compressed mapping as well
//                                 (the device planner body, P:142 / P:144);
//   C (grid = chunks x experts):  stable compaction of the chunk's tokens routed to the expert
//                                 (ballot / popcount ranks) into token_idx / slot.
// Negative ids are masked slots (expert parallelism: slots owned by another rank) and are
// skipped silently.  Invalid entries (id >= E, or an id repeated later in the same token's
// list) are dropped consistently by A and C and reported in *status.
#include <cuda_runtime.h>

#include <climits>

#include "common.h"
#include "plan_body.cuh"
#include "sm100_ptx.cuh"

namespace moe {
void plan_shape(const moe_plan* p, int32_t* E, int32_t* H, int32_t* N, int32_t* bm, int32_t* bn, uint32_t* flags);
int32_t* plan_blob_dev_mut(moe_plan* p);
void plan_set_device_mode(moe_plan* p, bool on);
}  // namespace moe

namespace {

constexpr int kChunk = 1024;         // tokens per chunk (= threads of kernels A and C)
constexpr int kMaxE = 1024;
constexpr int kScanSmem = 6144;      // ints of the chunk histogram staged in shared memory (static smem budget)
static_assert(kChunk == moe::dplan::kPlanThreads, "route_count_scan_kernel: one thread per chunk token");
constexpr int64_t kOneBlockMaxEntries = 65536;   // one block's two passes stay under ~10 us up to here
constexpr int kOneBlockWarps = moe::dplan::kPlanThreads / 32;

// 1: a valid slot; 0: a masked slot (negative id); -1: invalid (id >= E or a duplicate).
__device__ __forceinline__ int classify(const int32_t* row, int j, int E) {
  const int x = row[j];
  if (x < 0) return 0;
  if (x >= E) return -1;
  for (int i = 0; i < j; ++i)
    if (row[i] == x) return -1;
  return 1;
}

__global__ void __launch_bounds__(kChunk) route_hist_kernel(const int32_t* __restrict__ topk, int T, int k, int E,
                                                           int32_t* __restrict__ chunk_counts,
                                                           int32_t* __restrict__ status) {
  __shared__ int hist[kMaxE];
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int t = blockIdx.x * kChunk + threadIdx.x;
  int bad = 0;
  if (t < T) {
    const int32_t* row = topk + (int64_t)t * k;
    for (int j = 0; j < k; ++j) {
      const int cl = classify(row, j, E);
      if (cl == 1) atomicAdd(&hist[row[j]], 1);
      bad |= cl < 0;
    }
  }
  const int any_bad = __syncthreads_or(bad);
  for (int e = threadIdx.x; e < E; e += blockDim.x) chunk_counts[(int64_t)blockIdx.x * E + e] = hist[e];
  if (any_bad && threadIdx.x == 0 && status) atomicOr(status, 1);
}

__global__ void __launch_bounds__(moe::dplan::kPlanThreads)
    route_scan_kernel(int32_t* __restrict__ chunk_counts, int n_chunks, int E, int32_t* __restrict__ counts,
                      int32_t* __restrict__ row_off, int H, int N, int bm, int bn, uint32_t flags,
                      int32_t* __restrict__ blob) {
  __shared__ long long s_warp[32];
  __shared__ int s_cc[kScanSmem];                    // the chunk x expert histogram, when it fits
  const int e = threadIdx.x;
  const int64_t cells = (int64_t)n_chunks * E;
  const bool staged = cells <= kScanSmem;
  if (staged)                                        // one coalesced pass instead of n_chunks serial loads
    for (int i = threadIdx.x; i < cells; i += blockDim.x) s_cc[i] = chunk_counts[i];
  __syncthreads();
  long long tot = 0;
  if (e < E)
    for (int c = 0; c < n_chunks; ++c) tot += staged ? s_cc[c * E + e] : chunk_counts[(int64_t)c * E + e];
  long long all;
  const long long incl = moe::dplan::block_scan_incl(tot, s_warp, &all);
  if (e < E) {
    long long run = incl - tot;                      // row_off[e]
    counts[e] = (int32_t)tot;
    row_off[e] = (int32_t)run;
    for (int c = 0; c < n_chunks; ++c) {             // chunk (c, e) starts at row_off[e] + earlier chunks
      const int64_t i = (int64_t)c * E + e;
      const long long n = staged ? s_cc[i] : chunk_counts[i];
      if (staged) s_cc[i] = (int32_t)run;
      else chunk_counts[i] = (int32_t)run;
      run += n;
    }
  }
  __syncthreads();
  if (staged)
    for (int i = threadIdx.x; i < cells; i += blockDim.x) chunk_counts[i] = s_cc[i];
  if (e == 0) row_off[E] = (int32_t)all;
  if (blob) moe::dplan::plan_body(e < E ? tot : 0, E, H, N, bm, bn, flags, blob);
}

// One block (kPlanThreads threads) for T*k <= kOneBlockMaxEntries; dynamic shared memory holds
// the per-(warp, expert) counters: kOneBlockWarps * E ints.
__global__ void __launch_bounds__(moe::dplan::kPlanThreads)
    route_one_block_kernel(const int32_t* __restrict__ topk, int T, int k, int E, int32_t* __restrict__ counts,
                           int32_t* __restrict__ row_off, int32_t* __restrict__ token_idx,
                           int32_t* __restrict__ slot, int32_t* __restrict__ status, int H, int N, int bm, int bn,
                           uint32_t flags, int32_t* __restrict__ blob) {
  extern __shared__ int s_we[];                      // [kOneBlockWarps][E]: counts, then running CSR rows
  __shared__ long long s_warp[32];
  moe::ptx::pdl_launch_dependents();                 // the GEMM prologue may start; it waits for us
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kOneBlockWarps * E; i += blockDim.x) s_we[i] = 0;
  __syncthreads();
  const int n = T * k;
  const int per = ((n + kOneBlockWarps - 1) / kOneBlockWarps + 31) & ~31;   // entries per warp (whole rounds)
  const int i0 = warp * per, i1 = min(n, i0 + per);
  int* my = s_we + warp * E;
  // Expert of entry i, or -1 (masked slot) / -2 (invalid: id >= E or repeated in its token's row).
  auto expert_of = [&](int i) -> int {
    if (i >= i1) return -1;
    const int t = i / k, j = i - t * k;
    const int cl = classify(topk + (int64_t)t * k, j, E);
    return cl == 1 ? __ldg(topk + i) : (cl == 0 ? -1 : -2);
  };
  int bad = 0;
  for (int b = i0; b < i1; b += 32) {                // pass 1: per-(warp, expert) counts
    const int e = expert_of(b + lane);
    bad |= e == -2;
    const unsigned grp = __match_any_sync(0xffffffffu, e);
    if (e >= 0 && lane == __ffs(grp) - 1) my[e] += __popc(grp);
    __syncwarp();
  }
  const int any_bad = __syncthreads_or(bad);
  if (threadIdx.x == 0 && status) *status = any_bad ? 1 : 0;
  const int e = threadIdx.x;                         // thread = expert
  long long tot = 0;
  if (e < E)
    for (int w = 0; w < kOneBlockWarps; ++w) tot += s_we[w * E + e];
  long long all;
  const long long incl = moe::dplan::block_scan_incl(tot, s_warp, &all);
  if (e < E) {
    long long run = incl - tot;                      // row_off[e]
    counts[e] = (int32_t)tot;
    row_off[e] = (int32_t)run;
    for (int w = 0; w < kOneBlockWarps; ++w) {       // warp w's entries for e start here
      const int c = s_we[w * E + e];
      s_we[w * E + e] = (int32_t)run;
      run += c;
    }
  }
  if (e == 0) row_off[E] = (int32_t)all;
  __syncthreads();
  for (int b = i0; b < i1; b += 32) {                // pass 2: stable placement (entry order = token order)
    const int i = b + lane;
    const int x = expert_of(i);
    const unsigned grp = __match_any_sync(0xffffffffu, x);
    if (x >= 0) {
      const int pos = my[x] + __popc(grp & ((1u << lane) - 1u));
      token_idx[pos] = i / k;
      if (slot) slot[pos] = i - (i / k) * k;
    }
    __syncwarp();
    if (x >= 0 && lane == __ffs(grp) - 1) my[x] += __popc(grp);
    __syncwarp();
  }
  if (blob) moe::dplan::plan_body(e < E ? tot : 0, E, H, N, bm, bn, flags, blob);
}

__global__ void __launch_bounds__(kChunk) route_scatter_kernel(const int32_t* __restrict__ topk, int T, int k, int E,
                                                              const int32_t* __restrict__ chunk_off,
                                                              int32_t* __restrict__ token_idx,
                                                              int32_t* __restrict__ slot) {
  moe::ptx::pdl_launch_dependents();               // let the GEMM's prologue start (it waits for us)
  const int c = blockIdx.x, e = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int s_warp[kChunk / 32];
  const int t = c * kChunk + threadIdx.x;
  int hit = -1;
  if (t < T) {
    const int32_t* row = topk + (int64_t)t * k;
    for (int j = 0; j < k; ++j)
      if (row[j] == e && classify(row, j, E) == 1) hit = j;
  }
  const unsigned m = __ballot_sync(0xffffffffu, hit >= 0);
  if (lane == 0) s_warp[warp] = __popc(m);
  __syncthreads();
  if (hit >= 0) {
    int pos = chunk_off[(int64_t)c * E + e] + __popc(m & ((1u << lane) - 1u));
    for (int w = 0; w < warp; ++w) pos += s_warp[w];
    token_idx[pos] = t;
    if (slot) slot[pos] = hit;
  }
}

moe_status route_impl(const int32_t* topk, int64_t T, int32_t k, int32_t E, int32_t* counts, int32_t* row_off,
                      int32_t* token_idx, int32_t* slot, int32_t* status, moe_plan* plan, void* stream) {
  moe::clear_error();
  if (T < 0 || k < 1 || k > 32 || E < 1 || E > kMaxE)
    MOE_FAIL(MOE_ERR_INVALID, "moe_route: T=%lld k=%d E=%d outside T>=0, 1<=k<=32, 1<=E<=1024", (long long)T, k, E);
  if (T * k >= INT_MAX) MOE_FAIL(MOE_ERR_CAPACITY, "moe_route: T*k >= 2^31");
  if (!counts || !row_off || (T > 0 && (!topk || !token_idx))) MOE_FAIL(MOE_ERR_INVALID, "moe_route: null pointer");
  int32_t pE = E, pH = 0, pN = 0, pbm = 0, pbn = 0;
  uint32_t pflags = 0;
  if (plan) {
    moe::plan_shape(plan, &pE, &pH, &pN, &pbm, &pbn, &pflags);
    if (pE != E) MOE_FAIL(MOE_ERR_INVALID, "moe_route_plan: plan has E=%d, routing E=%d", pE, E);
  }
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* blob = plan ? moe::plan_blob_dev_mut(plan) : nullptr;
  cudaError_t err = cudaSuccess;
  if (T * k <= kOneBlockMaxEntries) {
    const size_t smem = sizeof(int) * (size_t)kOneBlockWarps * E;
    static cudaError_t attr = cudaFuncSetAttribute(route_one_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)(sizeof(int) * kOneBlockWarps * kMaxE));
    if (attr != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_route: cudaFuncSetAttribute: %s", cudaGetErrorString(attr));
    route_one_block_kernel<<<1, moe::dplan::kPlanThreads, smem, s>>>(topk, (int)T, k, E, counts, row_off, token_idx,
                                                                     slot, status, pH, pN, pbm, pbn, pflags, blob);
    err = cudaGetLastError();
    if (err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_route launch: %s", cudaGetErrorString(err));
    if (plan) moe::plan_set_device_mode(plan, true);
    return MOE_OK;
  }
  const int n_chunks = (int)std::max<int64_t>(1, (T + kChunk - 1) / kChunk);
  int32_t* chunk = nullptr;
  err = cudaMallocAsync((void**)&chunk, sizeof(int32_t) * (size_t)n_chunks * E, s);
  if (err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_route scratch: %s", cudaGetErrorString(err));
  {
    if (status) cudaMemsetAsync(status, 0, sizeof(int32_t), s);
    route_hist_kernel<<<n_chunks, kChunk, 0, s>>>(topk, (int)T, k, E, chunk, status);
    route_scan_kernel<<<1, moe::dplan::kPlanThreads, 0, s>>>(chunk, n_chunks, E, counts, row_off, pH, pN, pbm, pbn,
                                                             pflags, blob);
  }
  if (T > 0) route_scatter_kernel<<<dim3(n_chunks, E), kChunk, 0, s>>>(topk, (int)T, k, E, chunk, token_idx, slot);
  cudaFreeAsync(chunk, s);
  err = cudaGetLastError();
  if (err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_route launch: %s", cudaGetErrorString(err));
  if (plan) moe::plan_set_device_mode(plan, true);
  return MOE_OK;
}

}  // namespace

extern "C" moe_status moe_route(const int32_t* topk, int64_t T, int32_t k, int32_t E, int32_t* counts,
                                int32_t* row_off, int32_t* token_idx, int32_t* slot, int32_t* status,
                                void* stream) {
  return route_impl(topk, T, k, E, counts, row_off, token_idx, slot, status, nullptr, stream);
}

extern "C" moe_status moe_route_plan(const int32_t* topk, int64_t T, int32_t k, int32_t E, int32_t* counts,
                                     int32_t* row_off, int32_t* token_idx, int32_t* slot, int32_t* status,
                                     moe_plan* plan, void* stream) {
  if (!plan) MOE_FAIL(MOE_ERR_INVALID, "moe_route_plan: null plan");
  return route_impl(topk, T, k, E, counts, row_off, token_idx, slot, status, plan, stream);
}
