// Token-index buckets on device (arXiv 2501.16103 §4.3), optionally fused with
// the device-side planner.
//
// The paper scatters tokens into per-expert buckets with atomics, which leaves the
// order inside a bucket to the hardware.  This build produces the same buckets in a
// canonical, deterministic order — ascending token id (reading R3) — so Y rows are
// reproducible run to run.
//
// Over 1024-token chunks:
//   A (grid = chunks):  per-chunk expert histogram — thread = token, one warp-aggregated shared
//                       atomic per (round, expert group) via __match_any_sync — and a per-chunk
//                       "invalid entry seen" flag;
//   B (grid = chunks x experts, launched with programmatic dependent launch behind A): every
//                       block derives its (chunk, expert) first CSR row from the histograms (a
//                       block scan over the per-expert totals) and compacts the chunk's tokens
//                       routed to its expert in token order (ballot / popcount ranks).  Block
//                       (0, 0) writes counts / row_off and, with a plan, runs the device planner
//                       body (P:142 / P:144).
// When chunks x experts exceeds kPlaceMaxCells, the scan runs once in a single-block kernel
// between A and the compaction (three launches).  Small batches (T <= 1024 tokens, E <= 16,
// k <= 8: the decode regime) take one single-block kernel instead (route_small_kernel: thread =
// token, experts in turn, ballot / popcount ranks; no scratch allocation).
// Negative ids are masked slots (expert parallelism: slots owned by another rank) and are
// skipped silently.  Invalid entries (id >= E, or an id repeated later in the same token's
// list) are dropped consistently by A and C and reported in *status.
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>

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
constexpr int kPlaceMaxCells = 16384;   // route_place_kernel: each block reads the chunks x experts histogram
constexpr int kRegK = 8;                 // top-k up to 8: a row / a warp's rounds live in registers

// 1: a valid slot; 0: a masked slot (negative id); -1: invalid (id >= E or a duplicate).
__device__ __forceinline__ int classify(const int32_t* row, int j, int E) {
  const int x = row[j];
  if (x < 0) return 0;
  if (x >= E) return -1;
  for (int i = 0; i < j; ++i)
    if (row[i] == x) return -1;
  return 1;
}

// Small batches: one block, thread = token.  Validation as route_hist_kernel; then for expert
// e = 0, 1, ... the tokens routed to e are ranked in token order by a ballot / popcount per warp
// and a prefix over the warps, so token_idx is the same stable CSR as the multi-kernel path.
constexpr int kSmallMaxE = 16;
__global__ void __launch_bounds__(kChunk)
    route_small_kernel(const int32_t* __restrict__ topk, int T, int k, int E, int32_t* __restrict__ counts,
                       int32_t* __restrict__ row_off, int32_t* __restrict__ token_idx, int32_t* __restrict__ slot,
                       int32_t* __restrict__ status, int H, int N, int bm, int bn, uint32_t flags,
                       int32_t* __restrict__ blob) {
  moe::ptx::pdl_launch_dependents();                 // the GEMM prologue may start; it waits for us
  __shared__ int s_wc[kChunk / 32][kSmallMaxE];
  __shared__ int s_cnt[kSmallMaxE], s_base[kSmallMaxE];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int32_t* row = topk + (int64_t)t * k;
  int r[kRegK], v[kRegK];
  int bad = 0;
#pragma unroll
  for (int j = 0; j < kRegK; ++j) r[j] = t < T && j < k ? __ldg(row + j) : -1;
#pragma unroll
  for (int j = 0; j < kRegK; ++j) {
    int x = j < k ? r[j] : -1;
    if (x >= E) {
      bad = 1;
      x = -1;
    }
#pragma unroll
    for (int i = 0; i < j; ++i)
      if (x >= 0 && r[i] == x) {
        bad = 1;
        x = -1;
      }
    v[j] = x;
  }
  // Per warp and expert: how many of the warp's tokens are routed there (one ballot per expert),
  // then one barrier; warp 0 turns the [warps x experts] counts into expert bases.
  const int n_warps = (T + 31) / 32;                 // warps holding tokens (T <= 1024)
  unsigned mk[kRegK];                                // slot j: this warp's ballot for expert v[j]
#pragma unroll
  for (int j = 0; j < kRegK; ++j) mk[j] = 0;
  if (warp < n_warps) {
    for (int e = 0; e < E; ++e) {
      bool hit = false;
#pragma unroll
      for (int j = 0; j < kRegK; ++j) hit |= v[j] == e;
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) s_wc[warp][e] = __popc(m);
#pragma unroll
      for (int j = 0; j < kRegK; ++j)
        if (v[j] == e) mk[j] = m;
    }
  }
  __syncthreads();
  if (warp == 0) {
    int tot = 0;                                     // lane e: tokens of expert e
    if (lane < E)
      for (int w = 0; w < n_warps; ++w) tot += s_wc[w][lane];
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane < E) {
      s_cnt[lane] = tot;
      s_base[lane] = incl - tot;
      counts[lane] = tot;
      row_off[lane] = incl - tot;
    }
    if (lane == E - 1) row_off[E] = incl;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kRegK; ++j) {                  // one write per (token, expert) hit
    if (v[j] < 0) continue;
    int pos = s_base[v[j]] + __popc(mk[j] & ((1u << lane) - 1u));
    for (int w = 0; w < warp; ++w) pos += s_wc[w][v[j]];
    token_idx[pos] = t;
    if (slot) slot[pos] = j;
  }
  bad = __syncthreads_or(bad);
  if (t == 0 && status) *status = bad ? 1 : 0;
  if (blob) moe::dplan::plan_body(t < E ? s_cnt[t] : 0, E, H, N, bm, bn, flags, blob);
}

__global__ void __launch_bounds__(kChunk) route_hist_kernel(const int32_t* __restrict__ topk, int T, int k, int E,
                                                           int32_t* __restrict__ chunk_counts,
                                                           int32_t* __restrict__ chunk_bad) {
  moe::ptx::pdl_launch_dependents();                 // the placement kernel may launch; it waits for us
  __shared__ int hist[kMaxE];
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int t = blockIdx.x * kChunk + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int bad = 0;
  const int32_t* row = topk + (int64_t)t * k;
  if (k <= kRegK) {
    // The token's row in registers (one load latency), validated by register compares.
    int r[kRegK];
#pragma unroll
    for (int j = 0; j < kRegK; ++j) r[j] = t < T && j < k ? __ldg(row + j) : -1;
#pragma unroll
    for (int j = 0; j < kRegK; ++j) {
      if (j >= k) break;                             // k is block-uniform
      int x = r[j];
      if (x >= E) {
        bad = 1;
        x = -1;
      }
#pragma unroll
      for (int i = 0; i < j; ++i)
        if (x >= 0 && r[i] == x) {
          bad = 1;
          x = -1;
        }
      const unsigned grp = __match_any_sync(0xffffffffu, x);
      if (x >= 0 && lane == __ffs(grp) - 1) atomicAdd(&hist[x], __popc(grp));
    }
  } else {
    for (int j = 0; j < k; ++j) {                    // warp-uniform loop: every lane takes part in match_any
      int x = -1;
      if (t < T) {
        const int cl = classify(row, j, E);
        bad |= cl < 0;
        if (cl == 1) x = row[j];
      }
      const unsigned grp = __match_any_sync(0xffffffffu, x);
      if (x >= 0 && lane == __ffs(grp) - 1) atomicAdd(&hist[x], __popc(grp));
    }
  }
  const int any_bad = __syncthreads_or(bad);
  for (int e = threadIdx.x; e < E; e += blockDim.x) chunk_counts[(int64_t)blockIdx.x * E + e] = hist[e];
  if (threadIdx.x == 0) chunk_bad[blockIdx.x] = any_bad ? 1 : 0;
}

// B, fused (chunks x experts <= kPlaceMaxCells): grid = chunks x experts, thread = token of the
// chunk.  Every block re-derives its (chunk, expert) first CSR row from the chunk histograms
// (per-expert totals, one block scan, the earlier chunks of its expert), then compacts the
// chunk's tokens routed to its expert in token order (ballot / popcount ranks).  Block (0, 0)
// writes counts / row_off / status and, with a plan, runs the device planner body.
__global__ void __launch_bounds__(kChunk)
    route_place_kernel(const int32_t* __restrict__ topk, int T, int k, int E, int n_chunks,
                       const int32_t* __restrict__ chunk_counts, const int32_t* __restrict__ chunk_bad,
                       int32_t* __restrict__ counts, int32_t* __restrict__ row_off, int32_t* __restrict__ token_idx,
                       int32_t* __restrict__ slot, int32_t* __restrict__ status, int H, int N, int bm, int bn,
                       uint32_t flags, int32_t* __restrict__ blob) {
  __shared__ long long s_warp[32];
  __shared__ int s_w[kChunk / 32];
  __shared__ int s_base;
  moe::ptx::pdl_wait();                              // the histograms of kernel A are complete
  moe::ptx::pdl_launch_dependents();                 // the GEMM prologue may start; it waits for us
  const int c = blockIdx.x, e = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = threadIdx.x;                         // thread = expert for the scan
  // With a plan the grid has one more column (e == E): block (0, E) only plans, in parallel with the
  // compaction blocks, instead of after block (0, 0)'s compaction (the planner reads counts only).
  const bool planner = e == E;
  if (planner && c != 0) return;
  long long tot = 0, before = 0;
  if (i < E) {
#pragma unroll 8
    for (int cc = 0; cc < n_chunks; ++cc) {
      const int v = __ldg(chunk_counts + (int64_t)cc * E + i);
      tot += v;
      before += cc < c ? v : 0;
    }
  }
  long long all;
  const long long incl = moe::dplan::block_scan_incl(tot, s_warp, &all);
  if (planner) {
    moe::dplan::plan_body(i < E ? tot : 0, E, H, N, bm, bn, flags, blob);
    return;
  }
  if (i == e) s_base = (int)(incl - tot + before);
  const bool lead = c == 0 && e == 0;
  if (lead) {
    if (i < E) {
      counts[i] = (int32_t)tot;
      row_off[i] = (int32_t)(incl - tot);
    }
    int bad = 0;
    for (int cc = threadIdx.x; cc < n_chunks; cc += blockDim.x) bad |= __ldg(chunk_bad + cc);
    bad = __syncthreads_or(bad);
    if (i == 0) {
      row_off[E] = (int32_t)all;
      if (status) *status = bad ? 1 : 0;
    }
  }
  const int t = c * kChunk + threadIdx.x;
  int hit = -1;
  if (t < T) {
    const int32_t* row = topk + (int64_t)t * k;
    for (int j = 0; j < k; ++j)
      if (__ldg(row + j) == e && classify(row, j, E) == 1) hit = j;
  }
  const unsigned m = __ballot_sync(0xffffffffu, hit >= 0);
  if (lane == 0) s_w[warp] = __popc(m);
  __syncthreads();
  if (hit >= 0) {
    int pos = s_base + __popc(m & ((1u << lane) - 1u));
    for (int w = 0; w < warp; ++w) pos += s_w[w];
    token_idx[pos] = t;
    if (slot) slot[pos] = hit;
  }
}

__global__ void __launch_bounds__(moe::dplan::kPlanThreads)
    route_scan_kernel(int32_t* __restrict__ chunk_counts, const int32_t* __restrict__ chunk_bad, int n_chunks, int E,
                      int32_t* __restrict__ counts, int32_t* __restrict__ row_off, int32_t* __restrict__ status,
                      int H, int N, int bm, int bn, uint32_t flags, int32_t* __restrict__ blob) {
  __shared__ long long s_warp[32];
  __shared__ int s_cc[kScanSmem];                    // the chunk x expert histogram, when it fits
  int bad = 0;
  for (int c = threadIdx.x; c < n_chunks; c += blockDim.x) bad |= chunk_bad[c];
  if (__syncthreads_or(bad) && threadIdx.x == 0 && status) *status = 1;
  else if (threadIdx.x == 0 && status) *status = 0;
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
                      int32_t* token_idx, int32_t* slot, int32_t* status, moe_plan* plan, uint32_t route_flags,
                      void* stream) {
  moe::NvtxRange nvtx(plan ? "moe_route_plan" : "moe_route");
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
  if (route_flags & ~(MOE_ROUTE_NO_SMALL | MOE_ROUTE_THREE_KERNELS))
    MOE_FAIL(MOE_ERR_INVALID, "moe_route_ex: unknown flags 0x%x", route_flags);
  const bool small_ok = !(route_flags & MOE_ROUTE_NO_SMALL);
  if (small_ok && T <= kChunk && E <= kSmallMaxE && k <= kRegK) {
    route_small_kernel<<<1, kChunk, 0, s>>>(topk, (int)T, k, E, counts, row_off, token_idx, slot, status, pH, pN,
                                            pbm, pbn, pflags, blob);
    cudaError_t e1 = cudaGetLastError();
    if (e1 != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_route launch: %s", cudaGetErrorString(e1));
    if (plan) moe::plan_set_device_mode(plan, true);
    return MOE_OK;
  }
  const int n_chunks = (int)std::max<int64_t>(1, (T + kChunk - 1) / kChunk);
  int32_t* scratch = nullptr;                        // chunk histograms [n_chunks][E], flags [n_chunks]
  cudaError_t err = cudaMallocAsync((void**)&scratch, sizeof(int32_t) * (size_t)n_chunks * (E + 1), s);
  if (err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_route scratch: %s", cudaGetErrorString(err));
  int32_t* chunk = scratch;
  int32_t* chunk_bad = scratch + (size_t)n_chunks * E;
  route_hist_kernel<<<n_chunks, kChunk, 0, s>>>(topk, (int)T, k, E, chunk, chunk_bad);
  const bool force_split = (route_flags & MOE_ROUTE_THREE_KERNELS) != 0;
  if ((int64_t)n_chunks * E <= kPlaceMaxCells && T > 0 && !force_split) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_chunks, E + (blob ? 1 : 0));   // + the planner column
    cfg.blockDim = dim3(kChunk);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    err = cudaLaunchKernelEx(&cfg, route_place_kernel, topk, (int)T, k, E, n_chunks, (const int32_t*)chunk,
                             (const int32_t*)chunk_bad, counts, row_off, token_idx, slot, status, pH, pN, pbm, pbn,
                             pflags, blob);
    if (err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_route place launch: %s", cudaGetErrorString(err));
  } else {
    route_scan_kernel<<<1, moe::dplan::kPlanThreads, 0, s>>>(chunk, chunk_bad, n_chunks, E, counts, row_off, status,
                                                             pH, pN, pbm, pbn, pflags, blob);
    if (T > 0) route_scatter_kernel<<<dim3(n_chunks, E), kChunk, 0, s>>>(topk, (int)T, k, E, chunk, token_idx, slot);
  }
  cudaFreeAsync(scratch, s);
  err = cudaGetLastError();
  if (err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_route launch: %s", cudaGetErrorString(err));
  if (plan) moe::plan_set_device_mode(plan, true);
  return MOE_OK;
}

}  // namespace

extern "C" moe_status moe_route(const int32_t* topk, int64_t T, int32_t k, int32_t E, int32_t* counts,
                                int32_t* row_off, int32_t* token_idx, int32_t* slot, int32_t* status,
                                void* stream) {
  return route_impl(topk, T, k, E, counts, row_off, token_idx, slot, status, nullptr, 0, stream);
}

extern "C" moe_status moe_route_plan(const int32_t* topk, int64_t T, int32_t k, int32_t E, int32_t* counts,
                                     int32_t* row_off, int32_t* token_idx, int32_t* slot, int32_t* status,
                                     moe_plan* plan, void* stream) {
  if (!plan) MOE_FAIL(MOE_ERR_INVALID, "moe_route_plan: null plan");
  return route_impl(topk, T, k, E, counts, row_off, token_idx, slot, status, plan, 0, stream);
}

extern "C" moe_status moe_route_ex(const int32_t* topk, int64_t T, int32_t k, int32_t E, int32_t* counts,
                                   int32_t* row_off, int32_t* token_idx, int32_t* slot, int32_t* status,
                                   moe_plan* plan, uint32_t route_flags, void* stream) {
  return route_impl(topk, T, k, E, counts, row_off, token_idx, slot, status, plan, route_flags, stream);
}

cudaError_t moe::preload_route_kernels() {
  cudaFuncAttributes fa;
  const void* ks[] = {(const void*)route_small_kernel, (const void*)route_hist_kernel, (const void*)route_place_kernel,
                      (const void*)route_scan_kernel, (const void*)route_scatter_kernel};
  for (const void* k : ks) {
    const cudaError_t e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) return e;
  }
  return moe::preload_plan_kernel();
}
