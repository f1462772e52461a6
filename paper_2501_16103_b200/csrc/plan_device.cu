// Device-side planner: device-resident expert token counts -> the compressed mapping,
// written in place into the plan's device blob by ONE single-block kernel launch.
//
// P:142 "this can be either pre-computed on the host and then copied to the device, or
// directly generated on the device"; "the prefix sum can be computed with parallel
// implementation".  Same arithmetic as moe_plan_build (Alg. 1 over the non-empty tasks of
// Alg. 4's extra stage; padding P:203), as block-wide scans: one thread per
// expert.  The blob layout is the header file's, with M_pad fixed at pad32(E) so the
// layout does not depend on the counts (the GEMM can be launched without knowing them).
#include <cuda_runtime.h>

#include <climits>

#include "common.h"

namespace moe {
bool plan_device_mode(const moe_plan* p);
void plan_set_device_mode(moe_plan* p, bool on);
void plan_shape(const moe_plan* p, int32_t* E, int32_t* H, int32_t* N, int32_t* bm, int32_t* bn, uint32_t* flags);
int32_t* plan_blob_dev_mut(moe_plan* p);
}  // namespace moe

namespace {

constexpr int kPlanThreads = 1024;

// Inclusive block scan of one int64 per thread (blockDim = 1024); *total = block sum.
__device__ long long block_scan_incl(long long x, long long* s_warp, long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    long long w = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;                     // inclusive prefix of warp totals
  }
  __syncthreads();
  const long long off = warp > 0 ? s_warp[warp - 1] : 0;
  *total = s_warp[31];
  __syncthreads();                        // s_warp is reused by the next scan
  return x + off;
}

__global__ void __launch_bounds__(kPlanThreads)
    plan_device_kernel(const int32_t* __restrict__ counts, int E, int H, int N, int bm, int bn, uint32_t flags,
                       int32_t* __restrict__ blob) {
  __shared__ long long s_warp[32];
  const int t = threadIdx.x;                                       // expert t
  const bool split = (flags & MOE_SPLIT_TAIL) != 0;
  const long long m = t < E ? (long long)max(counts[t], 0) : 0;
  const long long col_tiles = (N + bn - 1) / bn;
  const long long row_tiles = (m + bm - 1) / bm;
  const long long nu = m > 0 ? row_tiles * col_tiles : 0;         // nu(T_t)
  long long rows_total, tiles_total, ne_total;
  const long long rows_incl = block_scan_incl(m, s_warp, &rows_total);
  block_scan_incl(nu, s_warp, &tiles_total);                       // total tiles
  const long long ne_incl = block_scan_incl(nu > 0 ? 1 : 0, s_warp, &ne_total);
  const int M = (int)ne_total;                                      // |eta|
  const int M_pad = E <= 32 ? 32 : (E + 31) / 32 * 32;
  const bool overflow = rows_total >= INT_MAX || tiles_total >= INT_MAX;
  int32_t* pre = blob + MOE_PLAN_HEADER;
  int32_t* sig = pre + M_pad;
  int32_t* par = sig + M_pad;
  int32_t* roff = par + (long long)MOE_PLAN_TASK_WORDS * E;
  if (t < MOE_PLAN_HEADER) {
    int32_t w = 0;
    switch (t) {
      case 0: w = MOE_PLAN_MAGIC; break;
      case 1: w = overflow ? 0 : M; break;
      case 2: w = overflow ? 0 : (int32_t)tiles_total; break;
      case 3: w = M_pad; break;
      case 4: w = E; break;
      case 5: w = N; break;
      case 6: w = H; break;
      case 7: w = bm; break;
      case 8: w = bn; break;
      case 9: w = E; break;
      case 10: w = (int32_t)flags; break;
      case 11: w = overflow ? 3 : 0; break;          // device planner status (3 = capacity)
      default: w = 0;
    }
    blob[t] = w;
  }
  // sigma: natural order (slot = non-empty index), or a §4.2 ordering over the non-empty tasks
  // (rank by load descending, ties lower id first; then the alternating / bit-reversal slot).
  __shared__ int s_m[kPlanThreads];
  __shared__ long long s_nu[kPlanThreads];
  __shared__ int s_sig[kPlanThreads];
  s_m[t] = nu > 0 ? (int)m : -1;
  __syncthreads();
  if (t < E && nu > 0) {
    int slot = (int)(ne_incl - 1);
    if (flags & (MOE_ORDER_ALTERNATING | MOE_ORDER_HALF_INTERVAL)) {
      int r = 0;                                     // rank in descending load order
      for (int j = 0; j < E; ++j) {
        const int mj = s_m[j];
        r += mj > (int)m || (mj == (int)m && j < t);
      }
      if (flags & MOE_ORDER_ALTERNATING) {
        const int h = (M + 1) / 2;
        slot = r < h ? 2 * r : 2 * (r - h) + 1;
      } else {
        int w = 0;
        while ((1 << w) < M) ++w;
        int seen = 0;
        for (int i = 0; i < (1 << w); ++i) {         // r-th element of the bit-reversal sequence < M
          const int rev = (int)(__brev((unsigned)i) >> (32 - w));
          if (w == 0 || rev < M) {
            if (seen == r) {
              slot = w == 0 ? 0 : rev;
              break;
            }
            ++seen;
          }
        }
      }
    }
    s_nu[slot] = nu;
    s_sig[slot] = t;
  }
  __syncthreads();
  long long scan_total;
  const long long pre_incl = block_scan_incl(t < M ? s_nu[t] : 0, s_warp, &scan_total);   // Alg. 1 in sigma order
  if (t < M) {
    pre[t] = (int32_t)pre_incl;
    sig[t] = s_sig[t];
  }
  if (t < E) {
    int32_t* p = par + (long long)MOE_PLAN_TASK_WORDS * t;
    p[0] = t;
    p[1] = (int32_t)(rows_incl - m);
    p[2] = (int32_t)m;
    p[3] = split && (m % bm) ? 1 : 0;               // kind 1: last row tile is a swap-AB tail
    p[4] = bm;
    p[5] = bn;
    p[6] = (int32_t)row_tiles;
    p[7] = (int32_t)col_tiles;
    roff[t] = (int32_t)(rows_incl - m);
  }
  for (int i = M + t; i < M_pad; i += blockDim.x) {                 // P:203 padding
    pre[i] = (flags & MOE_PAD_REPEAT) && M > 0 ? (int32_t)tiles_total : INT_MAX;
    sig[i] = 0;
  }
  if (t == 0) roff[E] = (int32_t)rows_total;
}

}  // namespace

extern "C" moe_status moe_plan_device(moe_plan* plan, const int32_t* counts_dev, void* stream) {
  moe::clear_error();
  if (!plan || !counts_dev) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_device: null argument");
  int32_t E, H, N, bm, bn;
  uint32_t flags;
  moe::plan_shape(plan, &E, &H, &N, &bm, &bn, &flags);
  if (E > kPlanThreads) MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_plan_device: E=%d > %d", E, kPlanThreads);
  plan_device_kernel<<<1, kPlanThreads, 0, (cudaStream_t)stream>>>(counts_dev, E, H, N, bm, bn, flags,
                                                                   moe::plan_blob_dev_mut(plan));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_plan_device launch: %s", cudaGetErrorString(e));
  moe::plan_set_device_mode(plan, true);
  return MOE_OK;
}
