// Device-side planner body shared by moe_plan_device and moe_route_plan (one block of
// kPlanThreads threads, thread t = expert t).  See plan_device.cu for the passages.
#pragma once
#include <climits>
#include <cstdint>

#include "common.h"

namespace moe {
namespace dplan {

constexpr int kPlanThreads = 1024;

// Inclusive block scan of one int64 per thread (blockDim = 1024); *total = block sum.
__device__ __forceinline__ long long block_scan_incl(long long x, long long* s_warp, long long* total) {
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

// Four inclusive block scans in one pass (the planner's latency is its barriers: one pass = 3 instead of 12).
__device__ __forceinline__ void block_scan_incl4(long long (&x)[4], long long* s_warp4, long long (&total)[4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x[i], o);
      if (lane >= o) x[i] += y;
    }
  }
  if (lane == 31)
#pragma unroll
    for (int i = 0; i < 4; ++i) s_warp4[4 * warp + i] = x[i];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      long long w = s_warp4[4 * lane + i];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_warp4[4 * lane + i] = w;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[i] += warp > 0 ? s_warp4[4 * (warp - 1) + i] : 0;
    total[i] = s_warp4[4 * 31 + i];
  }
  __syncthreads();
}

// All kPlanThreads threads of the block call this; m = tokens of expert threadIdx.x (0 if >= E).
__device__ __forceinline__ void plan_body(long long m, int E, int H, int N, int bm, int bn, uint32_t flags,
                                          int32_t* __restrict__ blob) {
  __shared__ long long s_warp[32];
  __shared__ long long s_warp4[4 * 32];
  const int t = threadIdx.x;                                       // expert t
  // The catalog (header words 12-15, written at plan creation and never rewritten here): kind of
  // each expert's last row tile by its r = m mod bm rows (include/moe_sm100.h).
  int32_t kind = MOE_KIND_WIDE, kind_nogemv = MOE_KIND_WIDE;
  {
    const long long r = m % bm;
    if (m > 0 && r > 0) {
      const bool ride_shape = bm == 256 && bn == 512 && N % bn == 0;   // MOE_KIND_RIDE's tiles (plan.cpp)
      for (int i = MOE_MAX_RULES - 1; i >= 0; --i) {               // the first matching rule wins
        const int32_t ki = blob[12 + 2 * i];
        if (r > blob[13 + 2 * i]) continue;
        if (ki == MOE_KIND_RIDE && (m < bm || !ride_shape)) continue;   // needs a full row tile to ride on
        if (ki != MOE_KIND_GEMV) kind_nogemv = ki;
        if (ki != MOE_KIND_GEMV || m < bm) kind = ki;              // GEMV: whole single-tile tasks only
      }
    }
  }
  __syncthreads();                                                 // every thread read the catalog
  const long long col_tiles = (N + bn - 1) / bn;
  const long long row_tiles = (m + bm - 1) / bm;
  {
    // GEMV only when the other tasks' tiles cover the GEMV streams and the candidates are a real share of the
    // launch (MOE_GEMV_MIN_TILES, MOE_GEMV_MIN_SHARE; plan.cpp)
    long long v4[4] = {m > 0 && kind != MOE_KIND_GEMV ? row_tiles * col_tiles : 0, m > 0 && kind == MOE_KIND_GEMV ? 1 : 0,
                       0, 0};
    long long t4[4];
    block_scan_incl4(v4, s_warp4, t4);
    const long long other_tiles = t4[0], gemv_any = t4[1];
    if (gemv_any > 0 && (other_tiles < MOE_GEMV_MIN_TILES ||
                         gemv_any * col_tiles * 100 < (long long)MOE_GEMV_MIN_SHARE * other_tiles))
      kind = kind_nogemv;
  }
  const long long nu = m > 0 && kind != MOE_KIND_GEMV ? row_tiles * col_tiles : 0;   // nu(T_t); GEMV: no tiles
  // MOE_ORDER_LIGHT_LAST: heavy non-empty tasks first, then the light ones (both in expert order)
  const bool heavy = nu > 0 && m > MOE_LIGHT_ROWS;
  long long sc4[4] = {m, nu, nu > 0 ? 1 : 0, heavy ? 1 : 0}, tot4[4];
  block_scan_incl4(sc4, s_warp4, tot4);                            // rows, tiles, non-empty, heavy
  const long long rows_incl = sc4[0], ne_incl = sc4[2], heavy_incl = sc4[3];
  const long long rows_total = tot4[0], tiles_total = tot4[1], ne_total = tot4[2], heavy_total = tot4[3];
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
      default: w = blob[t];                          // [12, 16): the catalog, kept
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
    if (flags & MOE_ORDER_LIGHT_LAST) {
      // light task: after every heavy one, at its rank among the light ones (ne_incl - heavy_incl of them
      // up to and including t)
      slot = heavy ? (int)(heavy_incl - 1) : (int)(heavy_total + (ne_incl - heavy_incl) - 1);
    } else if (flags & (MOE_ORDER_ALTERNATING | MOE_ORDER_HALF_INTERVAL)) {
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
    p[3] = kind;                                    // the catalog's strategy for the last row tile
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

}  // namespace dplan
}  // namespace moe
