// Single-launch statically batched MoE expert GEMM for sm_100a (B200).
//
// One persistent, warp-specialised kernel executes every (expert, output-tile)
// task of a plan (arXiv 2501.16103, Alg. 3/4):
//   * every role warp decodes its virtual tile v with the warp vote/popcount
//     mapping over TilePrefix (Alg. 2 + chunk loop) and sigma (Alg. 4
//     line 289) — "let all warps execute the algorithm";
//   * warps 0-3 (A producers) stage, per 64-wide K block, the tile's 128 token
//     rows per CTA straight from X through the token-index array (no
//     gathered copy): cp.async on the LSU path by default, TMA tile::gather4 as an
//     option, one tile TMA when the rows are already in CSR order (token_idx NULL);
//   * warp 4 (B producer) stages the expert's W block with 4-D TMA tile loads;
//     both feed an SW128 shared-memory ring guarded by mbarriers (4-6 stages;
//     P:352-353's two-stage prefetch, deepened);
//   * warp 5 issues tcgen05.mma (bf16 x bf16 -> fp32 in TMEM): 128 x BN tiles on one
//     CTA, 256 x BN on a CTA pair (cta_group::2), and the default 256 x 512 wide pair
//     tile with two N = 256 accumulator blocks, block-staggered (P:351's WGMMA,
//     Blackwell-native);
//   * warps 6-13 drain TMEM with tcgen05.ld (two warps per lane quarter), convert and
//     store Y through TMA tile stores (or masked register stores for a task's last
//     rows), overlapping the next tile's main loop.
// Static batching: CTA (pair) b processes v = b, b + grid, b + 2*grid, ... (no
// dynamic scheduler, no atomics).  Within a task, tiles are ordered row-tile
// fastest (R5), so CTAs of one wave share W column blocks in L2
// (the paper's "tile swizzle").
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.h"
#include "moe_sm100_debug.h"
#include "sm100_ptx.cuh"

namespace moe {
const int32_t* plan_blob_host(const moe_plan* p, int64_t* words);
const int32_t* plan_blob_dev(const moe_plan* p);
bool plan_device_mode(const moe_plan* p);
bool plan_has_swap(const moe_plan* p);
int32_t* plan_sched_dev(const moe_plan* p);
float* plan_sk_ws(const moe_plan* p, int32_t** cnt, int32_t* ctas);
void plan_shape(const moe_plan* p, int32_t* E, int32_t* H, int32_t* N, int32_t* bm, int32_t* bn, uint32_t* flags);
}  // namespace moe

namespace {

using namespace moe::ptx;

constexpr int kBM = 128;                        // tile rows = tcgen05 M
constexpr int kBK = 64;                         // K block: 64 bf16 = one 128-byte swizzle row
constexpr int kABytes = kBM * kBK * 2;          // 16 KB: 128 gathered rows x 64
constexpr int kBBoxBytes = 64 * kBK * 2;        // 8 KB: one TMA box of W (64 N x 64 K)
constexpr int kBStageBytes = 4 * kBBoxBytes;    // up to BN = 256
constexpr int kAWarps = 4;                      // A producers (token rows): warps 0-3
constexpr int kBWarp = kAWarps;                 // B producer (W block, TMA): warp 4
constexpr int kMmaWarp = kAWarps + 1;           // tcgen05 issuer: warp 5
#ifndef MOE_EPI_WARPS
#define MOE_EPI_WARPS 8
#endif
// Epilogue: warps 6.. ; warp w drains TMEM lane quarter w % 4 (the tcgen05.ld lane rule), and the
// kEpiWarps / 4 warps of one quarter take alternate 32-column chunks.
constexpr int kEpiWarps = MOE_EPI_WARPS;
static_assert(kEpiWarps == 4 || kEpiWarps == 8 || kEpiWarps == 16, "1, 2 or 4 warps per TMEM lane quarter");
// TMA-store staging per epilogue warp: two 2 KB buffers (converting chunk i+1 overlaps the store
// of chunk i) with four warps or MOE_EPI_DBUF, else one.
#ifndef MOE_EPI_DBUF
#define MOE_EPI_DBUF 0
#endif
constexpr bool kEpiDbuf = kEpiWarps == 4 || MOE_EPI_DBUF;
constexpr uint32_t kEpiBufBytes = kEpiDbuf ? 4096u : 2048u;
constexpr int kEpiGroups = kEpiWarps / 4;
constexpr int kThreads = 32 * (kAWarps + 2 + kEpiWarps);
constexpr int kDefaultAMode = 1;                // A staging: cp.async (see the A-producer comment)
constexpr uint32_t kTmemCols = 512;             // 2 accumulators x 256 fp32 columns
constexpr uint32_t kAccCols = 256;
constexpr int kMaxMPad = 1024;
#ifndef MOE_TIMELINE
#define MOE_TIMELINE 0      // 1: %globaltimer stamps per CTA at the kernel's phase boundaries (study builds,
#endif                      //    scripts/timeline.py)
#if MOE_TIMELINE
__device__ unsigned long long g_moe_tl[1024 * 8];
#define MOE_TL(i)                                                              \
  do {                                                                         \
    unsigned long long t_;                                                     \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)::"memory");          \
    g_moe_tl[blockIdx.x * 8 + (i)] = t_;                                       \
  } while (0)
#else
#define MOE_TL(i) \
  do {            \
  } while (0)
#endif
#ifndef MOE_L2_PREFETCH
#define MOE_L2_PREFETCH 8
#endif
constexpr int kL2Pf = MOE_L2_PREFETCH;          // memory-bound tiles: W K blocks prefetched into L2 ahead
constexpr int kBarBytes = 512;                  // 8 B per mbarrier (<= 2*6+4) + TMEM address slot + tile queue
                                                // [0,256); kProf stage timestamps [256,512)
constexpr int kQ = 4;                           // dynamic tile order: tile-queue slots per CTA

struct GemmArgs {
  const int32_t* plan;       // device plan blob
  const int32_t* token_idx;  // CSR token-index array
  void* Y;
  int32_t y_f32;
  int32_t N;
  int32_t num_kb;
  int32_t total;             // < 0: device-planned, read the tile count from the blob header
  int32_t M_pad;
  int32_t off_params;
  int32_t T;
  int32_t w4d;               // W map is 4-D {64, H, N/64, E}: one TMA per B stage
  long long* prof;           // kProf builds only: per-CTA cycle counters (moe_gemm_profile)
  int32_t a_mode;            // A staging: 0 = TMA tile::gather4, 1 = cp.async (LSU path), 2 = contiguous
                             // rows (token_idx NULL: X row = CSR row) by one tile TMA per stage; DESIGN.md
  int32_t H;
  const __nv_bfloat16* X;
  int32_t experiment;        // MOE_EXPERIMENTS builds only (timing studies, wrong Y), bit mask: 1 = no A reads,
                             // 2 = no B loads, 4 = A as contiguous tile TMA (pairs), 8 = no Y stores
  const int32_t* y_row_map;  // nullable: Y row of CSR row i is y_row_map[i] (EP combine buffer)
  int32_t tma_store;         // bf16 Y in CSR row order: full 32-row quarters leave through TMA tile stores
  const float* scale;        // FP8 path, nullable: Y rows of expert e are scaled by scale[e] (fp32, epilogue)
  const unsigned long long* y_row_ptr;   // nullable: CSR row i is stored at address y_row_ptr[i] (any device
                                         // memory the SM can write: the EP combine buffers of peer ranks)
  int32_t balance;           // balanced grid: only ceil(total / ceil(total / grid)) CTAs (pairs) take tiles
  int32_t* sched;            // nullable: dynamic tile order — [0] next virtual tile (- n_pairs), [1] pairs done
  const uint8_t* W;          // W base (bytes), for the load/store-path L2 prefetch of memory-bound tiles
  int32_t pf_dist;           // that prefetch's distance in K blocks (0: off); one-CTA tiles: every tile,
                             // CTA pairs: swap-AB tiles only
  float* sk_ws;              // nullable: stream-K partial accumulators (one-CTA tiles)
  int32_t* sk_cnt;           //           and per-tile arrival counters (zero between launches)
  int32_t light_merge;       // MOE_ORDER_LIGHT_LAST plan under the dynamic tile order: interleave the light
                             // (memory-bound) tail of the virtual tiles among the others in proportion
  int32_t narrow_last;      // > 1: column tiles per task, the last (narrower) column block of every task is fetched
                             // after the full-width ones (dynamic order of wide tiles)
  int32_t half_last;        // MOE_SCHED_HALF_LAST: dynamic order of wide tiles with each task's <= 128-row last
                             // row tile (a half tile) after every full tile (LPT-like end)
  int32_t* gemv_q;           // nullable: the plan may hold MOE_KIND_GEMV tasks (wide pair kernels): [0] next
                             // GEMV unit, [1] epilogue warps done (both zero between launches)
};

// Per-CTA counters written by the instrumented build (kProf = true).
enum ProfSlot {
  kProfMmaWaitTmem = 0,   // MMA warp: cycles waiting for the epilogue to free an accumulator
  kProfMmaWaitFull,       // MMA warp: cycles waiting for TMA bytes
  kProfMmaTotal,          // MMA warp: cycles in its tile loop
  kProfProdWaitEmpty,     // producer warp 0: cycles waiting for a free stage
  kProfEpiWaitFull,       // epilogue warp (quarter 0): cycles waiting for an accumulator
  kProfEpiWork,           // epilogue warp (quarter 0): cycles draining + storing
  kProfTiles,             // tiles processed by the CTA
  kProfProdTotal,         // producer warp 0: cycles in its tile loop
  kProfMmaIssue,          // MMA warp: cycles from `full` observed to the stage's commit issued
  kProfMmaTileGap,        // MMA warp: cycles between tiles (decode + accumulator hand-off)
  kProfBWaitEmpty,        // B warp: cycles waiting for a free stage
  kProfBTotal,            // B warp: cycles in its tile loop
  kProfLatB,              // sum over stages: MMA sees `full` - B warp issued the W TMA (this CTA)
  kProfLatA,              // sum over stages: MMA sees `full` - A warp 0 issued its row copies
  kProfRelease,           // sum over stages: B warp re-issues into a slot - MMA committed that slot
  kProfStages,            // stages counted
  kProfSlots
};

// ---------------------------------------------------------------------------
// Alg. 2 with the chunk loop and Alg. 4's sigma.
// Executed by a full warp; v must be warp-uniform and < total.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void map_tile(const int32_t* prefix, const int32_t* sigma, int M_pad, int v,
                                         int& h, int& task, int& l) {
  const int lane = threadIdx.x & 31;
  int hh = 0;
  for (int c = 0; c < M_pad; c += 32) {
    const bool p = v >= prefix[c + lane];                  // p <- B >= TilePrefix[t]
    const unsigned mask = __ballot_sync(0xffffffffu, p);   // warp vote
    const int cnt = __popc(mask);                          // population count
    hh += cnt;
    if (cnt < 32) break;
  }
  const int base = hh > 0 ? prefix[hh - 1] : 0;            // k <- TilePrefix[h-1] (or 0)
  h = hh;
  l = v - base;                                            // l <- B - k
  task = sigma[hh];                                        // h~ <- sigma(h)
}

// Split-K of one-CTA memory-bound tiles: each tile's K blocks in S equal parts; unit
// u = p * total + v is part p of virtual tile v (part-major), and CTA c of G takes units c, c + G, c + 2G,
// ... < U = total * S (static stride: the CTAs working at the same time stream neighbouring W column
// strips over the same K rows, as whole tiles do).  The CTA finishing the last part of tile v sums the S
// partials in part (K) order (deterministic) and stores Y.
__device__ __forceinline__ int sk_parts(int total, int grid, int num_kb) {
  // the smallest S >= 2 whose units fill the CTAs to >= 90 % (else the fullest), S <= num_kb and
  // total * S <= kSKUnitsPerCta * grid; 0 when no S beats whole tiles on the balanced grid
  const int per = (total + grid - 1) / grid, used = (total + per - 1) / per;
  float best = (float)used / grid;
  int best_s = 0;
  for (int S = 2; S <= num_kb && (long long)total * S <= (long long)moe::kSKUnitsPerCta * grid; ++S) {
    const long long U = (long long)total * S;
    const float e = (float)U / (float)(grid * ((U + grid - 1) / grid));
    if (e > best + 0.02f) {
      best = e;
      best_s = S;
      if (e >= 0.9f) break;
    }
  }
  return best_s;
}

struct Tile {
  int expert, row0, rows, bn, rt, ct;
  int kind;     // of THIS tile: 0 = bm rows x bn cols (MOE_KIND_WIDE); 1 = swap-AB tile (MOE_KIND_SWAP);
                // 3 = ride tile (MOE_KIND_RIDE): body row tile rt, 256-column half hh, plus the tail rows
  int height;   // kind 1 / 3: tail rows rounded up to 16 (the swap MMA's N)
  int hh, trow0, trows;   // kind 3: the half, the tail's first CSR row and its row count
};

template <bool kSplit = false>
__device__ __forceinline__ Tile load_tile(const int32_t* params, int task, int l, bool ride_ok = false) {
  const int4 pa = __ldg(reinterpret_cast<const int4*>(params + task * MOE_PLAN_TASK_WORDS));
  const int4 pb = __ldg(reinterpret_cast<const int4*>(params + task * MOE_PLAN_TASK_WORDS + 4));
  Tile t;
  t.expert = pa.x;
  t.row0 = pa.y;
  t.rows = pa.z;
  t.bn = pb.y;
  t.rt = l % pb.z;   // row tile fastest (R5)
  t.ct = l / pb.z;
  t.kind = 0;
  t.height = pb.x;
  t.hh = t.trow0 = t.trows = 0;
  if constexpr (kSplit) {
    // The catalog: a kind-1 task runs its last row tile (rows [rt*bm, rows)) swap-AB.
    if (pa.w == 1 && t.rt == pb.z - 1) {
      const int tail = t.rows - t.rt * pb.x;
      t.kind = 1;
      t.height = (tail + 15) / 16 * 16;
      t.row0 += t.rt * pb.x;                       // kind 1: row0 / rows are the tail's
      t.rows = tail;
    } else if (pa.w == MOE_KIND_RIDE && ride_ok && t.rt >= pb.z - 2) {
      // The catalog's ride strategy: slots R-2 / R-1 are the two 256-column halves of row
      // tile R-2; each also computes the r = rows - 256 (R-1) tail rows x its columns (swap-AB MMA).
      t.kind = 3;
      t.hh = t.rt - (pb.z - 2);
      t.rt = pb.z - 2;
      t.trow0 = t.row0 + (pb.z - 1) * pb.x;
      t.trows = t.rows - (pb.z - 1) * pb.x;
      t.height = (t.trows + 15) / 16 * 16;
    }
  }
  return t;
}

// Wide tiles: the columns MMA block hf of column tile ct actually computes — all bn/2 of them,
// except in a column tile passing N, where they are trimmed to the block's columns below N
// rounded up to 128 (each CTA's half then stays on the 64-column W chunk grid); 0 = no MMA.
// (FP8: W chunks are 128 columns, so blocks are trimmed to multiples of 256.)
template <bool kFp8 = false>
__device__ __forceinline__ int wide_block_cols(int bn, int ct, int N, int hf) {
  constexpr int kGran = kFp8 ? 256 : 128;
  const int bnp = bn / 2;
  const int nvalid = min(bn, N - ct * bn) - hf * bnp;
  return nvalid <= 0 ? 0 : min(bnp, (nvalid + kGran - 1) & ~(kGran - 1));
}

// Wide 512-column tiles that lie inside N (and every swap-AB tile) stage W as ONE 4-D TMA box of
// 256 columns per CTA per stage instead of one 128-column box per MMA block: TMA issues a box every
// ~330 ns per SM whatever its size up to 32 KB (scripts/stream_probe.cu), so bigger
// boxes stream W faster.  CTA r then holds tile columns [256 r, 256 r + 256): MMA block hf takes its
// half [256 r + 128 hf, +128), so D column n of block hf is W column 256 (n >= 128) + 128 hf + n % 128
// (two boxes: 256 hf + n; for swap-AB tiles the D row plays n's role).
template <bool kWide, bool kGated>
__device__ __forceinline__ bool one_box(int bn, int ct, int N, int w4d, bool swap) {
  return kWide && !kGated && w4d && bn == 512 && (swap || (ct + 1) * bn <= N);
}
__device__ __forceinline__ int w_col(bool one, int ct, int bn, int hf, int half, int j) {
  // column of W for block hf, D half `half` (= the CTA whose shared memory holds it), offset j < 128
  return ct * bn + (one ? 256 * half + 128 * hf : 256 * hf + 128 * half) + j;
}

// Wide kind-0 tiles whose valid rows fit in 128 ("half" tiles: an expert's short last row tile)
// run M = 128 pair MMAs — 64 rows per CTA, half the tensor time; the D layout then folds each
// block's columns: [0, N/2) in TMEM lanes 0-63, [N/2, N) in lanes 64-127 (CUTLASS's UMMA_2SM
// "2x2" data path for M = 128), each over TMEM columns [0, N/2).
template <bool kWide, bool kGated>
__device__ __forceinline__ bool half_tile(int rows, int rt, bool swap) {
  return kWide && !kGated && !swap && rows - rt * 256 <= 128;
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) {
  __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<uint32_t*>(&b);
}

// Store 32 consecutive fp32 accumulator columns [col0, col0+32) of one Y row,
// masked to col < col_end (col_end is a multiple of 8).
__device__ __forceinline__ void store_chunk(const GemmArgs& a, uint8_t* yrow_ptr, int col0, int col_end,
                                            const uint32_t (&v)[32]) {
  if (a.y_f32) {
    float* y = reinterpret_cast<float*>(yrow_ptr);
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const int c = col0 + 4 * g;
      if (c + 4 <= col_end) {
        uint4 q = make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
        *reinterpret_cast<uint4*>(y + c) = q;
      }
    }
  } else {
    __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(yrow_ptr);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const int c = col0 + 8 * g;
      if (c + 8 <= col_end) {
        uint4 q = make_uint4(pack_bf16(v[8 * g], v[8 * g + 1]), pack_bf16(v[8 * g + 2], v[8 * g + 3]),
                             pack_bf16(v[8 * g + 4], v[8 * g + 5]), pack_bf16(v[8 * g + 6], v[8 * g + 7]));
        *reinterpret_cast<uint4*>(y + c) = q;
      }
    }
  }
}

template <bool kProf>
__device__ __forceinline__ void wait_timed(uint32_t bar, uint32_t parity, long long& acc) {
  if constexpr (kProf) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    acc += clock64() - t0;
  } else {
    mbar_wait(bar, parity);
  }
}

// ---------------------------------------------------------------------------
// MOE_KIND_GEMV tasks: Alg. 3's per-task strategy for tasks of <= MOE_GEMV_MAX_ROWS
// rows.  They have no tiles; the epilogue warps of every CTA take GEMV units from a global queue and
// work on them whenever they would otherwise wait for an accumulator, so the tasks' W streams while the
// tensor cores compute the other tasks' tiles.  A unit = one task x 128 output columns x all of K, owned
// by one warp: lanes 0-15 take K rows k..k+7, lanes 16-31 rows k+8..k+15 of each 16-row round, lane l
// columns 8 (l mod 16) + [0, 8); fp32 accumulation in registers, the two half-warps summed at the end.
// A round loads 16 W rows per batch (4 KB per warp in flight) and accumulates them; an L2 prefetch of rows
// further ahead measured slower (paper worst 0.811 / 0.724 of peak at 6 / 16 rounds ahead vs 0.830 without).
// ---------------------------------------------------------------------------
constexpr int kGemvCols = 128;
#ifndef MOE_GEMV_LOAD
#define MOE_GEMV_LOAD 1   // W loads of GEMV units: 1 = ld.global.nc.L1::no_allocate (paper worst +2.4 %), 0 = ld.global.cs
#endif
#ifndef MOE_GEMV_BATCH
#define MOE_GEMV_BATCH 1
#endif
constexpr int kGemvBatch = MOE_GEMV_BATCH;   // 16-row batches per round

template <bool kFp8>
struct GemvUnit {
  int task = -1, rows = 0, row0 = 0, expert = 0, col0 = 0, kpos = 0;
  float acc[MOE_GEMV_MAX_ROWS][8];

  // 8 values (bf16: a uint4; E4M3: a uint2) -> fp32
  __device__ __forceinline__ static void widen(const uint4& q, float (&f)[8]) {
    if constexpr (kFp8) {
      const uint32_t w[2] = {q.x, q.y};
#pragma unroll
      for (int i = 0; i < 2; ++i) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint32_t h2;
          const uint16_t pair = (uint16_t)(w[i] >> (16 * j));
          asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(pair));
          const __half2 hh = *reinterpret_cast<const __half2*>(&h2);
          const float2 ff = __half22float2(hh);
          f[4 * i + 2 * j] = ff.x;
          f[4 * i + 2 * j + 1] = ff.y;
        }
      }
    } else {
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
      }
    }
  }
  __device__ __forceinline__ static uint4 load8(const uint8_t* p) {
#if MOE_GEMV_LOAD == 1
    // read-only path, no L1 allocation (the W stream is used once)
    if constexpr (kFp8) {
      uint32_t x, y;
      asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "l"(p));
      return make_uint4(x, y, 0u, 0u);
    } else {
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(p));
      return v;
    }
#else
    if constexpr (kFp8) {
      const uint2 v = __ldcs(reinterpret_cast<const uint2*>(p));
      return make_uint4(v.x, v.y, 0u, 0u);
    } else {
      return __ldcs(reinterpret_cast<const uint4*>(p));
    }
#endif
  }
};

// Pipeline geometry per CTA-group size: a CTA pair (cta_group::2) splits the B block across the
// two CTAs, so a stage is 32 KB instead of 48 KB and six stages fit.  A wide pair tile (256 x 512,
// kWide) stages 128 rows + 256 W columns per CTA: 48 KB, four stages.
template <int kCta, bool kSplit = false, bool kWide = false>
struct Geo {
#ifndef MOE_WIDE_STAGES
#define MOE_WIDE_STAGES 4
#endif
#ifndef MOE_CTA1_STAGES
#define MOE_CTA1_STAGES 4
#endif
  static constexpr int kStages = kWide ? MOE_WIDE_STAGES : kCta == 2 ? 6 : MOE_CTA1_STAGES;   // 7th pair stage: no gain
  static_assert(8 * (2 * kStages + 4 + 2 * kQ) + 4 * kQ + 8 <= 256, "barrier block overlaps the kProf stamps");
  static constexpr int kBStage = (kWide ? 2 : 1) * kBStageBytes / kCta;   // bytes of W per CTA per stage
  // 16 KB: a 2 KB bf16 staging buffer per epilogue warp for the TMA-store epilogue (two per warp
  // with four warps).
  static constexpr int kEpiStage = 16384 > kEpiWarps * kEpiBufBytes ? 16384 : kEpiWarps * kEpiBufBytes;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * (kABytes + kBStage) + kEpiStage + kBarBytes;
};

// kSplit: the plan's catalog has a swap-AB rule (kind-1 tiles may exist); a separate instantiation so
// the plain path carries none of the swap-AB code.
// kWide: wide pair tiles (bm = 256, bn = 512).  Each K block feeds two N = 256 MMAs into the two
// TMEM accumulators (columns 0-255 and 256-511): every staged token row serves 512 output columns,
// so per FLOP the tile stages 3/4 of the bytes of a 256 x 256 tile (fewer L2 -> SM bytes, fewer
// shared-memory fills, half the barrier round trips).  The accumulator is not double-buffered: the
// MMA waits for the epilogue to drain half 0 before the next tile's first MMAs, half 1 before the
// next tile's first half-1 MMAs.
// kGated (with kWide; moe_gemm_swiglu): a tile covers bn = 256 output columns
// n0 + [0, 256).  MMA block b (N = 256) multiplies [W_gate cols n0 + 128b + [0,128) | W_up cols
// n0 + 128b + [0,128)] — the pair leader stages the gate half, the peer the up half — so TMEM
// block b holds gate in columns [0,128) and up in [128,256) of the same 128 outputs, and the
// epilogue writes silu(gate) * up (R14) block by block, freeing each as the plain wide
// tile does.
// kFp8 (moe_gemm_fp8): X and W in FP8 E4M3, tcgen05.mma kind::f8f6f4, fp32 accumulate, optional
// per-expert fp32 scale in the epilogue.  Stages keep their byte sizes: a K block is 128 FP8 values.
template <bool kProf, int kCta, bool kSplit, bool kWide = false, bool kGated = false, bool kFp8 = false>
__global__ void __launch_bounds__(kThreads, 1)
    moe_gemm_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                    const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmY,
                    const GemmArgs a) {
  static_assert(!kSplit || kCta == 2, "swap-AB tail tiles need CTA pairs (M = 256)");
  static_assert(!kWide || kCta == 2, "wide tiles are CTA-pair tiles");
  static_assert(!(kSplit && kGated), "swap-AB tail tiles are not gated");
  static_assert(!kGated || kWide, "gated tiles use the wide tile's two accumulator blocks");
  constexpr int kSt = Geo<kCta, kSplit, kWide>::kStages;
  constexpr int kBSt = Geo<kCta, kSplit, kWide>::kBStage;
  constexpr int kHalves = kWide ? 2 : 1;                   // N = 256 MMA blocks per tile
  // Element type: a stage holds 128-byte K rows either way, so a K block is 64 bf16 or 128 FP8
  // values; a W box is 64 (bf16) or 128 (FP8) columns x one K block (8 / 16 KB); one MMA consumes
  // 32 bytes of K (K = 16 bf16 / 32 FP8), i.e. 16 / 32 rows of the MN-major W box (+2 / +4 KB).
  constexpr int kKB = kFp8 ? 128 : kBK;
  constexpr int kCS = kFp8 ? 7 : 6;                        // log2(W columns per box)
  constexpr int kBox = kFp8 ? 128 * 128 : kBBoxBytes;
  constexpr int kKStep = kFp8 ? 4096 : 2048;
  static_assert(!kFp8 || (!kSplit && !kGated), "FP8: plain and wide tiles");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;            // SW128 atoms need 1024-byte alignment
  uint8_t* smem = smem_raw + (base - raw);
  const uint32_t sA = base;
  const uint32_t sB = sA + kSt * kABytes;
  const uint32_t sEpi = sB + kSt * kBSt;                   // TMA-store staging buffers
  const uint32_t sBar = sEpi + Geo<kCta, kSplit, kWide>::kEpiStage;
  auto full_bar = [&](int s) { return sBar + 8u * s; };
  auto empty_bar = [&](int s) { return sBar + 8u * (kSt + s); };
  auto tfull_bar = [&](int i) { return sBar + 8u * (2 * kSt + i); };
  auto tempty_bar = [&](int i) { return sBar + 8u * (2 * kSt + 2 + i); };
  // Dynamic tile order: queue slot i holds the CTA pair's i-th virtual tile; qfull[i] completes when the
  // leader's B warp has published it (in both CTAs), qempty[i] when every consumer warp has read it.
  auto qfull_bar = [&](int i) { return sBar + 8u * (2 * kSt + 4 + i); };
  auto qempty_bar = [&](int i) { return sBar + 8u * (2 * kSt + 4 + kQ + i); };
  const uint32_t s_q = sBar + 8u * (2 * kSt + 4 + 2 * kQ);          // kQ int32 tile ids
  volatile int32_t* q_slot = reinterpret_cast<volatile int32_t*>(smem + (s_q - base));
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + (s_q - base) + 4 * kQ);
  int32_t* s_prefix = reinterpret_cast<int32_t*>(smem + (sBar - base) + kBarBytes);
  long long* s_ts = reinterpret_cast<long long*>(smem + (sBar - base) + 256);   // kProf: [3][kSt] stamps
  int32_t* s_sigma = s_prefix + a.M_pad;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) MOE_TL(0);                   // kernel entry
  // Everything up to the TMEM allocation overlaps the previous kernel (PDL); the plan, the
  // token-index array and X are only touched after griddepcontrol.wait.
  int total = a.total;
  // CTA pair: rank 0 (leader) issues the MMAs for both CTAs; all consumers of the
  // data path (full / tmem-empty barriers) live in the leader.
  const uint32_t rank = kCta == 2 ? cluster_ctarank() : 0;
  const int pair_id = blockIdx.x / kCta;
  int n_pairs = gridDim.x / kCta;
  auto leader = [&](uint32_t addr) { return kCta == 2 ? mapa_shared(addr, 0) : addr; };

  const int a_mode = a.a_mode == 2 ? 2 : kCta == 2 && !kWide ? 1 : a.a_mode;
  // MOE_KIND_RIDE tiles need the gathered (cp.async) token rows: with contiguous-row A (a_mode 2) the plan's
  // ride slots run as the plain wide tiles they partition (same rows, same columns).
  const bool ride_ok = kSplit && kWide && !kGated && a_mode == 1;
  if (threadIdx.x == 0) {
    // full[s] arrivals: A stage done (gather4: one expect_tx per A warp; cp.async: one asynchronous
    // arrive per A thread; contiguous rows: the 1-CTA A thread's expect_tx, while in a pair the
    // A tile TMAs of both CTAs complete on the leader's barrier under the B warp's expect_tx), the
    // B warp's expect_tx (leader), and in a pair the peer's relay (leader; not in a_mode 2).
    // (a CTA pair's gather4 rows complete on the leader's barrier under the B warp's expect_tx, like a_mode 2)
    const uint32_t a_arrivals = a_mode == 2 ? (kCta == 1 ? 1u : 0u) : a_mode == 0 ? (kCta == 1 ? kAWarps : 0u)
                                                                                  : 32 * kAWarps;
    const uint32_t relay = kCta == 2 && a_mode == 1 ? 1u : 0u;
    const uint32_t full_count = a_arrivals + (rank == 0 ? 1u + relay : 0u);
    for (int s = 0; s < kSt; ++s) {
      mbar_init(full_bar(s), full_count > 0 ? full_count : 1u);   // a pair peer's are unused in a_mode 2
      mbar_init(empty_bar(s), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull_bar(i), 1);
      mbar_init(tempty_bar(i), kCta * kEpiWarps);
    }
    // queue consumers (one arrival per warp, on the leader's qempty): A warps, MMA warp (leader) or
    // relay lane (peer, unless rows are contiguous), the peer's B warp, epilogue warps
    const uint32_t q_consumers = kCta == 2 ? 2 * (kAWarps + kEpiWarps) + 2 + (a_mode == 1 ? 1u : 0u)
                                           : kAWarps + 1 + kEpiWarps;
    for (int i = 0; i < kQ; ++i) {
      mbar_init(qfull_bar(i), 1);
      mbar_init(qempty_bar(i), q_consumers);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW);
    if (kGated || kWide) prefetch_tmap(&tmW2);
    if (a.tma_store) prefetch_tmap(&tmY);
  }
  if (warp == kMmaWarp) tmem_alloc<kTmemCols, kCta>(smem_u32(tmem_holder));
  pdl_wait();                                        // routing / plan of this step are complete
  if (threadIdx.x == 0) MOE_TL(1);                   // after the PDL wait
  // TilePrefix and sigma are adjacent in the blob: one copy into shared memory.
  for (int i = threadIdx.x; i < 2 * a.M_pad; i += blockDim.x) s_prefix[i] = a.plan[MOE_PLAN_HEADER + i];
  if (total < 0) total = __ldg(a.plan + 2);
  // Stream-K for one-CTA tiles when whole tiles would leave SMs idle (the balanced grid uses fewer CTAs
  // than launched) and every task is short enough for the partial-accumulator slots (decode batches).
  bool sk = false;
  int sk_s = 0;                                     // parts per tile
  if constexpr (kCta == 1 && !kWide && !kSplit && !kGated) {
    __shared__ int s_sk_rows;
    if (a.sk_ws != nullptr && total > 0 && total <= moe::kSKMaxTiles) {
      sk_s = sk_parts(total, (int)gridDim.x, a.num_kb);
      if (sk_s > 0) {
        if (threadIdx.x == 0) s_sk_rows = 0;
        __syncthreads();
        const int n_tasks = __ldg(a.plan + 9);
        int mx = 0;
        for (int i = threadIdx.x; i < n_tasks; i += blockDim.x)
          mx = max(mx, __ldg(a.plan + a.off_params + i * MOE_PLAN_TASK_WORDS + 2));
        atomicMax(&s_sk_rows, mx);
        __syncthreads();
        sk = s_sk_rows <= moe::kSKRows;
      }
    }
  }
  if (!sk && a.balance && total > 0) {
    // Balanced grid: with W = ceil(total / grid) tiles for the busiest CTA (pair) anyway, spread the
    // tiles over ceil(total / W) CTAs so every active one takes W or W - 1 and no short last wave
    // runs on a few SMs — for HBM-bound (decode) tiles the kernel's streaming rate then stays the
    // chip's instead of dropping to a few SMs' for the tail.
    const int per = (total + n_pairs - 1) / n_pairs;
    const int used = (total + per - 1) / per;
    if (pair_id >= used) total = 0;                  // this CTA (pair) takes no tile
    n_pairs = used;
  }
  tc_fence_before();
  if constexpr (kCta == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (threadIdx.x == 0) MOE_TL(2);                   // prologue done (plan in shared memory, TMEM allocated)
  const int32_t* params = a.plan + a.off_params;
  constexpr int kPairRows = kBM * kCta;                     // rows of a virtual tile

  // The virtual tiles of this CTA (pair), in the order every role warp walks them.  Static: v = pair_id
  // + i * n_pairs (P:75-77's static batching).  Dynamic (a.sched): tile 0 is pair_id, then the leader's B
  // warp takes the next v from a global counter as the pair frees up — the order in which the hardware
  // dispatches the paper's one-block-per-tile launch — and publishes it through the tile queue.
  const bool dyn = a.sched != nullptr;
  auto tile_of = [&](uint32_t i) -> int {                   // consumer warps (all lanes)
    if (!dyn) return pair_id + (int)i * n_pairs;
    const int sl = (int)(i % kQ);
    mbar_wait_acq_cluster(qfull_bar(sl), (i / kQ) & 1u);
    const int v = q_slot[sl];
    __syncwarp();
    if (lane == 0) {
      if constexpr (kCta == 2) mbar_arrive_cluster(leader(qempty_bar(sl)));
      else mbar_arrive(qempty_bar(sl));
    }
    return v;
  };
  auto tile_of_lane = [&](uint32_t i) -> int {              // a single-lane consumer (the pair relay)
    if (!dyn) return pair_id + (int)i * n_pairs;
    const int sl = (int)(i % kQ);
    mbar_wait_acq_cluster(qfull_bar(sl), (i / kQ) & 1u);
    const int v = q_slot[sl];
    mbar_arrive_cluster(leader(qempty_bar(sl)));
    return v;
  };
  // The i-th unit of work of this CTA (pair): a virtual tile v and its K blocks [k0, k1) — the whole tile,
  // or under stream-K the tile's part inside this CTA's share of the K-block sequence.  Every role warp
  // walks the same units (its own cursor).
  const long long sk_units = sk ? (long long)total * sk_s : 0;
  long long sk_pos = blockIdx.x;                    // split-K: the next unit u (static stride over units)
  auto next_unit = [&](uint32_t i, int& v, int& k0, int& k1) -> bool {
    if (sk) {
      if (sk_pos >= sk_units) return false;
      const int p = (int)(sk_pos / total);
      v = (int)(sk_pos - (long long)p * total);
      k0 = p * a.num_kb / sk_s;
      k1 = (p + 1) * a.num_kb / sk_s;
      sk_pos += gridDim.x;
      return true;
    }
    v = tile_of(i);
    k0 = 0;
    k1 = a.num_kb;
    return v < total;
  };

  if (warp < kAWarps) {
    // ===================== A producers: this CTA's 128 token rows, 64 columns per stage =====================
    // Gathered straight from X through the token-index array: no gathered copy of X.
    // a_mode 0 (1-CTA only): TMA tile::gather4 — warp p stages rows [32p, 32p+32), 4 rows per lane.
    // a_mode 1: cp.async 16 B per thread, 8 threads per 128-byte row (coalesced), SW128 swizzle
    //           applied by hand; rows past the task's end (and columns past H) are zero-filled
    //           without a read.  Completion: cp.async.mbarrier.arrive — the hardware arrives on
    //           this CTA's full barrier when the thread's copies land; the thread never blocks.
    //           In a CTA pair the peer's MMA warp relays its completed stages to the leader.
    const uint64_t pol_x = policy_evict_last();    // X_e is re-read by every column tile of the task
    const int p = warp;
    uint32_t g = 0;                                 // stages issued by this warp, over all tiles
    long long c_wait = 0, c_t0 = kProf ? clock64() : 0;
    const int ch = threadIdx.x & 7;                 // cp.async: 16-byte chunk of the 128-byte row
    const int rsub = threadIdx.x >> 3;              // cp.async: row within a 16-row group
    const uint32_t dst_off = rsub * 128 + ((ch ^ (rsub & 7)) << 4);
    for (uint32_t qi = 0;; ++qi) {
      int v, k0, k1;
      if (!next_unit(qi, v, k0, k1)) break;
      int h, task, l;
      map_tile(s_prefix, s_sigma, a.M_pad, v, h, task, l);
      const Tile t = load_tile<kSplit>(params, task, l, ride_ok);
      // kind 0: this CTA's 128 rows of the tile; kind 1 (swap-AB tail): this CTA's half of the
      // tail's `height` token rows, which the MMA reads as its N operand.
      const bool hlf = half_tile<kWide, kGated>(t.rows, t.rt, kSplit && t.kind == 1);
      const int n_alloc = kSplit && t.kind == 1 ? t.height / kCta : hlf ? kBM / 2 : kBM;
      const int rbeg = kSplit && t.kind == 1 ? (int)rank * n_alloc : t.rt * kPairRows + (int)rank * n_alloc;
      const int nvalid = min(n_alloc, t.rows - rbeg);   // may be <= 0 for the second CTA of a pair tile
      const int32_t* idx = a.token_idx + t.row0;
      if (a_mode == 2) {
        // Contiguous rows (X row = CSR row): one 128-row tile TMA per stage, issued by one thread.
        // Rows past the task's end are the next task's (never stored); past X they are zero-filled.
        if (p == 0 && lane == 0) {
          for (int kb = k0; kb < k1; ++kb, ++g) {
            const int s = g % kSt;
            wait_timed<kProf>(empty_bar(s), ((g / kSt) & 1u) ^ 1u, c_wait);
            if constexpr (kCta == 2) {
              tma_load_2d_pair(&tmX, leader(full_bar(s)), sA + s * kABytes, kb * kKB, t.row0 + rbeg, pol_x);
            } else {
              mbar_arrive_expect_tx(full_bar(s), kABytes);
              tma_load_2d(&tmX, full_bar(s), sA + s * kABytes, kb * kKB, t.row0 + rbeg, pol_x);
            }
          }
        }
        __syncwarp();
      } else if (a_mode == 0) {
        // Rows past the task's end repeat its last valid token (their results are never stored).
        const int rr = 32 * p + 4 * (lane & 7);
        const int r0 = __ldg(idx + rbeg + min(rr + 0, nvalid - 1));
        const int r1 = __ldg(idx + rbeg + min(rr + 1, nvalid - 1));
        const int r2 = __ldg(idx + rbeg + min(rr + 2, nvalid - 1));
        const int r3 = __ldg(idx + rbeg + min(rr + 3, nvalid - 1));
        for (int kb = k0; kb < k1; ++kb, ++g) {
          const int s = g % kSt;
          wait_timed<kProf>(empty_bar(s), ((g / kSt) & 1u) ^ 1u, c_wait);
          if constexpr (kCta == 2) {
            if (lane < 8)
              tma_gather4_pair(&tmX, leader(full_bar(s)), sA + s * kABytes + rr * 128, kb * kKB, r0, r1, r2, r3, pol_x);
          } else {
            if (lane == 0) mbar_arrive_expect_tx(full_bar(s), kABytes / kAWarps);
            __syncwarp();
            if (lane < 8) tma_gather4(&tmX, full_bar(s), sA + s * kABytes + rr * 128, kb * kKB, r0, r1, r2, r3, pol_x);
          }
        }
      } else {
        // Byte addressing: a row of X is H * (1 or 2) bytes; thread ch copies bytes [16 ch, 16 ch + 16)
        // of the row's 128-byte K block.
        const int64_t row_bytes = (int64_t)a.H * (kFp8 ? 1 : 2);
        const uint8_t* src[8];
        uint32_t rowok = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = rsub + 16 * j;
          const int tok = r < nvalid ? __ldg(idx + rbeg + r) : 0;
          src[j] = reinterpret_cast<const uint8_t*>(a.X) + (int64_t)tok * row_bytes + ch * 16;
          rowok |= (r < nvalid ? 1u : 0u) << j;
        }
        // Ride tile (kind 3): this CTA's half of the tail's `height` token rows (<= 16: one row per 16-row
        // group thread), staged K-major SW128 in the half of the B slot the tile's W does not use; the swap
        // MMA reads them as its N operand.
        const bool ride = kSplit && t.kind == 3;
        const int ride_n = ride ? t.height / kCta : 0;
        const bool ride_row = rsub < ride_n && (int)rank * ride_n + rsub < (ride ? t.trows : 0);
        const uint8_t* ride_src = reinterpret_cast<const uint8_t*>(a.X) + ch * 16;
        if (ride_row) ride_src += (int64_t)__ldg(a.token_idx + t.trow0 + (int)rank * ride_n + rsub) * row_bytes;
        const uint32_t ride_off = (uint32_t)(1 - t.hh) * (uint32_t)(kBSt / 2) + dst_off;
        // Memory-bound tiles: the A warps (idle but for a few token rows) also pull this CTA's W lines
        // of K block kb + pf_dist into L2 through the load/store path, so the ring's W boxes hit in L2
        // (TMA moves one box per ~330 ns per SM from HBM).
        const bool lsu_pf = a.pf_dist > 0 &&
                            (kCta == 1 || (kSplit && t.kind == 1 && one_box<kWide, kGated>(t.bn, t.ct, a.N, a.w4d, true)));
        const int esz = kFp8 ? 1 : 2;
        const int wcols = kCta == 1 ? t.bn : 256;              // this CTA's W columns of the tile (one box)
        const int wcol0 = kCta == 1 ? t.ct * t.bn : t.ct * t.bn + (int)rank * 256;
        const int lines_row = min(wcols, a.N - wcol0) * esz / 128;   // 128-byte lines per K row (N % 64 == 0)
        const uint8_t* wexp = a.W + (int64_t)t.expert * a.H * a.N * esz + (int64_t)wcol0 * esz;
        for (int kb = k0; kb < k1; ++kb, ++g) {
          const int s = g % kSt;
          if (lsu_pf && lines_row > 0) {
            const int kp = kb == k0 ? kb : kb + a.pf_dist - 1;    // unit start: the first pf_dist blocks
            for (int k2 = kp; k2 < min(kb + a.pf_dist, k1); ++k2) {
              const int n_lines = kKB * lines_row;
              for (int i = threadIdx.x; i < n_lines; i += 32 * kAWarps) {
                const int kr = k2 * kKB + i / lines_row;
                if (kr < a.H) prefetch_l2(wexp + ((int64_t)kr * a.N) * esz + (i % lines_row) * 128);
              }
            }
          }
          wait_timed<kProf>(empty_bar(s), ((g / kSt) & 1u) ^ 1u, c_wait);
          if constexpr (kProf) {
            if (p == 0 && lane == 0) s_ts[kSt + s] = clock64();
          }
#ifdef MOE_EXPERIMENTS
          if (kCta == 2 && (a.experiment & 4)) {
            // 128 CONTIGUOUS X rows by one tile TMA into the leader's barrier (wrong Y: timing only).
            if (p == 0 && lane == 0) {
              const int xr = (t.row0 + rbeg) % max(1, a.T - kBM);
              tma_load_2d_pair(&tmX, leader(full_bar(s)), sA + s * kABytes, kb * kBK, xr, pol_x);
            }
            mbar_arrive(full_bar(s));
            continue;
          }
#endif
#ifdef MOE_EXPERIMENTS
          if (a.experiment & 32) {   // no cp.async at all: plain arrivals (timing only)
            mbar_arrive(full_bar(s));
            continue;
          }
#endif
          const int64_t kbyte = (int64_t)kb * 128;
          const bool colok = kbyte + ch * 16 < row_bytes;
          const uint32_t dst = sA + s * kABytes + dst_off;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
#ifdef MOE_EXPERIMENTS
            const bool ok = !(a.experiment & 1) && colok && ((rowok >> j) & 1u);
#else
            const bool ok = colok && ((rowok >> j) & 1u);
#endif
            cp_async_16(dst + j * 16 * 128, ok ? (const void*)(src[j] + kbyte) : (const void*)a.X, ok ? 16u : 0u);
          }
          if (kSplit && rsub < ride_n) {
            const bool ok = colok && ride_row;
            cp_async_16(sB + s * kBSt + ride_off, ok ? (const void*)(ride_src + kbyte) : (const void*)a.X, ok ? 16u : 0u);
          }
          cp_async_mbar_arrive_noinc(full_bar(s));
        }
      }
    }
    if constexpr (kProf) {
      if (p == 0 && lane == 0) {
        a.prof[blockIdx.x * kProfSlots + kProfProdWaitEmpty] = c_wait;
        a.prof[blockIdx.x * kProfSlots + kProfProdTotal] = clock64() - c_t0;
      }
    }
  } else if (warp == kBWarp) {
    // ===================== B producer: this CTA's share of the W block, one TMA per stage =====================
    const uint64_t pol_w = policy_evict_normal();
    uint32_t g = 0;
    long long c_wait = 0, c_t0 = kProf ? clock64() : 0, c_rel = 0;
    int v_next = pair_id;                           // dynamic order, leader lane 0: the next position fetched
    // MOE_ORDER_LIGHT_LAST: virtual tiles [0, C) are heavy tasks', [C, total) light tasks'.
    // Fetch position i takes the Bresenham merge of the two runs: light iff floor((i+1) L / total) >
    // floor(i L / total), L = total - C, so every window of consecutive fetches holds both kinds in
    // proportion while each run keeps its own order (row tiles of a column block stay together).
    int light0 = total;
    if (dyn && rank == 0 && a.light_merge) {
      const int M = __ldg(a.plan + 1);
      int h = 0;
      while (h < M && __ldg(params + s_sigma[h] * MOE_PLAN_TASK_WORDS + 2) > MOE_LIGHT_ROWS) ++h;
      light0 = h == 0 ? 0 : s_prefix[h - 1];
    }
    auto merged = [&](int i) -> int {
      if (i >= total || light0 >= total) return i;
      const long long L = total - light0;
      const int before = (int)((long long)i * L / total), upto = (int)((long long)(i + 1) * L / total);
      return upto > before ? light0 + before : i - before;
    };
    // Half tiles last: fetch positions [0, n_full) walk the full tiles in virtual order
    // (each task's row tiles [0, R - f) of every column block, row tile fastest), [n_full, total) the half
    // tiles (f = 1: the task's last row tile holds <= 128 rows).  All 32 lanes: per-lane task data, a warp
    // scan of the per-task counts and a vote find the task holding position pos (Alg. 2's search on a
    // derived prefix), then the tile's virtual index in the plan's own order.
    const int mt = __ldg(a.plan + 1);               // tasks with tiles (sigma's length)
    auto task_rf = [&](int hh, int& R, int& f, int& C) {
      const int tk = s_sigma[hh];
      const int4 pb = __ldg(reinterpret_cast<const int4*>(params + tk * MOE_PLAN_TASK_WORDS + 4));
      const int rows = __ldg(params + tk * MOE_PLAN_TASK_WORDS + 2);
      R = pb.z;
      C = pb.w;
      f = rows - (R - 1) * kPairRows <= kPairRows / 2 ? 1 : 0;
    };
    int n_full = total;
    if (dyn && rank == 0 && a.half_last) {
      int nh = 0;
      for (int c = 0; c < mt; c += 32) {
        int R = 0, f = 0, C = 0;
        if (c + lane < mt) task_rf(c + lane, R, f, C);
        nh += __reduce_add_sync(0xffffffffu, f * C);
      }
      n_full = total - nh;
    }
    // Narrow column block last: when N is not a multiple of bn the last column block of
    // every task is narrower; fetch positions [0, total (C-1)/C) walk the full-width column blocks, the rest
    // the narrow ones, each run in the plan's order.  Task h owns R_h (C-1) / R_h tiles of each run, i.e.
    // TilePrefix x (C-1) / C and TilePrefix / C (exact: every task has R_h x C tiles): Alg. 2's vote on the
    // scaled prefix finds the task, and the tile keeps its (rt, ct), so a column block stays together.
    auto narrow_reorder = [&](int pos) -> int {
      const int C = a.narrow_last;                     // column tiles per task (> 1)
      const int n_wide = (int)((long long)total * (C - 1) / C);
      if (pos >= total) return pos;
      const bool second = pos >= n_wide;
      const int q = second ? pos - n_wide : pos;
      for (int c = 0; c < mt; c += 32) {
        const int hh = c + lane;
        const long long pf = hh < mt ? (long long)s_prefix[hh] : (long long)total;
        const long long pref = second ? pf / C : pf * (C - 1) / C;
        const unsigned mask = __ballot_sync(0xffffffffu, hh < mt && q >= pref);
        const int nb = __popc(mask);
        if (nb < 32) {
          const int h = c + nb;
          const int first = h > 0 ? s_prefix[h - 1] : 0;
          const int start = second ? first / C : (int)((long long)first * (C - 1) / C);
          const int l = q - start;
          const int R = (s_prefix[h] - first) / C;
          return second ? first + (C - 1) * R + l : first + l;
        }
      }
      return pos;
    };
    auto half_reorder = [&](int pos) -> int {
      if (pos >= total || n_full >= total) return pos;
      const bool second = pos >= n_full;
      const int q = second ? pos - n_full : pos;
      int base = 0;
      for (int c = 0; c < mt; c += 32) {
        const int hh = c + lane;
        int R = 1, f = 0, C = 0;
        if (hh < mt) task_rf(hh, R, f, C);
        int cnt = hh < mt ? (second ? f * C : (R - f) * C) : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, cnt, o);
          if (lane >= o) cnt += y;
        }
        const int pref = base + cnt;                 // this kind's tiles through task hh
        const unsigned before_mask = __ballot_sync(0xffffffffu, hh < mt && q >= pref);
        const int nb = __popc(before_mask);
        if (nb < 32) {
          const int h = c + nb;
          const int start = nb == 0 ? base : __shfl_sync(0xffffffffu, pref, nb - 1);
          const int Rh = __shfl_sync(0xffffffffu, R, nb), fh = __shfl_sync(0xffffffffu, f, nb);
          const int l = q - start;
          const int first = h > 0 ? s_prefix[h - 1] : 0;
          if (second) return first + l * Rh + (Rh - 1);            // column block l, last row tile
          const int rf = Rh - fh;
          return first + (l / rf) * Rh + (l % rf);
        }
        base = __shfl_sync(0xffffffffu, pref, 31);
      }
      return pos;
    };
    for (uint32_t qi = 0;; ++qi) {
      int v, k0 = 0, k1 = a.num_kb;
      if (dyn && rank == 0) {                       // the producer of the pair's tile queue
        const int pos = __shfl_sync(0xffffffffu, v_next, 0);
        v = a.light_merge ? merged(pos) : a.half_last ? half_reorder(pos) : a.narrow_last > 1 ? narrow_reorder(pos) : pos;
        const int sl = (int)(qi % kQ);
        mbar_wait(qempty_bar(sl), ((qi / kQ) & 1u) ^ 1u);
        if (lane == 0) {
          q_slot[sl] = v;
          if constexpr (kCta == 2) {
            st_shared_cluster_u32(mapa_shared(s_q + 4u * sl, 1), (uint32_t)v);
            mbar_arrive_release_cluster(mapa_shared(qfull_bar(sl), 1));
          }
          mbar_arrive(qfull_bar(sl));
          // fetch the next position now: the atomic's latency hides behind this tile's loads
          if (pos < total) v_next = n_pairs + atomicAdd(a.sched, 1);
        }
        __syncwarp();
      } else if (!next_unit(qi, v, k0, k1)) {
        break;
      }
      if (v >= total) break;
      int h, task, l;
      map_tile(s_prefix, s_sigma, a.M_pad, v, h, task, l);
      const Tile t = load_tile<kSplit>(params, task, l, ride_ok);
      const int bnp = t.bn / kHalves;               // columns of one MMA block (gated: 128 gate + 128 up)
      const int bnc = kGated ? 128 : bnp / kCta;    // columns of an MMA block staged by this CTA
      const int n0 = kGated ? t.ct * t.bn : t.ct * t.bn + (int)rank * bnc;   // block h at n0 + h * bnp
      const int nbox = (bnc + (1 << kCS) - 1) >> kCS;
      // (a ride tile stages only its half's block, in the two-box layout: block hh at offset hh * kBSt / 2)
      const bool one = kCta == 2 && !(kSplit && t.kind == 3) &&
                       one_box<kWide, kGated>(t.bn, t.ct, a.N, a.w4d, kSplit && t.kind == 1);
      const int n_one = t.ct * t.bn + (int)rank * 256;   // one box: this CTA's 256 columns
      for (int kb = k0; kb < k1; ++kb, ++g) {
        const int s = g % kSt;
        wait_timed<kProf>(empty_bar(s), ((g / kSt) & 1u) ^ 1u, c_wait);
        if constexpr (kProf) {
          if (lane == 0) {
            const long long now = clock64();
            if (g >= (uint32_t)kSt) c_rel += now - s_ts[2 * kSt + s];   // slot's previous commit
            s_ts[s] = now;
          }
        }
#ifdef MOE_EXPERIMENTS
        if (a.experiment & 2) {
          if (lane == 0 && rank == 0) mbar_arrive(full_bar(s));
          __syncwarp();
          continue;
        }
#endif
        if (lane == 0) {
          const uint32_t dstB = sB + s * kBSt;
          if (kCta == 2 && one) {
            // both blocks' W columns of this CTA in one box (tmW2 has the 2 x nbox-chunk box)
            const uint32_t fb = leader(full_bar(s));
            uint32_t bytes = (uint32_t)(kCta * 2 * nbox * kBox);
            if (a_mode == 2 || a_mode == 0) bytes += kCta * kABytes;
            if (rank == 0) mbar_arrive_expect_tx(full_bar(s), bytes);
            tma_load_4d_pair(&tmW2, fb, dstB, 0, kb * kKB, n_one >> kCS, t.expert, pol_w);
          } else if constexpr (kCta == 2) {
            const uint32_t fb = leader(full_bar(s));
            // Per block: this CTA's first column and boxes.  Wide kind-0 tiles passing N stage only
            // the trimmed block (wide_block_cols); the 4-D box always moves nbox chunks.
            int nh[kHalves], nbx[kHalves];
            uint32_t bytes = 0;
#pragma unroll
            for (int hf = 0; hf < kHalves; ++hf) {
              nh[hf] = n0 + hf * bnp;
              nbx[hf] = nbox;
              if constexpr (kWide && !kGated) {
                if (!(kSplit && t.kind == 1)) {
                  const int nc = wide_block_cols<kFp8>(t.bn, t.ct, a.N, hf);
                  nh[hf] = t.ct * t.bn + hf * bnp + (int)rank * (nc / 2);
                  nbx[hf] = nc == 0 ? 0 : a.w4d ? nbox : (nc / 2 + (1 << kCS) - 1) >> kCS;
                  if (kSplit && t.kind == 3 && hf != t.hh) nbx[hf] = 0;   // ride: the tile's half only
                }
              }
              bytes += kCta * nbx[hf] * kBox;
            }
            if (a_mode == 2 || a_mode == 0) bytes += kCta * kABytes;   // both CTAs' contiguous-row A tiles
#ifdef MOE_EXPERIMENTS
            if (rank == 0) mbar_arrive_expect_tx(full_bar(s), bytes + ((a.experiment & 4) ? kCta * kABytes : 0));
#else
            if (rank == 0) mbar_arrive_expect_tx(full_bar(s), bytes);
#endif
#pragma unroll
            for (int hf = 0; hf < kHalves; ++hf) {
              if (nbx[hf] == 0) continue;
              const uint32_t dst = dstB + hf * nbox * kBox;
              const CUtensorMap* wm = kGated && rank == 1 ? &tmW2 : &tmW;   // gated: leader gate, peer up
              if (a.w4d) {
                tma_load_4d_pair(wm, fb, dst, 0, kb * kKB, nh[hf] >> kCS, t.expert, pol_w);
              } else {
                for (int j = 0; j < nbx[hf]; ++j)
                  tma_load_3d_pair(wm, fb, dst + j * kBox, nh[hf] + (j << kCS), kb * kKB, t.expert, pol_w);
              }
            }
          } else {
            mbar_arrive_expect_tx(full_bar(s), nbox * kBox);
            if (a.w4d) {
              tma_load_4d(&tmW, full_bar(s), dstB, 0, kb * kKB, n0 >> kCS, t.expert, pol_w);
            } else {
              for (int j = 0; j < nbox; ++j)
                tma_load_3d(&tmW, full_bar(s), dstB + j * kBox, n0 + (j << kCS), kb * kKB, t.expert, pol_w);
            }
          }
        }
        __syncwarp();
      }
    }
    if (dyn && rank == 0 && lane == 0) {
      // Every pair ends here exactly once; the last one resets the counters for the next launch on
      // this plan (launches on one plan are stream-ordered).
      __threadfence();
      if (atomicAdd(a.sched + 1, 1) == n_pairs - 1) {
        atomicExch(a.sched, 0);
        atomicExch(a.sched + 1, 0);
      }
    }
    if constexpr (kProf) {
      if (lane == 0) {
        a.prof[blockIdx.x * kProfSlots + kProfBWaitEmpty] = c_wait;
        a.prof[blockIdx.x * kProfSlots + kProfBTotal] = clock64() - c_t0;
        a.prof[blockIdx.x * kProfSlots + kProfRelease] = c_rel;
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (pair leader): one thread drives tcgen05 =====================
    if (rank == 0) {
      uint32_t g = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      long long c_tmem = 0, c_full = 0, c_t0 = kProf ? clock64() : 0, c_lb = 0, c_la = 0, c_ns = 0;
      long long c_issue = 0, c_gap = 0, t_end = 0;
      int n_tiles = 0;
      for (uint32_t qi = 0;; ++qi) {
        int v, k0, k1;
        if (!next_unit(qi, v, k0, k1)) break;
        ++n_tiles;
        int h, task, l;
        map_tile(s_prefix, s_sigma, a.M_pad, v, h, task, l);
        const Tile t = load_tile<kSplit>(params, task, l, ride_ok);
        const bool swap = kSplit && t.kind == 1;
        // kind 0: D[tokens, cols] = A[tokens (K-major)] * B[W block (MN-major)], N = bn.
        // kind 1: D[cols, tokens] = A[W block as MN-major M-operand] * B[tail tokens (K-major)],
        //         M = the pair's 256 output columns, N = the tail height (swap-AB).
        const uint32_t idesc = swap ? idesc_bf16_f32(kPairRows, t.height, /*A MN-major*/ 1, /*B K-major*/ 0)
                                    : idesc_f32acc<kFp8>(kPairRows, kGated ? 256 : t.bn / kHalves,
                                                         /*A K-major*/ 0, /*B MN-major*/ 1);
        // Wide tiles past N (the last column tile when N is not a multiple of bn): each block's MMA
        // covers wide_block_cols columns (zero: the block is skipped), matching what the B warp staged.
        uint32_t idesc_blk[2] = {idesc, idesc};
        int ncol_blk[2] = {1, 1};
        if constexpr (kWide && !kGated) {
          if (!swap) {
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              ncol_blk[hf] = wide_block_cols<kFp8>(t.bn, t.ct, a.N, hf);
              const int m = half_tile<kWide, kGated>(t.rows, t.rt, false) ? kPairRows / 2 : kPairRows;
              if (ncol_blk[hf] > 0) idesc_blk[hf] = idesc_f32acc<kFp8>(m, ncol_blk[hf], 0, 1);
            }
          }
        }
        // Ride tile (kind 3): block 0 = the body (M = 256 rows x the half's 256 columns), block 1 = the tail
        // (swap-AB: the same staged W as the M = 256 operand, the tail tokens as N = height) in TMEM
        // columns [256, 256 + height).
        const bool ride = kSplit && t.kind == 3;
        if (ride) idesc_blk[1] = idesc_bf16_f32(kPairRows, t.height, /*A MN-major*/ 1, /*B K-major*/ 0);
        if constexpr (kWide) {
          // Wide tiles (TMEM holds one accumulator: block 0 = columns [0,256), block 1 = [256,512)).
          // Block-staggered order so the epilogue drains one block while the other is still
          // accumulating:
          //   prologue  block 0 over K blocks [0, D)      (needs only block 0 of the last tile drained)
          //             block 1 over [0, D), freeing each stage
          //   middle    both blocks per K block, freeing each stage
          //   tail      block 0 over [tail0, n), commit "block 0 full"; block 1 over [tail0, n), freeing,
          //             commit "block 1 full"
          // D = min(stages, n); the tail holds at most the whole ring.
          const int n = a.num_kb;
          const int D = min(kSt, n);
          const int tail0 = max(D, n - D);
          const uint32_t g0 = g;
          auto slot = [&](int kb) { return (int)((g0 + kb) % kSt); };
          auto wait_kb = [&](int kb) {
            if constexpr (kProf) {
              if (kb == 0 && n_tiles > 1) c_gap += clock64() - t_end;
            }
            wait_timed<kProf>(full_bar(slot(kb)), ((g0 + kb) / kSt) & 1u, c_full);
            if constexpr (kProf) {
              const long long now = clock64();
              c_lb += now - s_ts[slot(kb)];
              c_la += now - s_ts[kSt + slot(kb)];
              ++c_ns;
            }
            tc_fence_after();
          };
          auto issue = [&](int hf, int kb) {
            if (lane == 0) {
              const uint32_t a0 = sA + slot(kb) * kABytes;
              const uint32_t b0 = sB + slot(kb) * kBSt + hf * (kBSt / 2);
              const uint32_t d = tmem_base + hf * kAccCols;
              if (kSplit && swap) {
                // swap-AB tail (kSplit kind 1): the W block is the M = 256 operand, tokens the N one
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk)
                  mma_bf16_pair(d, smem_desc_sw128(b0 + kk * 2048, kBBoxBytes, 1024),
                                smem_desc_sw128(a0 + kk * 32, 16, 1024), idesc, (kb | kk) != 0);
              } else if (kSplit && ride) {
                const uint32_t wB = sB + slot(kb) * kBSt + t.hh * (kBSt / 2);         // the half's staged W
                if (hf == 0) {
#pragma unroll
                  for (int kk = 0; kk < kBK / 16; ++kk)
                    mma_issue<kFp8, 2>(d, smem_desc_sw128(a0 + kk * 32, 16, 1024),
                                       smem_desc_sw128(wB + kk * kKStep, kBox, 1024), idesc_blk[0], (kb | kk) != 0);
                } else {
                  const uint32_t tok = sB + slot(kb) * kBSt + (1 - t.hh) * (kBSt / 2);   // the tail tokens
#pragma unroll
                  for (int kk = 0; kk < kBK / 16; ++kk)
                    mma_bf16_pair(d, smem_desc_sw128(wB + kk * 2048, kBBoxBytes, 1024),
                                  smem_desc_sw128(tok + kk * 32, 16, 1024), idesc_blk[1], (kb | kk) != 0);
                }
              } else if (ncol_blk[hf] > 0) {
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk)
                  mma_issue<kFp8, 2>(d, smem_desc_sw128(a0 + kk * 32, 16, 1024),
                                     smem_desc_sw128(b0 + kk * kKStep, kBox, 1024), idesc_blk[hf], (kb | kk) != 0);
              }
            }
            __syncwarp();
          };
          auto release = [&](int kb) {
            if constexpr (kProf) {
              if (lane == 0) s_ts[2 * kSt + slot(kb)] = clock64();
            }
            if (lane == 0) mma_commit_pair(empty_bar(slot(kb)), 0x3);   // frees the slot in both CTAs
            __syncwarp();
          };
          auto block_full = [&](int hf) {
            if (lane == 0) mma_commit_pair(tfull_bar(hf), 0x3);          // block hf final in both CTAs
            __syncwarp();
          };
          const long long t_i = kProf ? clock64() : 0;
#ifdef MOE_EXPERIMENTS
          if (!(a.experiment & 64))                                      // 64: never wait (timing only)
#endif
          wait_timed<kProf>(tempty_bar(0), acc_phase ^ 1u, c_tmem);    // block 0 of the last tile drained
          tc_fence_after();
          for (int kb = 0; kb < D; ++kb) {
            wait_kb(kb);
            issue(0, kb);
          }
          if (n == D) block_full(0);
#ifdef MOE_EXPERIMENTS
          if (!(a.experiment & 64))
#endif
          wait_timed<kProf>(tempty_bar(1), acc_phase ^ 1u, c_tmem);
          tc_fence_after();
          for (int kb = 0; kb < D; ++kb) {
            issue(1, kb);
            release(kb);
          }
          if (n == D) block_full(1);
          for (int kb = D; kb < tail0; ++kb) {
            wait_kb(kb);
            issue(0, kb);
            issue(1, kb);
            release(kb);
          }
          if (tail0 < n) {
            for (int kb = tail0; kb < n; ++kb) {
              wait_kb(kb);
              issue(0, kb);
            }
            block_full(0);
            for (int kb = tail0; kb < n; ++kb) {
              issue(1, kb);
              release(kb);
            }
            block_full(1);
          }
          g += n;
          if constexpr (kProf) {
            c_issue += clock64() - t_i;
            t_end = clock64();
          }
        } else {
          // Double-buffered: wait for accumulator `acc`.
          wait_timed<kProf>(tempty_bar(acc), acc_phase ^ 1u, c_tmem);     // epilogue(s) drained this accumulator
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * kAccCols;
          for (int kb = k0; kb < k1; ++kb, ++g) {
            const int s = g % kSt;
            const uint32_t par = (g / kSt) & 1u;
            if constexpr (kProf) {
              if (kb == k0 && n_tiles > 1) c_gap += clock64() - t_end;  // decode + accumulator hand-off
            }
            wait_timed<kProf>(full_bar(s), par, c_full);                   // both CTAs' bytes landed
            if (g == 0 && lane == 0) MOE_TL(3);                             // first stage landed (1-CTA / pair)
            long long t_i = 0;
            if constexpr (kProf) {
              const long long now = clock64();
              c_lb += now - s_ts[s];
              c_la += now - s_ts[kSt + s];
              ++c_ns;
              t_i = now;
            }
            tc_fence_after();
            if (lane == 0) {
              const uint32_t a0 = sA + s * kABytes;
              const uint32_t b0 = sB + s * kBSt;
              // Token rows: K-major SW128, 8-row groups 1024 B apart; K step of 16 = +32 B in the row.
              // W block: MN-major SW128; 64-wide chunks 8 KB apart (LBO), 8-row K groups 1 KB apart
              // (SBO); K step of 16 rows = +2 KB.  The two kinds only swap the operand roles.
#ifdef MOE_EXPERIMENTS
              if (!kFp8 && (a.experiment & 16)) {   // B read as K-major (wrong Y): is the MN-major B operand slower?
                const uint32_t idk = idesc_bf16_f32(kPairRows, kGated ? 256 : t.bn / kHalves, 0, 0);
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk) {
                  const uint64_t ad = smem_desc_sw128(a0 + kk * 32, 16, 1024);
                  const uint64_t bd = smem_desc_sw128(b0 + kk * 32, 16, 1024);
                  if constexpr (kCta == 2) mma_bf16_pair(d_tmem, ad, bd, idk, (kb | kk) != 0);
                  else mma_bf16(d_tmem, ad, bd, idk, (kb | kk) != 0);
                }
              } else
#endif
              if (!kSplit || !swap) {
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk) {
                  const uint64_t ad = smem_desc_sw128(a0 + kk * 32, 16, 1024);
                  const uint64_t bd = smem_desc_sw128(b0 + kk * kKStep, kBox, 1024);
                  mma_issue<kFp8, kCta>(d_tmem, ad, bd, idesc, kb != k0 || kk != 0);
                }
              } else {
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk) {
                  const uint64_t ad = smem_desc_sw128(b0 + kk * 2048, kBBoxBytes, 1024);
                  const uint64_t bd = smem_desc_sw128(a0 + kk * 32, 16, 1024);
                  if constexpr (kCta == 2) mma_bf16_pair(d_tmem, ad, bd, idesc, kb != k0 || kk != 0);
                  else mma_bf16(d_tmem, ad, bd, idesc, kb != k0 || kk != 0);
                }
              }
              if constexpr (kProf) s_ts[2 * kSt + s] = clock64();
              if constexpr (kCta == 2) mma_commit_pair(empty_bar(s), 0x3);  // frees the slot in both CTAs
              else mma_commit(empty_bar(s));
            }
            __syncwarp();
            if constexpr (kProf) c_issue += clock64() - t_i;
          }
          if constexpr (kProf) t_end = clock64();
          if (lane == 0) {
            if constexpr (kCta == 2)   // accumulator ready in both CTAs of this pair
              mma_commit_pair(tfull_bar(acc), 0x3);
            else mma_commit(tfull_bar(acc));
          }
          __syncwarp();
        }
        if constexpr (kWide) {
          acc_phase ^= 1u;                        // one (two-half) accumulator per tile
        } else if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
      }
      if (lane == 0) MOE_TL(4);                             // last MMA issued
      if constexpr (kProf) {
        if (lane == 0) {
          long long* o = a.prof + blockIdx.x * kProfSlots;
          o[kProfMmaWaitTmem] = c_tmem;
          o[kProfMmaWaitFull] = c_full;
          o[kProfMmaTotal] = clock64() - c_t0;
          o[kProfTiles] = n_tiles;
          o[kProfLatB] = c_lb;
          o[kProfLatA] = c_la;
          o[kProfStages] = c_ns;
          o[kProfMmaIssue] = c_issue;
          o[kProfMmaTileGap] = c_gap;
        }
      }
    } else if (lane == 0 && a_mode == 1) {
      // Pair peer: relay "my A stage landed" (local full barrier, fed by cp.async arrivals) to the
      // leader's full barrier, where the MMA issuer waits for both CTAs' bytes.
      uint32_t g = 0;
      for (uint32_t qi = 0;; ++qi) {
        if (tile_of_lane(qi) >= total) break;
        for (int kb = 0; kb < a.num_kb; ++kb, ++g) {
          const int s = g % kSt;
          mbar_wait(full_bar(s), (g / kSt) & 1u);
          mbar_arrive_cluster(leader(full_bar(s)));
        }
      }
    }
  } else {
    // ===================== epilogue: TMEM -> registers -> Y =====================
    const int q = warp & 3;                                   // TMEM lane quarter of this warp
    const int ew = warp - (kMmaWarp + 1);                     // epilogue warp index
    const int cg = ew >> 2;                                   // column group: chunks c/32 = cg mod kEpiGroups
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t n_chunk = 0;                                     // TMA-store chunks issued by this warp
    const uint32_t ebuf = sEpi + (uint32_t)ew * kEpiBufBytes;
    long long c_wait = 0, c_work = 0;
    // ---- MOE_KIND_GEMV side work (wide kernels) ----
    GemvUnit<kFp8> gu;
    int g_units = -1;                               // -1: not counted yet; 0: none / queue exhausted
    const int nb_cols = (a.N + kGemvCols - 1) / kGemvCols;
    const int n_tasks_all = __ldg(a.plan + 9);
    auto is_gemv = [&](int tk) {
      return tk < n_tasks_all && __ldg(params + tk * MOE_PLAN_TASK_WORDS + 3) == MOE_KIND_GEMV &&
             __ldg(params + tk * MOE_PLAN_TASK_WORDS + 2) > 0;
    };
    auto count_gemv = [&]() {
      int n = 0;
      for (int b = 0; b < n_tasks_all; b += 32) n += __popc(__ballot_sync(0xffffffffu, is_gemv(b + lane)));
      return n;
    };
    auto find_gemv = [&](int j) -> int {           // the j-th GEMV task in task order
      for (int b = 0; b < n_tasks_all; b += 32) {
        const unsigned m = __ballot_sync(0xffffffffu, is_gemv(b + lane));
        const int c = __popc(m);
        if (j < c) return b + __fns(m, 0, j + 1);
        j -= c;
      }
      return -1;
    };
    const size_t esz_in = kFp8 ? 1 : 2;
    auto gemv_round = [&]() -> bool {               // one 16-row round of this warp's unit; false: no work left
      if constexpr (!kWide || kGated) {
        return false;
      } else {
        if (a.gemv_q == nullptr || g_units == 0) return false;
        if (gu.task < 0) {
          if (g_units < 0) g_units = count_gemv() * nb_cols;
          int u = 0;
          if (lane == 0) u = g_units > 0 ? atomicAdd(a.gemv_q, 1) : 0;
          u = __shfl_sync(0xffffffffu, u, 0);
          if (u >= g_units) {
            if (lane == 0 && atomicAdd(a.gemv_q + 1, 1) == (int)(gridDim.x * kEpiWarps) - 1) {
              a.gemv_q[0] = 0;                      // every epilogue warp is done: reset for the next launch
              a.gemv_q[1] = 0;
            }
            g_units = 0;
            return false;
          }
          const int j = u / nb_cols;
          gu.task = find_gemv(j);
          gu.expert = __ldg(params + gu.task * MOE_PLAN_TASK_WORDS + 0);
          gu.row0 = __ldg(params + gu.task * MOE_PLAN_TASK_WORDS + 1);
          gu.rows = __ldg(params + gu.task * MOE_PLAN_TASK_WORDS + 2);
          gu.col0 = (u - j * nb_cols) * kGemvCols + (lane & 15) * 8;
          gu.kpos = 0;
#pragma unroll
          for (int t = 0; t < MOE_GEMV_MAX_ROWS; ++t)
#pragma unroll
            for (int i = 0; i < 8; ++i) gu.acc[t][i] = 0.f;
        }
        const bool colok = gu.col0 < a.N;
        const uint8_t* wbase = a.W + ((size_t)gu.expert * a.H) * a.N * esz_in + (size_t)gu.col0 * esz_in;
        // a round = kGemvBatch batches of 16 K rows: batch b, half-warp h takes rows kpos + 16 b + 8 h + [0, 8)
        const int64_t xrow = (int64_t)a.H * esz_in;
#pragma unroll
        for (int b = 0; b < kGemvBatch; ++b) {
          const int kr = gu.kpos + 16 * b + 8 * (lane >> 4);
          if (colok && kr < a.H) {
            uint4 wv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) wv[i] = GemvUnit<kFp8>::load8(wbase + (size_t)(kr + i) * a.N * esz_in);
#pragma unroll
            for (int t = 0; t < MOE_GEMV_MAX_ROWS; ++t) {
              if (t < gu.rows) {
                const int tok = a.token_idx ? __ldg(a.token_idx + gu.row0 + t) : gu.row0 + t;
                const uint8_t* xp = reinterpret_cast<const uint8_t*>(a.X) + tok * xrow + (int64_t)kr * esz_in;
                uint4 xq;
                if constexpr (kFp8) {
                  const uint2 v2 = __ldg(reinterpret_cast<const uint2*>(xp));
                  xq = make_uint4(v2.x, v2.y, 0u, 0u);
                } else {
                  xq = __ldg(reinterpret_cast<const uint4*>(xp));
                }
                float xf[8];
                GemvUnit<kFp8>::widen(xq, xf);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  float wf[8];
                  GemvUnit<kFp8>::widen(wv[i], wf);
#pragma unroll
                  for (int c = 0; c < 8; ++c) gu.acc[t][c] = fmaf(xf[i], wf[c], gu.acc[t][c]);
                }
              }
            }
          }
        }
        gu.kpos += 16 * kGemvBatch;
        if (gu.kpos >= a.H) {                       // unit done: sum the two half-warps, store the rows
          float sc = 1.f;
          if constexpr (kFp8) sc = a.scale ? __ldg(a.scale + gu.expert) : 1.f;
#pragma unroll
          for (int t = 0; t < MOE_GEMV_MAX_ROWS; ++t) {
            uint32_t r[32];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float v2 = gu.acc[t][c] + __shfl_xor_sync(0xffffffffu, gu.acc[t][c], 16);
              r[c] = __float_as_uint(kFp8 ? v2 * sc : v2);
            }
            if (t < gu.rows && lane < 16 && colok) {
              const int grow = gu.row0 + t;
              uint8_t* yp = a.y_row_ptr ? reinterpret_cast<uint8_t*>(__ldg(a.y_row_ptr + grow))
                                        : reinterpret_cast<uint8_t*>(a.Y) +
                                              (a.y_row_map ? (int64_t)__ldg(a.y_row_map + grow) : (int64_t)grow) *
                                                  a.N * (a.y_f32 ? 4 : 2);
              if (a.y_f32) {
                float* y = reinterpret_cast<float*>(yp) + gu.col0;
                *reinterpret_cast<uint4*>(y) = make_uint4(r[0], r[1], r[2], r[3]);
                *reinterpret_cast<uint4*>(y + 4) = make_uint4(r[4], r[5], r[6], r[7]);
              } else {
                *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(yp) + gu.col0) =
                    make_uint4(pack_bf16(r[0], r[1]), pack_bf16(r[2], r[3]), pack_bf16(r[4], r[5]),
                               pack_bf16(r[6], r[7]));
              }
            }
          }
          gu.task = -1;
        }
        return true;
      }
    };
    // Wait for an accumulator phase; with GEMV work queued, work on it while the phase is pending.
    auto wait_acc = [&](uint32_t bar, uint32_t phase) {
      if (a.gemv_q != nullptr && g_units != 0) {
        while (!mbar_test_wait(bar, phase)) {
          if (!gemv_round()) {
            wait_timed<kProf>(bar, phase, c_wait);
            return;
          }
        }
        return;
      }
      wait_timed<kProf>(bar, phase, c_wait);
    };
    // Wide tiles: "block 0 full" is awaited with the tile, "block 1 full" before draining block 1.
    auto wait_block1 = [&](int hf) {
      if (kWide && hf == 1) {
        wait_acc(tfull_bar(1), acc_phase);
        tc_fence_after();
      }
    };
    for (uint32_t qi = 0;; ++qi) {
      int v, k0, k1;
      const long long unit = sk_pos;                // split-K: this unit's index (its partial slot)
      if (!next_unit(qi, v, k0, k1)) break;
      int h, task, l;
      map_tile(s_prefix, s_sigma, a.M_pad, v, h, task, l);
      const Tile t = load_tile<kSplit>(params, task, l, ride_ok);
      wait_acc(tfull_bar(acc), acc_phase);
      const long long w0 = kProf ? clock64() : 0;
      tc_fence_after();
      if (kSplit && t.kind == 1) {
        // Swap-AB tile (tail / small task, the catalog's second strategy): TMEM lane = output column
        // (this CTA's 128 of each 256-column block: t.ct * bn + 256 hf + 128 rank + lane), TMEM column
        // = token.  Warp (q, cg) drains lanes 32q..32q+31 for the token chunks c = 32 cg, 32 cg +
        // 32 kEpiGroups, ...; for each token j of a chunk the warp stores 32 consecutive columns of
        // that token's Y row (one coalesced 64 / 128-byte store) — no transpose through shared
        // memory, no barrier between warps.  Every warp frees each block as on kind-0 tiles.
        const int esz = a.y_f32 ? 4 : 2;
        const int bnb = t.bn / kHalves;                           // columns of one TMEM block
#pragma unroll 1
        for (int hf = 0; hf < kHalves; ++hf) {
          wait_block1(hf);
          const int slot = kWide ? hf : acc;
          const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + slot * kAccCols;
          const bool one = kCta == 2 && one_box<kWide, kGated>(t.bn, t.ct, a.N, a.w4d, true);
          const int col = one ? w_col(true, t.ct, t.bn, hf, (int)rank, q * 32 + lane)
                              : t.ct * t.bn + hf * bnb + (int)rank * (bnb / kCta) + q * 32 + lane;
          const bool col_ok = col < a.N && (one || col < t.ct * t.bn + hf * bnb + ((int)rank + 1) * (bnb / kCta));
          for (int c = 32 * cg; c < t.height; c += 32 * kEpiGroups) {
            uint32_t r[32];
            tmem_ld32(taddr + c, r);
            // token row address of token c + lane (broadcast per j below)
            const int tk = min(c + lane, t.rows - 1);
            uint8_t* rp = a.y_row_ptr ? reinterpret_cast<uint8_t*>(__ldg(a.y_row_ptr + t.row0 + tk))
                                      : reinterpret_cast<uint8_t*>(a.Y) +
                                            (a.y_row_map ? (int64_t)__ldg(a.y_row_map + t.row0 + tk)
                                                         : (int64_t)t.row0 + tk) * a.N * esz;
            tmem_wait_ld();
            const int ntok = min(32, t.rows - c);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              uint8_t* row = reinterpret_cast<uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(rp), j));
              if (j < ntok && col_ok) {
                if (a.y_f32)
                  reinterpret_cast<float*>(row)[col] = __uint_as_float(r[j]);
                else
                  reinterpret_cast<__nv_bfloat16*>(row)[col] = __float2bfloat16_rn(__uint_as_float(r[j]));
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (kCta == 2) mbar_arrive_cluster(leader(tempty_bar(slot)));
            else mbar_arrive(tempty_bar(slot));
          }
        }
        if constexpr (kProf) c_work += clock64() - w0;
        if constexpr (kWide) {
          acc_phase ^= 1u;
        } else if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
        continue;
      }
      // Half tiles (M = 128 pair MMA): lane quarters 0/1 hold rows 0-31 / 32-63 of this CTA's 64
      // for the block's first half of columns, quarters 2/3 the same rows for the second half.
      const bool hlf = half_tile<kWide, kGated>(t.rows, t.rt, kSplit && t.kind == 1);
      const int grow = hlf ? t.rt * kPairRows + (int)rank * (kBM / 2) + (q & 1) * 32 + lane
                           : t.rt * kPairRows + (int)rank * kBM + q * 32 + lane;   // row within the task
      const bool valid = grow < t.rows;
      const int64_t yrow = a.y_row_map ? (int64_t)__ldg(a.y_row_map + t.row0 + min(grow, t.rows - 1))
                                       : (int64_t)t.row0 + grow;
      uint8_t* const yrow_ptr =
          a.y_row_ptr ? reinterpret_cast<uint8_t*>(__ldg(a.y_row_ptr + t.row0 + min(grow, t.rows - 1)))
                      : reinterpret_cast<uint8_t*>(a.Y) + yrow * a.N * (a.y_f32 ? 4 : 2);
      const int wrow0 = grow - lane;                // first task row of this warp's quarter
      const bool tma_rows = a.tma_store && wrow0 + 32 <= t.rows;
      const uint32_t xr = (uint32_t)((lane >> 1) & 3);
      // Write 32 fp32 results of this lane's row at columns [col, col + 32).  Full 32-row quarters:
      // bf16 into a 64B-swizzled 32 x 32 staging buffer (conflict-free 16-byte st.shared) and one TMA
      // tile store (with four warps two buffers alternate, so converting chunk i+1 overlaps storing
      // chunk i).  Quarters holding the task's last rows take masked register stores: a box must not
      // touch the next task's rows.
      auto put_chunk = [&](uint32_t (&r)[32], int col, int col_end) {
#ifdef MOE_EXPERIMENTS
        if (a.experiment & 8) return;
#endif
        if (tma_rows && col + 32 <= col_end) {        // a box never crosses the block / N
          const uint32_t buf = kEpiDbuf ? ebuf + (n_chunk & 1u) * 2048u : ebuf;
          if (lane == 0) {                                  // the store that last used buf has read it
            if constexpr (kEpiDbuf) bulk_wait_group_read<1>();
            else bulk_wait_group_read<0>();
          }
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; ++j)
            st_shared_v4(buf + lane * 64 + ((j ^ xr) << 4), pack_bf16(r[8 * j], r[8 * j + 1]),
                         pack_bf16(r[8 * j + 2], r[8 * j + 3]), pack_bf16(r[8 * j + 4], r[8 * j + 5]),
                         pack_bf16(r[8 * j + 6], r[8 * j + 7]));
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmY, buf, col, t.row0 + wrow0);
            bulk_commit_group();
          }
          ++n_chunk;
        } else if (valid) {
          store_chunk(a, yrow_ptr, col, col_end, r);
        }
      };
      if (sk) {
        // Split-K part of a tile (rows <= kSKRows: lane quarter 0 holds them).  1. the partial accumulator
        // goes to the unit's slot and TMEM is freed; 2. the epilogue warps meet, one thread counts this
        // part's arrival at the tile; 3. the CTA finishing the last part sums the S parts in K order.
        const int slot = acc;
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + slot * kAccCols;
        const int wslot = (int)unit;
        const int n0 = t.ct * t.bn;
        const int col_end = min(n0 + t.bn, a.N);
        if (q == 0) {
          float* wrow = a.sk_ws + ((size_t)wslot * moe::kSKRows + lane) * moe::kSKCols;
          for (int c = 32 * cg; c < t.bn; c += 32 * kEpiGroups) {
            uint32_t r[32];
            tmem_ld32(taddr + c, r);
            tmem_wait_ld();
            if (valid) {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                *reinterpret_cast<uint4*>(wrow + c + 4 * i) = make_uint4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty_bar(slot));
        // Release / acquire through one thread (the CTA barrier orders the other warps' partial stores
        // before its fence; a fence per thread costs an L1 invalidate each, measured 25 % of dec1's time).
        // The partials of other CTAs are then read with ld.global.cg (L2, never a stale L1 line).
        __shared__ int s_sk_last;
        named_bar_sync(1, 32 * kEpiWarps);
        if (ew == 0 && lane == 0) {
          __threadfence();
          s_sk_last = atomicAdd(a.sk_cnt + v, 1) == sk_s - 1;
          if (s_sk_last) __threadfence();
        }
        named_bar_sync(1, 32 * kEpiWarps);
        if (s_sk_last) {
          if (q == 0 && valid) {
            for (int c = 32 * cg; c < t.bn; c += 32 * kEpiGroups) {
              uint32_t r[32];                         // the fp32 sum, as store_chunk takes it
#pragma unroll
              for (int i = 0; i < 32; ++i) r[i] = 0u;
              for (int pp = 0; pp < sk_s; ++pp) {
                const int ws2 = pp * total + v;
                const float4* src =
                    reinterpret_cast<const float4*>(a.sk_ws + ((size_t)ws2 * moe::kSKRows + lane) * moe::kSKCols + c);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const float4 f = __ldcg(src + i);
                  r[4 * i] = __float_as_uint(__uint_as_float(r[4 * i]) + f.x);
                  r[4 * i + 1] = __float_as_uint(__uint_as_float(r[4 * i + 1]) + f.y);
                  r[4 * i + 2] = __float_as_uint(__uint_as_float(r[4 * i + 2]) + f.z);
                  r[4 * i + 3] = __float_as_uint(__uint_as_float(r[4 * i + 3]) + f.w);
                }
              }
              if constexpr (kFp8) {
                if (a.scale) {
                  const float sc = __ldg(a.scale + t.expert);
#pragma unroll
                  for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * sc);
                }
              }
              store_chunk(a, yrow_ptr, n0 + c, col_end, r);
            }
          }
          if (ew == 0 && lane == 0) a.sk_cnt[v] = 0;   // for the next launch on this plan
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
        continue;
      }
      if constexpr (kGated) {
        // Block b: gate in TMEM columns [0,128), up in [128,256) of outputs n0 + 128b + [0,128).
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
          wait_block1(hf);
          const int n0 = t.ct * t.bn + hf * 128;
          const int col_end = min(n0 + 128, a.N);
          const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + hf * kAccCols;
          for (int c = 32 * cg; c < 128 && (!tma_rows || n0 + c < a.N); c += 32 * kEpiGroups) {
            uint32_t g[32], u[32];
            tmem_ld32(ta + c, g);
            tmem_ld32(ta + 128 + c, u);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              // silu(g) = g * sigmoid(g) = 0.5 g (1 + tanh(g / 2)): one SFU op (tanh.approx, relative
              // error ~2^-11, below the bf16 rounding of h that follows) and two FMAs.
              const float hg = 0.5f * __uint_as_float(g[i]);
              g[i] = __float_as_uint(fmaf(hg, tanh_approx(hg), hg) * __uint_as_float(u[i]));
            }
            put_chunk(g, n0 + c, col_end);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(leader(tempty_bar(hf)));
        }
      } else {
        const int bnp = t.bn / kHalves;             // columns of one accumulator block
        const bool ride = kSplit && t.kind == 3;
        const bool one = kCta == 2 && !ride && one_box<kWide, kGated>(t.bn, t.ct, a.N, a.w4d, false);
#pragma unroll 1
        for (int hf = 0; hf < kHalves; ++hf) {
          wait_block1(hf);
          if (kSplit && ride && hf == 1) {
            // Ride tile, the tail (TMEM block 1, swap-AB): lane = output column (this CTA's 128 of the half's
            // 256: t.ct * bn + 256 hh + 128 rank + lane), TMEM column = tail token; as on kind-1 tiles, each
            // warp stores, token by token, 32 consecutive columns of the token's Y row.
            const int esz = a.y_f32 ? 4 : 2;
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + kAccCols;
            const int col = t.ct * t.bn + t.hh * bnp + (int)rank * (bnp / kCta) + q * 32 + lane;
            const bool col_ok = col < a.N;
            for (int c = 32 * cg; c < t.height; c += 32 * kEpiGroups) {
              uint32_t r[32];
              tmem_ld32(taddr + c, r);
              const int tk = min(c + lane, t.trows - 1);
              uint8_t* rp = a.y_row_ptr ? reinterpret_cast<uint8_t*>(__ldg(a.y_row_ptr + t.trow0 + tk))
                                        : reinterpret_cast<uint8_t*>(a.Y) +
                                              (a.y_row_map ? (int64_t)__ldg(a.y_row_map + t.trow0 + tk)
                                                           : (int64_t)t.trow0 + tk) * a.N * esz;
              tmem_wait_ld();
              const int ntok = min(32, t.trows - c);
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                uint8_t* row = reinterpret_cast<uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(rp), j));
                if (j < ntok && col_ok) {
                  if (a.y_f32)
                    reinterpret_cast<float*>(row)[col] = __uint_as_float(r[j]);
                  else
                    reinterpret_cast<__nv_bfloat16*>(row)[col] = __float2bfloat16_rn(__uint_as_float(r[j]));
                }
              }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(leader(tempty_bar(1)));
            continue;
          }
          // columns of this warp's lanes: the whole block, or (half tile) its first / second half
          const int hw = hlf ? wide_block_cols<kFp8>(t.bn, t.ct, a.N, hf) / 2 : bnp;
          const int n0 = t.ct * t.bn + (ride ? t.hh : hf) * bnp + (hlf ? (q >> 1) * hw : 0);
          const int slot = kWide ? hf : acc;        // TMEM block and its tmem-empty barrier
          const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + slot * kAccCols;
          for (int c = 32 * cg; c < hw && (!tma_rows || n0 + c < a.N); c += 32 * kEpiGroups) {
            // W column of TMEM column c (one box per CTA: the D half picks the CTA's 256 columns)
            const int col = one ? w_col(true, t.ct, t.bn, hf, hlf ? (q >> 1) : (c >> 7), hlf ? c : (c & 127)) : n0 + c;
            const int col_end = one ? col + 32 : min(n0 + hw, a.N);
            uint32_t r[32];
            tmem_ld32(taddr + c, r);
            tmem_wait_ld();
            if constexpr (kFp8) {
              if (a.scale) {
                const float sc = __ldg(a.scale + t.expert);
#pragma unroll
                for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * sc);
              }
            }
            put_chunk(r, col, col_end);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (kCta == 2) mbar_arrive_cluster(leader(tempty_bar(slot)));
            else mbar_arrive(tempty_bar(slot));
          }
        }
      }
      if constexpr (kProf) c_work += clock64() - w0;
      if constexpr (kWide) {
        acc_phase ^= 1u;
      } else if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
    while (gemv_round()) {
    }                                                         // the GEMV units left after the last tile
    if (ew == 0 && lane == 0) MOE_TL(5);                      // epilogue done, stores in flight
    if (lane == 0) bulk_wait_group<0>();                      // TMA stores complete before exit
    if (ew == 0 && lane == 0) MOE_TL(6);
    if constexpr (kProf) {
      if (q == 0 && lane == 0) {
        a.prof[blockIdx.x * kProfSlots + kProfEpiWaitFull] = c_wait;
        a.prof[blockIdx.x * kProfSlots + kProfEpiWork] = c_work;
      }
    }
  }

  tc_fence_before();
  if constexpr (kCta == 2) cluster_sync(); else __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<kTmemCols, kCta>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// Decode-regime tiles (bm = 64: every expert has <= 64 rows; SURVEY §8's skinny batches).
// The GEMM is HBM-bound on W, so the tile is swap-AB on one CTA: the W block (256 columns,
// two M = 128 blocks, MN-major) is the MMA's M operand and the tile's <= 64 token rows its N
// operand (N = rows rounded up to 16).  A stage is 32 KB of W + 8 KB of tokens, so five stages
// keep 160 KB of W in flight per SM (the 128 x 256 tile: 4 x 32 KB behind 16 KB token stages).
// TMEM lane = output column, TMEM column = token: the epilogue stores each token row's 32
// columns per warp with one coalesced 64 / 128-byte store, no transpose.  DESIGN.md §6.4.
// ---------------------------------------------------------------------------
constexpr int kDecRows = 64;                       // tokens per tile (the plan's bm)
constexpr int kDecCols = 256;                      // W columns per tile (the plan's bn)
constexpr int kDecSt = 5;
constexpr int kDecTokBytes = kDecRows * kBK * 2;   // 8 KB
constexpr int kDecWBytes = kDecCols * kBK * 2;     // 32 KB
constexpr int kDecAccCols = 128;                   // per accumulator: 2 blocks x 64 token columns
constexpr size_t kDecSmem = 1024 + (size_t)kDecSt * (kDecTokBytes + kDecWBytes) + kBarBytes;
static_assert(8 * (2 * kDecSt + 4) + 4 <= 256, "decode barrier block overlaps its timestamps");

__global__ void __launch_bounds__(kThreads, 1)
    moe_gemm_decode_kernel(const __grid_constant__ CUtensorMap tmW, const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  const uint32_t sTok = base;
  const uint32_t sW = sTok + kDecSt * kDecTokBytes;
  const uint32_t sBar = sW + kDecSt * kDecWBytes;
  auto full_bar = [&](int s) { return sBar + 8u * s; };
  auto empty_bar = [&](int s) { return sBar + 8u * (kDecSt + s); };
  auto tfull_bar = [&](int i) { return sBar + 8u * (2 * kDecSt + i); };
  auto tempty_bar = [&](int i) { return sBar + 8u * (2 * kDecSt + 2 + i); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + (sBar - base) + 8 * (2 * kDecSt + 4));
  int32_t* s_prefix = reinterpret_cast<int32_t*>(smem + (sBar - base) + kBarBytes);
  int32_t* s_sigma = s_prefix + a.M_pad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int total = a.total;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDecSt; ++s) {
      mbar_init(full_bar(s), 32 * kAWarps + 1);    // token copies (one arrive per A thread) + W bytes
      mbar_init(empty_bar(s), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull_bar(i), 1);
      mbar_init(tempty_bar(i), kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) prefetch_tmap(&tmW);
  if (warp == kMmaWarp) tmem_alloc<256, 1>(smem_u32(tmem_holder));
  pdl_wait();
  for (int i = threadIdx.x; i < 2 * a.M_pad; i += blockDim.x) s_prefix[i] = a.plan[MOE_PLAN_HEADER + i];
  if (total < 0) total = __ldg(a.plan + 2);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int32_t* params = a.plan + a.off_params;

  if (warp < kAWarps) {
    // ===== token rows: 64 per tile, cp.async 16 B per thread, 8 threads per 128-byte row =====
    const int ch = threadIdx.x & 7, rsub = threadIdx.x >> 3;    // rsub in [0, 16)
    const uint32_t dst_off = rsub * 128 + ((ch ^ (rsub & 7)) << 4);
    uint32_t g = 0;
    for (int v = blockIdx.x; v < total; v += gridDim.x) {
      int h, task, l;
      map_tile(s_prefix, s_sigma, a.M_pad, v, h, task, l);
      const Tile t = load_tile(params, task, l);
      const int rbeg = t.rt * kDecRows;
      const int nvalid = min(kDecRows, t.rows - rbeg);
      const __nv_bfloat16* src[4];
      uint32_t rowok = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = rsub + 16 * j;
        const int tok = r < nvalid ? (a.token_idx ? __ldg(a.token_idx + t.row0 + rbeg + r) : t.row0 + rbeg + r) : 0;
        src[j] = a.X + (int64_t)tok * a.H + ch * 8;
        rowok |= (r < nvalid ? 1u : 0u) << j;
      }
      for (int kb = 0; kb < a.num_kb; ++kb, ++g) {
        const int s = g % kDecSt;
        mbar_wait(empty_bar(s), ((g / kDecSt) & 1u) ^ 1u);
        const int kcol = kb * kBK;
        const bool colok = kcol + ch * 8 < a.H;
        const uint32_t dst = sTok + s * kDecTokBytes + dst_off;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const bool ok = colok && ((rowok >> j) & 1u);
          cp_async_16(dst + j * 16 * 128, ok ? src[j] + kcol : a.X, ok ? 16u : 0u);
        }
        cp_async_mbar_arrive_noinc(full_bar(s));
      }
    }
  } else if (warp == kBWarp) {
    // ===== the W block: 256 columns x 64 K per stage, one 4-D TMA (or 4 3-D boxes) =====
    const uint64_t pol_w = policy_evict_normal();
    uint32_t g = 0;
    for (int v = blockIdx.x; v < total; v += gridDim.x) {
      int h, task, l;
      map_tile(s_prefix, s_sigma, a.M_pad, v, h, task, l);
      const Tile t = load_tile(params, task, l);
      const int n0 = t.ct * kDecCols;
      for (int kb = 0; kb < a.num_kb; ++kb, ++g) {
        const int s = g % kDecSt;
        mbar_wait(empty_bar(s), ((g / kDecSt) & 1u) ^ 1u);
        if (lane == 0) {
          const uint32_t dst = sW + s * kDecWBytes;
          mbar_arrive_expect_tx(full_bar(s), kDecWBytes);
          if (a.w4d) {
            tma_load_4d(&tmW, full_bar(s), dst, 0, kb * kBK, n0 >> 6, t.expert, pol_w);
          } else {
            for (int j = 0; j < kDecCols / 64; ++j)
              tma_load_3d(&tmW, full_bar(s), dst + j * kBBoxBytes, n0 + j * 64, kb * kBK, t.expert, pol_w);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    // ===== swap-AB MMAs: D[col, token] += W_block[k, col]^T tokens[token, k], two M = 128 blocks =====
    uint32_t g = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int v = blockIdx.x; v < total; v += gridDim.x) {
      int h, task, l;
      map_tile(s_prefix, s_sigma, a.M_pad, v, h, task, l);
      const Tile t = load_tile(params, task, l);
      const int ntok = (min(kDecRows, t.rows - t.rt * kDecRows) + 15) & ~15;
      const uint32_t idesc = idesc_bf16_f32(128, ntok, /*A MN-major*/ 1, /*B K-major*/ 0);
      mbar_wait(tempty_bar(acc), acc_phase ^ 1u);
      tc_fence_after();
      for (int kb = 0; kb < a.num_kb; ++kb, ++g) {
        const int s = g % kDecSt;
        mbar_wait(full_bar(s), (g / kDecSt) & 1u);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t w0 = sW + s * kDecWBytes, t0 = sTok + s * kDecTokBytes;
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              mma_bf16(tmem_base + acc * kDecAccCols + hf * 64,
                       smem_desc_sw128(w0 + hf * 2 * kBBoxBytes + kk * 2048, kBBoxBytes, 1024),
                       smem_desc_sw128(t0 + kk * 32, 16, 1024), idesc, (kb | kk) != 0);
          mma_commit(empty_bar(s));
        }
        __syncwarp();
      }
      if (lane == 0) mma_commit(tfull_bar(acc));
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  } else {
    // ===== epilogue: warp -> (block cg, TMEM lane quarter q): 32 output columns, every token =====
    const int q = warp & 3;
    const int cg = (warp - (kMmaWarp + 1)) >> 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int v = blockIdx.x; v < total; v += gridDim.x) {
      int h, task, l;
      map_tile(s_prefix, s_sigma, a.M_pad, v, h, task, l);
      const Tile t = load_tile(params, task, l);
      const int rbeg = t.rt * kDecRows;
      const int nvalid = min(kDecRows, t.rows - rbeg);
      const int col = t.ct * kDecCols + cg * 128 + q * 32 + lane;
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * kDecAccCols + cg * 64;
      for (int c = 0; c < nvalid; c += 32) {
        uint32_t r[32];
        tmem_ld32(taddr + c, r);
        tmem_wait_ld();
        if (col < a.N) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (c + j < nvalid) {
              const int csr = t.row0 + rbeg + c + j;
              const int64_t yr = a.y_row_map ? (int64_t)__ldg(a.y_row_map + csr) : (int64_t)csr;
              if (a.y_f32)
                reinterpret_cast<float*>(a.Y)[yr * a.N + col] = __uint_as_float(r[j]);
              else
                reinterpret_cast<__nv_bfloat16*>(a.Y)[yr * a.N + col] = __float2bfloat16_rn(__uint_as_float(r[j]));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty_bar(acc));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<256, 1>(tmem_base);
  }
}

// Decode every virtual tile with the same device function as the GEMM.
__global__ void decode_debug_kernel(const int32_t* plan, int total, int M_pad, int off_params, int32_t* out) {
  extern __shared__ int32_t s_pre[];
  for (int i = threadIdx.x; i < 2 * M_pad; i += blockDim.x) s_pre[i] = plan[MOE_PLAN_HEADER + i];
  __syncthreads();
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < total; v += warps) {
    int h, task, l;
    map_tile(s_pre, s_pre + M_pad, M_pad, v, h, task, l);
    const Tile t = load_tile(plan + off_params, task, l);
    if ((threadIdx.x & 31) == 0) {
      int32_t* o = out + 5 * (int64_t)v;
      o[0] = h;
      o[1] = task;
      o[2] = l;
      o[3] = t.rt;
      o[4] = t.ct;
    }
  }
}

// Probe: one CTA gathers 128 rows x 64 columns with tile::gather4 into a SW128
// buffer and dumps the raw 16 KB of shared memory.
__global__ void probe_gather4_kernel(const __grid_constant__ CUtensorMap tmX, const int32_t* rows, int col0,
                                     uint8_t* out) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  const uint32_t bar = base + kABytes;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (lane == 0) mbar_arrive_expect_tx(bar, kABytes);
    __syncwarp();
    tma_gather4(&tmX, bar, base + lane * 512, col0, rows[4 * lane], rows[4 * lane + 1], rows[4 * lane + 2],
                rows[4 * lane + 3], policy_evict_normal());
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < kABytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(out)[i] = reinterpret_cast<const uint4*>(smem)[i];
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// fp8: X holds FP8 E4M3 bytes (a box is 128 values = 128 bytes, like 64 bf16).
moe_status make_x_map(CUtensorMap* m, const void* X, int64_t T, int64_t H, int box_rows = 1, bool fp8 = false) {
  auto fn = encode_fn();
  if (!fn) MOE_FAIL(MOE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  const cuuint64_t dims[2] = {(cuuint64_t)H, (cuuint64_t)T};
  const cuuint64_t strides[1] = {(cuuint64_t)H * (fp8 ? 1 : 2)};
  const cuuint32_t box[2] = {(cuuint32_t)(fp8 ? 128 : kBK), (cuuint32_t)box_rows};   // gather4: box_rows = 1
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(X), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) MOE_FAIL(MOE_ERR_CUDA, "cuTensorMapEncodeTiled(X) failed: %d", (int)r);
  return MOE_OK;
}

// Y viewed as {N, R} bf16 rows; box 32 x 32 with the 64-byte swizzle (the epilogue's staging layout).
moe_status make_y_map(CUtensorMap* m, void* Y, int64_t R, int64_t N) {
  auto fn = encode_fn();
  if (!fn) MOE_FAIL(MOE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)R};
  const cuuint64_t strides[1] = {(cuuint64_t)N * 2};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Y, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) MOE_FAIL(MOE_ERR_CUDA, "cuTensorMapEncodeTiled(Y) failed: %d", (int)r);
  return MOE_OK;
}

// bn_cta: W columns one CTA stages per K block (the 4-D box spans ceil(bn_cta / 64) chunks).
// fp8: W holds FP8 E4M3 bytes; chunks of 128 columns (128 bytes), K blocks of 128 rows (4-D only).
moe_status make_w_map(CUtensorMap* m, const void* W, int64_t E, int64_t H, int64_t N, int bn_cta, bool w4d,
                      bool fp8 = false) {
  auto fn = encode_fn();
  if (!fn) MOE_FAIL(MOE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  CUresult r;
  if (fp8) {
    if (!w4d) MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_gemm_fp8: needs N %% 128 == 0 and 128-column CTA blocks");
    const cuuint64_t dims[4] = {128, (cuuint64_t)H, (cuuint64_t)(N / 128), (cuuint64_t)E};
    const cuuint64_t strides[3] = {(cuuint64_t)N, 128, (cuuint64_t)H * N};
    const cuuint32_t box[4] = {128, 128, (cuuint32_t)((bn_cta + 127) / 128), 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(W), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (w4d) {
    // W viewed as {64 (n within chunk), H, N/64 (chunk), E}: one box = the whole B stage,
    // laid out chunk-major, then k, then n — the MN-major SW128 canonical layout.
    const cuuint64_t dims[4] = {64, (cuuint64_t)H, (cuuint64_t)(N / 64), (cuuint64_t)E};
    const cuuint64_t strides[3] = {(cuuint64_t)N * 2, 128, (cuuint64_t)H * N * 2};
    const cuuint32_t box[4] = {64, (cuuint32_t)kBK, (cuuint32_t)((bn_cta + 63) / 64), 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(W), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)H, (cuuint64_t)E};
    const cuuint64_t strides[2] = {(cuuint64_t)N * 2, (cuuint64_t)H * N * 2};
    const cuuint32_t box[3] = {64, (cuuint32_t)kBK, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(W), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) MOE_FAIL(MOE_ERR_CUDA, "cuTensorMapEncodeTiled(W) failed: %d", (int)r);
  return MOE_OK;
}

constexpr int kMaxDevices = 64;

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 || dev >= kMaxDevices ? 0 : dev;
}

// SM count of the current device (cached per device: a process may drive several GPUs).
int sm_count_cached() {
  static int n[kMaxDevices] = {};
  static std::once_flag once[kMaxDevices];
  const int dev = current_device();
  std::call_once(once[dev], [dev] { cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev); });
  return n[dev];
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

#if MOE_TIMELINE
extern "C" int moe_debug_timeline(unsigned long long* out, int n) {   // study builds only
  return (int)cudaMemcpyFromSymbol(out, g_moe_tl, sizeof(unsigned long long) * (size_t)n);
}
#endif

extern "C" moe_status moe_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
  moe::clear_error();
  int dev = 0, maj = 0, min = 0, n = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (sm_count) *sm_count = n;
  if (cc_major) *cc_major = maj;
  if (cc_minor) *cc_minor = min;
  if (maj != 10 || min != 0) MOE_FAIL(MOE_ERR_UNSUPPORTED, "device is sm_%d%d; this library is built for sm_100a", maj, min);
  return MOE_OK;
}

namespace {

constexpr size_t kMaxSmem = 232448;              // 227 KB of opt-in dynamic shared memory per CTA (sm_100)

template <bool kProf, int kCta, bool kSplit, bool kWide = false, bool kGated = false, bool kFp8 = false>
cudaError_t set_attr() {
  const size_t want = Geo<kCta, kSplit, kWide>::kSmem + 8 * kMaxMPad;
  return cudaFuncSetAttribute(moe_gemm_kernel<kProf, kCta, kSplit, kWide, kGated, kFp8>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(want < kMaxSmem ? want : kMaxSmem));
}

// Function attributes are per device: set once for each device the process launches on.
cudaError_t set_smem_attrs() {
  static std::once_flag once[kMaxDevices];
  static cudaError_t errs[kMaxDevices] = {};
  const int dev = current_device();
  cudaError_t& err = errs[dev];
  std::call_once(once[dev], [&err] {
    cudaError_t e[16] = {set_attr<false, 1, false>(),      set_attr<true, 1, false>(),
                        set_attr<false, 1, false, false, false, true>(), set_attr<false, 2, false, false, false, true>(),
                        set_attr<false, 2, false, true, false, true>(), set_attr<true, 2, false, true, false, true>(),
                        set_attr<false, 2, false>(),      set_attr<true, 2, false>(),
                        set_attr<false, 2, true>(),       set_attr<true, 2, true>(),
                        set_attr<false, 2, false, true>(), set_attr<true, 2, false, true>(),
                        set_attr<false, 2, false, true, true>(), set_attr<true, 2, false, true, true>(),
                        set_attr<false, 2, true, true>(), set_attr<true, 2, true, true>()};
    for (cudaError_t x : e)
      if (x != cudaSuccess && err == cudaSuccess) err = x;
    const cudaError_t d = cudaFuncSetAttribute(moe_gemm_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(kDecSmem + 8 * kMaxMPad));
    if (d != cudaSuccess && err == cudaSuccess) err = d;
  });
  return err;
}

}  // namespace
cudaError_t moe::preload_gemm_kernels() { return set_smem_attrs(); }
namespace {

static moe_status gemm_launch(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx,
                              const void* W, void* Y, int32_t y_dtype, void* stream, long long* prof,
                              const int32_t* y_row_map = nullptr, const void* W2 = nullptr, bool fp8 = false,
                              const float* scale = nullptr, const unsigned long long* y_row_ptr = nullptr) {
  moe::NvtxRange nvtx(W2 ? "moe_gemm_swiglu" : fp8 ? "moe_gemm_fp8" : "moe_gemm");
  moe::clear_error();
  if (!plan) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm: null plan");
  moe::BlobView v;
  const bool dev_planned = moe::plan_device_mode(plan);
  if (dev_planned) {
    // Counts live on the device (moe_plan_device): fixed-layout blob, tile count read in-kernel.
    int32_t E, H, N, bm, bn;
    uint32_t flags;
    moe::plan_shape(plan, &E, &H, &N, &bm, &bn, &flags);
    v.E = E; v.H = H; v.N = N; v.bm = bm; v.bn = bn; v.flags = flags; v.n_tasks = E;
    v.M_pad = E <= 32 ? 32 : (E + 31) / 32 * 32;
    v.M = -1;
    v.total = -1;
    v.off_prefix = MOE_PLAN_HEADER;
    v.off_sigma = v.off_prefix + v.M_pad;
    v.off_params = v.off_sigma + v.M_pad;
  }
  // MOE_KIND_GEMV tasks (no tiles; computed by the epilogue warps of wide kernels): a host
  // plan lists them in its task parameters, a device-planned one may have them when its catalog has the rule.
  bool has_gemv = false;
  {
    int64_t words = 0;
    const int32_t* blob = moe::plan_blob_host(plan, &words);
    if (dev_planned) {
      for (int i = 0; i < MOE_MAX_RULES; ++i) has_gemv |= blob[12 + 2 * i] == MOE_KIND_GEMV && blob[13 + 2 * i] > 0;
    } else {
      if (!moe::blob_view(blob, words, &v)) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm: corrupt plan");
      for (int i = 0; i < v.n_tasks; ++i) {
        const int32_t* p = blob + v.off_params + (int64_t)MOE_PLAN_TASK_WORDS * i;
        has_gemv |= p[3] == MOE_KIND_GEMV && p[2] > 0;
      }
      if (v.total == 0 && !has_gemv) return MOE_OK_EMPTY;
    }
  }
  if (!X || !W || !Y) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm: null tensor pointer");
  if (!aligned16(X) || !aligned16(W) || !aligned16(Y))
    MOE_FAIL(MOE_ERR_INVALID, "moe_gemm: X, W and Y must be 16-byte aligned");
  if (T < 1 || T >= INT_MAX) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm: T=%lld outside [1, 2^31)", (long long)T);
  if (y_dtype != MOE_DTYPE_BF16 && y_dtype != MOE_DTYPE_F32) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm: y_dtype=%d", y_dtype);
  if (v.M_pad > kMaxMPad) MOE_FAIL(MOE_ERR_CAPACITY, "moe_gemm: %d tasks exceed %d", v.M_pad, kMaxMPad);

  CUtensorMap tmX, tmW;
  int experiment = 0;
#ifdef MOE_EXPERIMENTS
  {
    const char* ex = getenv("MOE_GEMM_EXPERIMENT");
    experiment = ex ? atoi(ex) : 0;
  }
#endif
  // token_idx NULL: X rows are the plan's CSR rows (a_mode 2: 128-row tile boxes).
  if (fp8) {
    // FP8 E4M3 (moe_gemm_fp8): 1-CTA tiles (bn % 128 == 0) and CTA-pair / wide tiles whose CTA
    // blocks are 128 columns (bn = 256 or 512); TMA strides need 16-byte rows.
    if (W2) MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_gemm_fp8: no gated variant");
    if (prof && !(v.bm == 256 && v.bn > 256))
      MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_gemm_fp8_profile: instrumented for wide pair tiles only");
    // (The FP8 kernel runs every tile as MOE_KIND_WIDE: a plan's swap-AB catalog rules are ignored,
    // which changes nothing in Y — the tile partition is the same.)
    if (v.bm == kDecRows) MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_gemm_fp8: bm = 64 decode tiles are bf16-only");
    const bool ok_tile = v.bm == 128 ? v.bn % 128 == 0 : (v.bn == 256 || v.bn == 512);
    if (!ok_tile || v.N % 128 || v.H % 16)
      MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_gemm_fp8: needs N %% 128 == 0, H %% 16 == 0 and a %d x %d tile of "
               "128-column CTA blocks (1-CTA bn %% 128 == 0, pair bn = 256 or 512)", v.bm, v.bn);
  }
  moe_status st = make_x_map(&tmX, X, T, v.H, (experiment & 4) || !token_idx ? kBM : 1, fp8);
  if (st != MOE_OK) return st;
  const bool gated = W2 != nullptr;                // moe_gemm_swiglu: W_gate / W_up blocks
  if (gated && !(v.bm == 256 && v.bn == 256))
    MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_gemm_swiglu: the plan must have bm = 256, bn = 256 (got %d x %d)", v.bm, v.bn);
  if (gated && !aligned16(W2)) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm_swiglu: W_up must be 16-byte aligned");
  const bool wide = v.bm == 256 && v.bn > 256;    // wide pair tile: two N = bn/2 MMA blocks
  const int cta = v.bm == 256 ? 2 : 1;             // CTAs per tile: each stages bn / cta W columns
  const int bnc_blk = v.bn / cta / (wide ? 2 : 1); // W columns one CTA stages per MMA block
  // 4-D W view (one TMA per block): needs every CTA's block start on a 64-column chunk.
  const bool w4d = fp8 ? (v.N % 128) == 0 && bnc_blk % 128 == 0 : (v.N % 64) == 0 && bnc_blk % 64 == 0;
  st = make_w_map(&tmW, W, v.E, v.H, v.N, bnc_blk, w4d, fp8);
  if (st != MOE_OK) return st;
  CUtensorMap tmW2 = tmW;
  if (gated) {
    st = make_w_map(&tmW2, W2, v.E, v.H, v.N, v.bn / cta, w4d);
    if (st != MOE_OK) return st;
  } else if (wide && w4d && v.bn == 512) {
    // one box per CTA per stage for wide tiles inside N and swap-AB tiles: both blocks' 256 columns
    st = make_w_map(&tmW2, W, v.E, v.H, v.N, 2 * bnc_blk, w4d, fp8);
    if (st != MOE_OK) return st;
  }

  // TMA-store epilogue: bf16 Y in CSR row order (the EP combine path scatters rows: register stores).
  CUtensorMap tmY;
  std::memset(&tmY, 0, sizeof(tmY));
  bool tma_store = y_dtype == MOE_DTYPE_BF16 && !y_row_map && !y_row_ptr;
  if (y_row_ptr && (v.bm == kDecRows || W2))
    MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_gemm_rowptr: plain / pair / wide tiles only (no bm = 64, no gating)");
  if (v.flags & MOE_EPI_REGISTER) tma_store = false;   // plan option: register stores only
  if (tma_store) {
    // Rows of Y: the plan's total (host plan); a device plan's count is on the device, so the
    // map spans 2^31-1 rows — every box the kernel stores lies inside one task's rows.
    int64_t R = INT_MAX;
    if (!dev_planned) {
      int64_t words = 0;
      const int32_t* blob = moe::plan_blob_host(plan, &words);
      R = blob[v.off_row_off + v.E];
    }
    st = make_y_map(&tmY, Y, R, v.N);
    if (st != MOE_OK) return st;
  }

  GemmArgs a;
  a.plan = moe::plan_blob_dev(plan);
  a.token_idx = token_idx;
  a.Y = Y;
  a.y_f32 = y_dtype == MOE_DTYPE_F32;
  a.N = v.N;
  a.num_kb = (int32_t)moe::ceil_div(v.H, fp8 ? 128 : kBK);
  a.scale = scale;
  a.total = v.total;
  a.M_pad = v.M_pad;
  a.off_params = (int32_t)v.off_params;
  a.w4d = w4d ? 1 : 0;
  a.prof = prof;
  a.y_row_map = y_row_map;
  a.y_row_ptr = y_row_ptr;
  // Tile order: dynamic by default for CTA-pair tiles (compute-bound tiles of unequal
  // cost: wide / half / swap-AB; measured +1-5 %), static with the balanced grid for one-CTA
  // (decode-regime, HBM-bound) tiles; plan options force either.
  const bool dynamic = (v.flags & MOE_SCHED_DYNAMIC) ||
                       (!(v.flags & (MOE_GRID_STATIC | MOE_GRID_BALANCED)) && v.bm == 256);
  a.sched = dynamic ? moe::plan_sched_dev(plan) : nullptr;
  a.light_merge = dynamic && (v.flags & MOE_ORDER_LIGHT_LAST) ? 1 : 0;
  a.half_last = dynamic && wide && !gated && !a.light_merge && (v.flags & MOE_SCHED_HALF_LAST) ? 1 : 0;
  a.narrow_last = dynamic && wide && !gated && !a.light_merge && !a.half_last && v.N % v.bn != 0 && v.N > v.bn &&
                          !(v.flags & MOE_SCHED_PLAN_ORDER)
                      ? (int)moe::ceil_div(v.N, v.bn)
                      : 0;
  a.gemv_q = has_gemv ? moe::plan_sched_dev(plan) + 2 : nullptr;
  if (has_gemv && !(wide && !gated))
    MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_gemm: MOE_KIND_GEMV tasks need a wide pair tile plan (bm 256, bn > 256)");
  a.W = reinterpret_cast<const uint8_t*>(W);
  a.pf_dist = (v.flags & MOE_L2_PREFETCH) && v.N % 64 == 0 ? kL2Pf : 0;
  a.balance = a.sched ? 0 : (v.flags & MOE_GRID_BALANCED) ? 1 : (v.flags & MOE_GRID_STATIC) ? 0 : v.bm == 128;
  // Stream-K (one-CTA tiles; the kernel decides per launch from the tile count and task heights): needs
  // the plan's workspace, static tile order and one CTA per SM.
  a.sk_ws = nullptr;
  a.sk_cnt = nullptr;
  int sk_ctas = 0;
  if (v.bm == 128 && !a.sched && (v.flags & MOE_SPLIT_K) && !(v.flags & MOE_GRID_STATIC) && !prof) {
    a.sk_ws = moe::plan_sk_ws(plan, &a.sk_cnt, &sk_ctas);
    if (sk_ctas != sm_count_cached()) a.sk_ws = nullptr;   // workspace sized for another device
  }
  a.tma_store = tma_store ? 1 : 0;
  a.T = (int32_t)T;
  a.H = v.H;
  a.X = reinterpret_cast<const __nv_bfloat16*>(X);
  a.experiment = experiment;
  // A staging: contiguous rows by tile TMA (token_idx NULL), TMA gather4 (plan option), else cp.async.
  a.a_mode = !token_idx ? 2 : (v.flags & MOE_A_GATHER4) ? 0 : kDefaultAMode;
  if (fp8 && a.a_mode == 0) a.a_mode = 1;        // FP8 rows are staged by cp.async (or tile TMA)

  if (v.bm == 256 && (v.bn / 2) % 16) MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_gemm: pair tiles need bn %% 32 == 0");
  cudaError_t attr_err = set_smem_attrs();
  if (attr_err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(attr_err));
  if (v.bm == kDecRows) {
    // Decode-regime tiles: swap-AB on one CTA (moe_gemm_decode_kernel).
    if (gated || v.bn != kDecCols)
      MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_gemm: bm = 64 tiles need bn = 256, no split tails, not gated");
    const int grid = v.total < 0 ? sm_count_cached() : std::min(v.total, sm_count_cached());
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kDecSmem + 8 * (size_t)v.M_pad;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t le = cudaLaunchKernelEx(&cfg, moe_gemm_decode_kernel, tmW, a);
    if (le != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_gemm decode launch: %s", cudaGetErrorString(le));
  } else if (v.bm == 256) {
    // Two strategies in the launch when the catalog has a swap-AB rule (bf16, not gated).
    const bool split = moe::plan_has_swap(plan) && !fp8 && !gated;
    // (GEMV tasks: every CTA's epilogue warps take GEMV units, so all SMs launch)
    const int pairs = v.total < 0 || has_gemv ? sm_count_cached() / 2 : std::min(v.total, sm_count_cached() / 2);
    const size_t smem = (split && wide   ? Geo<2, true, true>::kSmem
                         : split         ? Geo<2, true>::kSmem
                         : wide || gated ? Geo<2, false, true>::kSmem
                                         : Geo<2, false>::kSmem) +
                        8 * (size_t)v.M_pad;
    if (smem > kMaxSmem) MOE_FAIL(MOE_ERR_CAPACITY, "moe_gemm: %d tasks need %zu B of shared memory", v.M_pad, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL: overlap the prologue
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t le;
    if (fp8 && wide)
      le = prof ? cudaLaunchKernelEx(&cfg, moe_gemm_kernel<true, 2, false, true, false, true>, tmX, tmW, tmW2, tmY, a)
                : cudaLaunchKernelEx(&cfg, moe_gemm_kernel<false, 2, false, true, false, true>, tmX, tmW, tmW2, tmY, a);
    else if (fp8)
      le = cudaLaunchKernelEx(&cfg, moe_gemm_kernel<false, 2, false, false, false, true>, tmX, tmW, tmW2, tmY, a);
    else if (gated)
      le = prof ? cudaLaunchKernelEx(&cfg, moe_gemm_kernel<true, 2, false, true, true>, tmX, tmW, tmW2, tmY, a)
                : cudaLaunchKernelEx(&cfg, moe_gemm_kernel<false, 2, false, true, true>, tmX, tmW, tmW2, tmY, a);
    else if (wide && split)
      le = prof ? cudaLaunchKernelEx(&cfg, moe_gemm_kernel<true, 2, true, true>, tmX, tmW, tmW2, tmY, a)
                : cudaLaunchKernelEx(&cfg, moe_gemm_kernel<false, 2, true, true>, tmX, tmW, tmW2, tmY, a);
    else if (wide)
      le = prof ? cudaLaunchKernelEx(&cfg, moe_gemm_kernel<true, 2, false, true>, tmX, tmW, tmW2, tmY, a)
                : cudaLaunchKernelEx(&cfg, moe_gemm_kernel<false, 2, false, true>, tmX, tmW, tmW2, tmY, a);
    else if (split)
      le = prof ? cudaLaunchKernelEx(&cfg, moe_gemm_kernel<true, 2, true>, tmX, tmW, tmW2, tmY, a)
                : cudaLaunchKernelEx(&cfg, moe_gemm_kernel<false, 2, true>, tmX, tmW, tmW2, tmY, a);
    else
      le = prof ? cudaLaunchKernelEx(&cfg, moe_gemm_kernel<true, 2, false>, tmX, tmW, tmW2, tmY, a)
                : cudaLaunchKernelEx(&cfg, moe_gemm_kernel<false, 2, false>, tmX, tmW, tmW2, tmY, a);
    if (le != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_gemm pair launch: %s", cudaGetErrorString(le));
  } else {
    // one CTA per SM when the kernel may choose stream-K (it spreads the K blocks over every CTA)
    const int grid = v.total < 0 || a.sk_ws ? sm_count_cached() : std::min(v.total, sm_count_cached());
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Geo<1>::kSmem + 8 * (size_t)v.M_pad;
    if (cfg.dynamicSmemBytes > kMaxSmem)
      MOE_FAIL(MOE_ERR_CAPACITY, "moe_gemm: %d tasks need %zu B of shared memory", v.M_pad, cfg.dynamicSmemBytes);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t le = fp8    ? cudaLaunchKernelEx(&cfg, moe_gemm_kernel<false, 1, false, false, false, true>, tmX, tmW,
                                                 tmW2, tmY, a)
                     : prof ? cudaLaunchKernelEx(&cfg, moe_gemm_kernel<true, 1, false>, tmX, tmW, tmW2, tmY, a)
                            : cudaLaunchKernelEx(&cfg, moe_gemm_kernel<false, 1, false>, tmX, tmW, tmW2, tmY, a);
    if (le != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_gemm launch: %s", cudaGetErrorString(le));
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_gemm launch: %s", cudaGetErrorString(e));
  return MOE_OK;
}

}  // namespace

extern "C" {

moe_status moe_gemm(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx, const void* W,
                    void* Y, int32_t y_dtype, void* stream) {
  return gemm_launch(plan, X, T, token_idx, W, Y, y_dtype, stream, nullptr);
}

moe_status moe_gemm_swiglu(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx,
                           const void* W_gate, const void* W_up, void* Y, int32_t y_dtype, void* stream) {
  if (!W_up) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm_swiglu: null W_up");
  return gemm_launch(plan, X, T, token_idx, W_gate, Y, y_dtype, stream, nullptr, nullptr, W_up);
}

moe_status moe_gemm_fp8(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx, const void* W,
                        const float* scale, void* Y, int32_t y_dtype, void* stream) {
  return gemm_launch(plan, X, T, token_idx, W, Y, y_dtype, stream, nullptr, nullptr, nullptr, true, scale);
}

moe_status moe_gemm_fp8_rowmap(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx,
                               const void* W, const float* scale, void* Y, int32_t y_dtype, const int32_t* y_row_map,
                               void* stream) {
  if (!y_row_map) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm_fp8_rowmap: null y_row_map");
  return gemm_launch(plan, X, T, token_idx, W, Y, y_dtype, stream, nullptr, y_row_map, nullptr, true, scale);
}

moe_status moe_gemm_rowptr(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx, const void* W,
                           int32_t x_dtype, const float* scale, const unsigned long long* y_row_ptr, int32_t y_dtype,
                           void* stream) {
  if (!y_row_ptr) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm_rowptr: null y_row_ptr");
  if (x_dtype != MOE_DTYPE_BF16 && x_dtype != MOE_DTYPE_E4M3) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm_rowptr: x_dtype");
  // Y is unused (every row has its own address); a non-null placeholder passes the argument checks.
  return gemm_launch(plan, X, T, token_idx, W, const_cast<unsigned long long*>(y_row_ptr), y_dtype, stream, nullptr,
                     nullptr, nullptr, x_dtype == MOE_DTYPE_E4M3, scale, y_row_ptr);
}

moe_status moe_gemm_rowmap(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx,
                           const void* W, void* Y, int32_t y_dtype, const int32_t* y_row_map, void* stream) {
  if (!y_row_map) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm_rowmap: null y_row_map");
  return gemm_launch(plan, X, T, token_idx, W, Y, y_dtype, stream, nullptr, y_row_map);
}

moe_status moe_gemm_profile(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx,
                            const void* W, void* Y, int32_t y_dtype, long long* prof_dev, void* stream) {
  if (!prof_dev) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm_profile: null prof_dev");
  return gemm_launch(plan, X, T, token_idx, W, Y, y_dtype, stream, prof_dev);
}

moe_status moe_gemm_fp8_profile(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx,
                                const void* W, const float* scale, void* Y, int32_t y_dtype, long long* prof_dev,
                                void* stream) {
  if (!prof_dev) MOE_FAIL(MOE_ERR_INVALID, "moe_gemm_fp8_profile: null prof_dev");
  return gemm_launch(plan, X, T, token_idx, W, Y, y_dtype, stream, prof_dev, nullptr, nullptr, true, scale);
}

moe_status moe_decode_debug(const moe_plan* plan, int32_t* out, void* stream) {
  moe::clear_error();
  if (!plan || !out) MOE_FAIL(MOE_ERR_INVALID, "moe_decode_debug: null argument");
  if (moe::plan_device_mode(plan)) MOE_FAIL(MOE_ERR_INVALID, "moe_decode_debug: device-resident plan (call moe_plan_sync)");
  int64_t words = 0;
  const int32_t* blob = moe::plan_blob_host(plan, &words);
  moe::BlobView v;
  if (!moe::blob_view(blob, words, &v)) MOE_FAIL(MOE_ERR_INVALID, "moe_decode_debug: corrupt plan");
  if (v.total == 0) return MOE_OK_EMPTY;
  const int threads = 256;
  const int grid = (int)std::min<int64_t>(moe::ceil_div(v.total, threads / 32), 4 * 148);
  decode_debug_kernel<<<grid, threads, 8 * v.M_pad, (cudaStream_t)stream>>>(moe::plan_blob_dev(plan), v.total,
                                                                          v.M_pad, (int)v.off_params, out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_decode_debug launch: %s", cudaGetErrorString(e));
  return MOE_OK;
}

moe_status moe_probe_gather4(const void* X, int64_t T, int64_t H, const int32_t* rows_dev, int32_t col0,
                             void* out_dev, void* stream) {
  moe::clear_error();
  if (!X || !rows_dev || !out_dev) MOE_FAIL(MOE_ERR_INVALID, "moe_probe_gather4: null argument");
  if (H % 8) MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_probe_gather4: H %% 8 != 0");
  CUtensorMap tmX;
  moe_status st = make_x_map(&tmX, X, T, H);
  if (st != MOE_OK) return st;
  const int smem = kABytes + 1024 + 64;
  probe_gather4_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(tmX, rows_dev, col0, (uint8_t*)out_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_probe_gather4 launch: %s", cudaGetErrorString(e));
  return MOE_OK;
}

}  // extern "C"
