// Host planner: expert token counts + tile shape -> the compressed mapping.
//
// Paper passages (P:n = line of PAPER.md):
//   Alg. 1  TilePrefix[i] = sum_{j<=i} nu(T_j)
//   P:203               pad TilePrefix to the warp size (INT32_MAX or repeat-last)
//   P:262-271, Alg. 4   TilePrefix only over the M non-empty tasks; sigma: [M] -> [N]
//   P:298-301           each expert is a task; p_i holds the expert's parameters
// The blob layout is documented in include/moe_sm100.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "common.h"

namespace moe {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

void clear_error() { g_last_error.clear(); }

static int32_t pad32(int64_t m) { return (int32_t)(m <= 32 ? 32 : ceil_div(m, 32) * 32); }

bool blob_view(const int32_t* blob, int64_t len, BlobView* v) {
  if (!blob || len < MOE_PLAN_HEADER || blob[0] != MOE_PLAN_MAGIC) return false;
  v->M = blob[1];
  v->total = blob[2];
  v->M_pad = blob[3];
  v->E = blob[4];
  v->N = blob[5];
  v->H = blob[6];
  v->bm = blob[7];
  v->bn = blob[8];
  v->n_tasks = blob[9];
  v->flags = (uint32_t)blob[10];
  v->off_prefix = MOE_PLAN_HEADER;
  v->off_sigma = v->off_prefix + v->M_pad;
  v->off_params = v->off_sigma + v->M_pad;
  v->off_row_off = v->off_params + (int64_t)MOE_PLAN_TASK_WORDS * v->n_tasks;
  v->words = v->off_row_off + v->E + 1;
  return v->words <= len;
}

}  // namespace moe

using moe::ceil_div;

extern "C" {

int64_t moe_plan_blob_words(int32_t E) {
  if (E < 1) return 0;
  const int64_t m_pad = moe::pad32(E);
  return MOE_PLAN_HEADER + 2 * m_pad + (int64_t)MOE_PLAN_TASK_WORDS * E + E + 1;
}

moe_status moe_plan_build(const int32_t* counts, int32_t E, int64_t H, int64_t N, int32_t bm,
                          int32_t bn, uint32_t flags, int32_t* blob, int64_t blob_cap,
                          int64_t* blob_len) {
  return moe_plan_build_catalog(counts, E, H, N, bm, bn, flags, nullptr, -1, blob, blob_cap, blob_len);
}

moe_status moe_plan_build_catalog(const int32_t* counts, int32_t E, int64_t H, int64_t N, int32_t bm, int32_t bn,
                                  uint32_t flags, const moe_tile_rule* rules, int32_t n_rules, int32_t* blob,
                                  int64_t blob_cap, int64_t* blob_len) {
  moe::clear_error();
  if (!counts || !blob) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_build: null counts or blob");
  if (E < 1 || E > 4096) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_build: E=%d outside [1, 4096]", E);
  if (H <= 0 || N <= 0) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_build: H=%lld N=%lld must be > 0", (long long)H, (long long)N);
  if (H % 8 || N % 8)
    MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_plan_build: H=%lld and N=%lld must be multiples of 8 (16-byte TMA strides)",
             (long long)H, (long long)N);
  if (H >= INT_MAX || N >= INT_MAX) MOE_FAIL(MOE_ERR_CAPACITY, "moe_plan_build: H or N >= 2^31");
  const bool auto_bn = bn == 0;
  if (auto_bn) bn = 256;
  if (bm == 0) {
    // Auto: executed rows under each tile height, CTA-pair tiles credited with
    // their measured ~1.10x per-row advantage (half the W traffic per SM, 6-stage ring).
    int64_t r128 = 0, r256 = 0;
    for (int32_t e = 0; e < E; ++e) {
      const int64_t m = counts[e] < 0 ? 0 : counts[e];
      r128 += ceil_div(m, 128) * 128;
      r256 += ceil_div(m, 256) * 256;
    }
    bm = bn > 256 || (r256 * 100 <= r128 * 110 && bn % 32 == 0) ? 256 : 128;
    // (bm = 64, the decode swap-AB tile, is opt-in: measured no faster than 128 x 256; §6.4.)
  }
  // Auto width: CTA-pair tiles go wide (256 x 512) whenever N has 512 columns.
  // (A last column tile past N trims its MMAs to the valid columns; narrower wide tiles such as
  // 3 x 480 for N = 1408 measured slower — their W boxes start off the 64-column chunk grid.)
  if (auto_bn && bm == 256 && N >= 512) bn = 512;
  if (bm != 64 && bm != 128 && bm != 256)
    MOE_FAIL(MOE_ERR_UNSUPPORTED,
             "moe_plan_build: bm=%d unsupported (64: decode swap-AB tile, 128: one CTA, 256: CTA pair, 0: auto)", bm);
  if (bm == 64 && (bn != 256 || (flags & MOE_SPLIT_TAIL)))
    MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_plan_build: bm=64 (decode tiles) needs bn=256 and no MOE_SPLIT_TAIL");
  // bm = 256, 256 < bn <= 512: wide pair tile (two N = bn/2 MMA blocks sharing the staged token rows).
  const bool wide_tile = bm == 256 && bn > 256 && bn <= 512 && bn % 32 == 0;
  if (!wide_tile && (bn < 16 || bn > 256 || bn % (bm == 256 ? 32 : 16)))
    MOE_FAIL(MOE_ERR_UNSUPPORTED,
             "moe_plan_build: bn=%d must be a multiple of %d in [16, 256] (or of 32 in (256, 512] with bm=256)", bn,
             bm == 256 ? 32 : 16);
  if (flags & ~(MOE_PAD_REPEAT | MOE_SPLIT_TAIL | MOE_ORDER_ALTERNATING | MOE_ORDER_HALF_INTERVAL | MOE_ORDER_LIGHT_LAST | MOE_GRID_BALANCED |
                MOE_GRID_STATIC | MOE_A_GATHER4 | MOE_EPI_REGISTER | MOE_SCHED_DYNAMIC | MOE_L2_PREFETCH | MOE_SPLIT_K |
                MOE_SCHED_HALF_LAST | MOE_SCHED_PLAN_ORDER))
    MOE_FAIL(MOE_ERR_INVALID, "moe_plan_build: unknown flags 0x%x", flags);
  if ((flags & MOE_GRID_BALANCED) && (flags & MOE_GRID_STATIC))
    MOE_FAIL(MOE_ERR_INVALID, "moe_plan_build: MOE_GRID_BALANCED and MOE_GRID_STATIC are exclusive");
  if (__builtin_popcount(flags & (MOE_ORDER_ALTERNATING | MOE_ORDER_HALF_INTERVAL | MOE_ORDER_LIGHT_LAST)) > 1)
    MOE_FAIL(MOE_ERR_INVALID, "moe_plan_build: choose one expert ordering");
  const bool split = (flags & MOE_SPLIT_TAIL) != 0;
  if (split && (bm != 256 || bn < 256))
    MOE_FAIL(MOE_ERR_UNSUPPORTED,
             "moe_plan_build: MOE_SPLIT_TAIL needs bm = 256 and bn = 256 or a wide tile (swap-AB tail tiles, M = 256)");
  // Tile-strategy catalog (Alg. 3): the kind of each expert's last row tile, chosen by its
  // row count r = m mod bm (the whole expert when m < bm): the first rule with r <= m_max.  Kind 1
  // (MOE_KIND_SWAP) needs CTA-pair tiles with 256-column MMA blocks; other shapes have no rules.
  moe_tile_rule cat[MOE_MAX_RULES];
  int32_t n_cat = 0;
  const bool pair_blocks = bm == 256 && bn >= 256;
  if (split) {
    cat[n_cat++] = {MOE_KIND_SWAP, bm};
  } else if (n_rules < 0) {
    if (bm == 256 && bn > 256) cat[n_cat++] = {MOE_KIND_GEMV, MOE_DEFAULT_GEMV_MAX};
  } else {
    if (n_rules > MOE_MAX_RULES) MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_plan_build: at most %d catalog rules", MOE_MAX_RULES);
    if (n_rules > 0 && !rules) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_build: null catalog");
    for (int32_t i = 0; i < n_rules; ++i) {
      if (rules[i].kind != MOE_KIND_WIDE && rules[i].kind != MOE_KIND_SWAP && rules[i].kind != MOE_KIND_GEMV &&
          rules[i].kind != MOE_KIND_RIDE)
        MOE_FAIL(MOE_ERR_INVALID, "moe_plan_build: catalog rule %d: kind %d", i, rules[i].kind);
      if (rules[i].kind == MOE_KIND_RIDE && (!(bm == 256 && bn > 256) || rules[i].m_max > MOE_RIDE_MAX_ROWS))
        MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_plan_build: MOE_KIND_RIDE needs wide pair tiles (bm = 256, bn > 256) and "
                 "m_max <= %d (got %d x %d, m_max %d)", MOE_RIDE_MAX_ROWS, bm, bn, rules[i].m_max);
      if (rules[i].kind == MOE_KIND_SWAP && !pair_blocks)
        MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_plan_build: MOE_KIND_SWAP needs bm = 256 and bn >= 256 (got %d x %d)", bm, bn);
      if (rules[i].kind == MOE_KIND_GEMV && (!(bm == 256 && bn > 256) || rules[i].m_max > MOE_GEMV_MAX_ROWS))
        MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_plan_build: MOE_KIND_GEMV needs wide pair tiles (bm = 256, bn > 256) and "
                 "m_max <= %d (got %d x %d, m_max %d)", MOE_GEMV_MAX_ROWS, bm, bn, rules[i].m_max);
      cat[n_cat++] = rules[i];
    }
  }
  bool allow_gemv = true;
  // RIDE: a full row tile to ride on (m > bm), 512-column tiles that all lie inside N (two 256-column halves)
  const bool ride_shape = bm == 256 && bn == 512 && N % bn == 0;
  auto kind_of = [&](int64_t m) -> int32_t {
    const int64_t r = m % bm;
    if (m <= 0 || r == 0) return MOE_KIND_WIDE;
    for (int32_t i = 0; i < n_cat; ++i) {
      // GEMV: whole single-row-tile tasks only, and only when the other tasks' tiles cover it
      if (cat[i].kind == MOE_KIND_GEMV && (m >= bm || !allow_gemv)) continue;
      if (cat[i].kind == MOE_KIND_RIDE && (m < bm || !ride_shape)) continue;
      if (r <= cat[i].m_max) return cat[i].kind;
    }
    return MOE_KIND_WIDE;
  };
  // CSR row offsets: exclusive prefix of counts in expert-id order.
  std::vector<int64_t> row_off(E + 1, 0);
  for (int32_t e = 0; e < E; ++e) {
    if (counts[e] < 0) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_build: counts[%d]=%d < 0", e, counts[e]);
    row_off[e + 1] = row_off[e] + counts[e];
  }
  if (row_off[E] >= INT_MAX) MOE_FAIL(MOE_ERR_CAPACITY, "moe_plan_build: sum of counts >= 2^31");

  // Tasks = experts.  nu = ceil(m/BM) * ceil(N/BN); K is not split.  With
  // MOE_SPLIT_TAIL an expert with m % BM != 0 is kind 1: its last row tile (the tail) runs as a
  // swap-AB tile of height roundup16(m % BM) — same tile partition, second tiling strategy.
  const int32_t n_tasks = E;
  const int64_t col_tiles = ceil_div(N, bn);
  std::vector<int64_t> nu(n_tasks);
  int32_t n_gemv = 0;                            // GEMV tasks have no tiles (Alg. 3's other strategy, §6.8)
  for (int pass = 0; pass < 2; ++pass) {
    n_gemv = 0;
    int64_t other_tiles = 0;
    for (int32_t i = 0; i < n_tasks; ++i) {
      const bool gemv = counts[i] > 0 && kind_of(counts[i]) == MOE_KIND_GEMV;
      n_gemv += gemv;
      nu[i] = counts[i] == 0 || gemv ? 0 : ceil_div(counts[i], bm) * col_tiles;
      other_tiles += nu[i];
    }
    if (n_gemv == 0 || (other_tiles >= MOE_GEMV_MIN_TILES &&
                        (int64_t)n_gemv * col_tiles * 100 >= (int64_t)MOE_GEMV_MIN_SHARE * other_tiles))
      break;
    allow_gemv = false;                          // too little tensor work to hide the GEMV streams
  }

  // Non-empty stage: sigma in natural order, then Alg. 1 over eta.
  std::vector<int32_t> sigma;
  for (int32_t i = 0; i < n_tasks; ++i)
    if (nu[i] > 0) sigma.push_back(i);
  if (flags & MOE_ORDER_LIGHT_LAST) {
    // heavy tasks, then the light (memory-bound) ones, each group in expert order
    std::stable_partition(sigma.begin(), sigma.end(), [&](int32_t i) { return counts[i] > MOE_LIGHT_ROWS; });
  } else if (flags & (MOE_ORDER_ALTERNATING | MOE_ORDER_HALF_INTERVAL)) {
    // §4.2 expert ordering: busy (compute-bound) and non-busy (memory-bound)
    // experts interleaved so a wave of CTAs mixes both.  sigma stays an injection.
    std::vector<int32_t> desc = sigma;
    std::stable_sort(desc.begin(), desc.end(), [&](int32_t x, int32_t y) { return counts[x] > counts[y]; });
    const int32_t n = (int32_t)desc.size();
    if (flags & MOE_ORDER_ALTERNATING) {
      const int32_t h = (n + 1) / 2;
      sigma.clear();
      for (int32_t i = 0; i < h; ++i) {
        sigma.push_back(desc[i]);
        if (h + i < n) sigma.push_back(desc[h + i]);
      }
    } else {
      int32_t w = 0;
      while ((1 << w) < n) ++w;
      std::vector<int32_t> slots;
      for (int32_t i = 0; i < (1 << w); ++i) {
        int32_t r = 0;
        for (int32_t b = 0; b < w; ++b) r |= ((i >> b) & 1) << (w - 1 - b);
        if (r < n) slots.push_back(r);
      }
      for (int32_t i = 0; i < n; ++i) sigma[slots[i]] = desc[i];
    }
  }
  std::vector<int64_t> prefix;
  int64_t acc = 0;
  for (int32_t i : sigma) {
    acc += nu[i];
    prefix.push_back(acc);
  }
  if (acc >= INT_MAX) MOE_FAIL(MOE_ERR_CAPACITY, "moe_plan_build: %lld tiles >= 2^31", (long long)acc);
  const int32_t M = (int32_t)sigma.size();
  const int32_t M_pad = moe::pad32(M);
  const int64_t words = MOE_PLAN_HEADER + 2 * (int64_t)M_pad + (int64_t)MOE_PLAN_TASK_WORDS * n_tasks + E + 1;
  if (blob_cap < words)
    MOE_FAIL(MOE_ERR_CAPACITY, "moe_plan_build: blob needs %lld words, cap %lld", (long long)words, (long long)blob_cap);

  std::memset(blob, 0, sizeof(int32_t) * words);
  blob[0] = MOE_PLAN_MAGIC;
  blob[1] = M;
  blob[2] = (int32_t)acc;
  blob[3] = M_pad;
  blob[4] = E;
  blob[5] = (int32_t)N;
  blob[6] = (int32_t)H;
  blob[7] = bm;
  blob[8] = bn;
  blob[9] = n_tasks;
  blob[10] = (int32_t)flags;
  for (int32_t i = 0; i < MOE_MAX_RULES; ++i) {          // [12 .. 16): the catalog (kind, m_max) pairs
    blob[12 + 2 * i] = i < n_cat ? cat[i].kind : MOE_KIND_WIDE;
    blob[13 + 2 * i] = i < n_cat ? cat[i].m_max : -1;
  }
  int32_t* pre = blob + MOE_PLAN_HEADER;
  int32_t* sig = pre + M_pad;
  int32_t* par = sig + M_pad;
  int32_t* roff = par + (int64_t)MOE_PLAN_TASK_WORDS * n_tasks;
  for (int32_t h = 0; h < M_pad; ++h) {
    if (h < M) {
      pre[h] = (int32_t)prefix[h];
      sig[h] = sigma[h];
    } else {
      // P:203 padding: "repeating its last element or padding with the maximum possible value".
      pre[h] = (flags & MOE_PAD_REPEAT) && M > 0 ? (int32_t)prefix[M - 1] : INT_MAX;
      sig[h] = 0;
    }
  }
  for (int32_t i = 0; i < n_tasks; ++i) {
    int32_t* p = par + (int64_t)MOE_PLAN_TASK_WORDS * i;
    p[0] = i;                                   // expert
    p[1] = (int32_t)row_off[i];                 // first CSR row of the task
    p[2] = counts[i];                           // rows
    p[3] = kind_of(counts[i]);                  // kind of the last row tile (1: swap-AB, the catalog)
    p[4] = bm;
    p[5] = bn;
    p[6] = (int32_t)ceil_div(counts[i], bm);    // row tiles
    p[7] = (int32_t)col_tiles;                  // col tiles
  }
  for (int32_t e = 0; e <= E; ++e) roff[e] = (int32_t)row_off[e];
  if (blob_len) *blob_len = words;
  return M == 0 && n_gemv == 0 ? MOE_OK_EMPTY : MOE_OK;
}

const char* moe_last_error(void) { return moe::g_last_error.c_str(); }

const char* moe_version(void) { return "moe_sm100 0.1 (sm_100a)"; }

}  // extern "C"

// ---------------------------------------------------------------------------
// Device-resident plan
// ---------------------------------------------------------------------------
constexpr int64_t kSchedWords = 32;   // device words after the blob for the dynamic tile order (one 128-B line)

struct moe_plan {
  std::vector<int32_t> blob;
  int64_t words = 0;
  int32_t* dev = nullptr;
  int64_t dev_words = 0;
  cudaStream_t stream = nullptr;
  int32_t E = 0;
  int64_t H = 0, N = 0;
  int32_t bm = 0, bn = 0;
  uint32_t flags = 0;
  std::vector<moe_tile_rule> rules;   // the catalog given at creation (n_rules < 0: built-in)
  int32_t n_rules = -1;
  bool device_mode = false;   // device blob written by moe_plan_device; host blob stale
  float* sk_ws = nullptr;     // one-CTA plans: split-K partials [kSKUnitsPerCta * sk_ctas][kSKRows][kSKCols]
  int32_t* sk_cnt = nullptr;  //                 per-tile arrival counters [kSKMaxTiles] (zero between launches)
  int32_t sk_ctas = 0;
};

namespace moe {
const int32_t* plan_blob_host(const moe_plan* p, int64_t* words) {
  if (words) *words = p->words;
  return p->blob.data();
}
const int32_t* plan_blob_dev(const moe_plan* p) { return p->dev; }
cudaStream_t plan_stream(const moe_plan* p) { return p->stream; }
bool plan_device_mode(const moe_plan* p) { return p->device_mode; }
void plan_set_device_mode(moe_plan* p, bool on) { p->device_mode = on; }
void plan_shape(const moe_plan* p, int32_t* E, int32_t* H, int32_t* N, int32_t* bm, int32_t* bn, uint32_t* flags) {
  *E = p->E;
  *H = (int32_t)p->H;
  *N = (int32_t)p->N;
  *bm = p->bm;
  *bn = p->bn;
  *flags = p->flags;
}
int32_t* plan_blob_dev_mut(moe_plan* p) { return p->dev; }
int32_t* plan_sched_dev(const moe_plan* p) { return p->dev + p->dev_words; }
float* plan_sk_ws(const moe_plan* p, int32_t** cnt, int32_t* ctas) {
  *cnt = p->sk_cnt;
  *ctas = p->sk_ctas;
  return p->sk_ws;
}
// The catalog (header words 12-15) holds a swap-AB or ride rule: the launch needs the two-strategy kernel.
bool plan_has_swap(const moe_plan* p) {
  for (int i = 0; i < MOE_MAX_RULES; ++i)
    if ((p->blob[12 + 2 * i] == MOE_KIND_SWAP || p->blob[12 + 2 * i] == MOE_KIND_RIDE) && p->blob[13 + 2 * i] > 0)
      return true;
  return false;
}
}  // namespace moe

extern "C" {

static moe_status upload(moe_plan* p, cudaStream_t s) {
  cudaError_t err = cudaMemcpyAsync(p->dev, p->blob.data(), sizeof(int32_t) * p->words,
                                    cudaMemcpyHostToDevice, s);
  if (err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "cudaMemcpyAsync(plan blob): %s", cudaGetErrorString(err));
  return MOE_OK;
}

moe_status moe_plan_create(const int32_t* counts, int32_t E, int64_t H, int64_t N, int32_t bm,
                           int32_t bn, uint32_t flags, void* stream, moe_plan** out) {
  return moe_plan_create_catalog(counts, E, H, N, bm, bn, flags, nullptr, -1, stream, out);
}

moe_status moe_plan_create_catalog(const int32_t* counts, int32_t E, int64_t H, int64_t N, int32_t bm, int32_t bn,
                                   uint32_t flags, const moe_tile_rule* rules, int32_t n_rules, void* stream,
                                   moe_plan** out) {
  moe::NvtxRange nvtx("moe_plan_create");
  moe::clear_error();
  if (!out) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_create: null out");
  *out = nullptr;
  if (E < 1) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_create: E=%d", E);
  auto* p = new moe_plan();
  p->blob.resize(moe_plan_blob_words(E));
  std::vector<int32_t> zeros;
  if (!counts) {                                // plan to be filled on the device (moe_plan_device)
    zeros.assign(E, 0);
    counts = zeros.data();
  }
  moe_status st = moe_plan_build_catalog(counts, E, H, N, bm, bn, flags, rules, n_rules, p->blob.data(),
                                         (int64_t)p->blob.size(), &p->words);
  if (st < 0) {
    delete p;
    return st;
  }
  if (n_rules > 0) p->rules.assign(rules, rules + n_rules);
  p->n_rules = n_rules;
  bm = p->blob[7];                              // resolved tile height (bm = 0 means auto)
  bn = p->blob[8];                              // resolved tile width (bn = 0 means auto)
  flags = (uint32_t)p->blob[10];                // auto may add MOE_SPLIT_TAIL
  p->stream = (cudaStream_t)stream;
  p->E = E;
  p->H = H;
  p->N = N;
  p->bm = bm;
  p->bn = bn;
  p->flags = flags;
  p->dev_words = (int64_t)p->blob.size();
  // + kSchedWords after the blob: the dynamic tile order's counters (zero between launches)
  cudaError_t err = cudaMallocAsync((void**)&p->dev, sizeof(int32_t) * (p->dev_words + kSchedWords), p->stream);
  if (err == cudaSuccess)
    err = cudaMemsetAsync(p->dev + p->dev_words, 0, sizeof(int32_t) * kSchedWords, p->stream);
  if (err != cudaSuccess) {
    if (p->dev) cudaFreeAsync(p->dev, p->stream);
    delete p;
    MOE_FAIL(MOE_ERR_CUDA, "cudaMallocAsync(plan): %s", cudaGetErrorString(err));
  }
  if (bm == 128 && (flags & MOE_SPLIT_K)) {
    // split-K workspace of one-CTA plans: kSKUnitsPerCta partial slots per SM, counters zeroed
    int dev = 0, sms = 0;
    err = cudaGetDevice(&dev);
    if (err == cudaSuccess) err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err == cudaSuccess) {
      p->sk_ctas = sms;
      const size_t ws = sizeof(float) * moe::kSKUnitsPerCta * (size_t)sms * moe::kSKRows * moe::kSKCols;
      err = cudaMallocAsync((void**)&p->sk_ws, ws + sizeof(int32_t) * moe::kSKMaxTiles, p->stream);
    }
    if (err == cudaSuccess) {
      p->sk_cnt = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(p->sk_ws) +
                                             sizeof(float) * moe::kSKUnitsPerCta * (size_t)p->sk_ctas * moe::kSKRows *
                                                 moe::kSKCols);
      err = cudaMemsetAsync(p->sk_cnt, 0, sizeof(int32_t) * moe::kSKMaxTiles, p->stream);
    }
    if (err != cudaSuccess) {
      if (p->sk_ws) cudaFreeAsync(p->sk_ws, p->stream);
      cudaFreeAsync(p->dev, p->stream);
      delete p;
      MOE_FAIL(MOE_ERR_CUDA, "plan stream-K workspace: %s", cudaGetErrorString(err));
    }
  }
  moe_status up = upload(p, p->stream);
  if (up != MOE_OK) {
    if (p->sk_ws) cudaFreeAsync(p->sk_ws, p->stream);
    cudaFreeAsync(p->dev, p->stream);
    delete p;
    return up;
  }
  *out = p;
  return st;
}

moe_status moe_plan_suggest_tile(int64_t rows, int32_t E, int64_t H, int64_t N, int32_t* bm, int32_t* bn) {
  moe::clear_error();
  if (!bm || !bn) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_suggest_tile: null output");
  if (rows < 0 || E < 1) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_suggest_tile: rows=%lld E=%d", (long long)rows, E);
  // The automatic rule of moe_plan_build applied to `rows` routed rows spread evenly over
  // min(E, rows) experts (the expectation for plans built before the counts exist).
  const int64_t active = std::max<int64_t>(1, std::min<int64_t>(E, rows));
  const int64_t per = std::max<int64_t>(1, ceil_div(rows, active));
  if (per >= INT_MAX) MOE_FAIL(MOE_ERR_CAPACITY, "moe_plan_suggest_tile: rows per expert >= 2^31");
  std::vector<int32_t> counts(E, 0);
  for (int64_t e = 0; e < active; ++e) counts[e] = (int32_t)per;
  std::vector<int32_t> blob(moe_plan_blob_words(E));
  int64_t len = 0;
  moe_status st = moe_plan_build(counts.data(), E, H, N, 0, 0, 0, blob.data(), (int64_t)blob.size(), &len);
  if (st < 0) return st;
  *bm = blob[7];
  *bn = blob[8];
  return MOE_OK;
}

moe_status moe_plan_create_expected(int64_t expected_rows, int32_t E, int64_t H, int64_t N, int32_t bm, int32_t bn,
                                    uint32_t flags, void* stream, moe_plan** out) {
  moe::clear_error();
  if (bm == 0 && bn == 0) {
    moe_status st = moe_plan_suggest_tile(expected_rows, E, H, N, &bm, &bn);
    if (st < 0) return st;
  }
  return moe_plan_create(nullptr, E, H, N, bm, bn, flags, stream, out);
}

moe_status moe_plan_update(moe_plan* p, const int32_t* counts, void* stream) {
  moe::clear_error();
  if (!p) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_update: null plan");
  int64_t words = 0;
  moe_status st = moe_plan_build_catalog(counts, p->E, p->H, p->N, p->bm, p->bn, p->flags, p->rules.data(), p->n_rules,
                                         p->blob.data(), (int64_t)p->blob.size(), &words);
  if (st < 0) return st;
  p->words = words;
  p->device_mode = false;
  if (stream) p->stream = (cudaStream_t)stream;
  moe_status up = upload(p, p->stream);
  return up != MOE_OK ? up : st;
}

moe_status moe_plan_sync(moe_plan* p, void* stream) {
  moe::clear_error();
  if (!p) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_sync: null plan");
  if (!p->device_mode) return MOE_OK;
  cudaStream_t s = stream ? (cudaStream_t)stream : p->stream;
  cudaError_t e = cudaMemcpyAsync(p->blob.data(), p->dev, sizeof(int32_t) * p->dev_words, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_plan_sync: %s", cudaGetErrorString(e));
  moe::BlobView v;
  if (!moe::blob_view(p->blob.data(), (int64_t)p->blob.size(), &v)) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_sync: corrupt device blob");
  p->words = v.words;
  p->device_mode = false;
  if (p->blob[11] != 0)
    MOE_FAIL(MOE_ERR_CAPACITY, "moe_plan_device: rows or tiles >= 2^31 (device planner status %d)", p->blob[11]);
  return p->blob[1] == 0 ? MOE_OK_EMPTY : MOE_OK;
}

moe_status moe_plan_query(const moe_plan* p, int32_t* M, int32_t* total, int32_t* M_pad) {
  if (!p) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_query: null plan");
  if (p->device_mode) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_query: plan is device-resident (call moe_plan_sync)");
  if (M) *M = p->blob[1];
  if (total) *total = p->blob[2];
  if (M_pad) *M_pad = p->blob[3];
  return MOE_OK;
}

moe_status moe_plan_blob(const moe_plan* p, int32_t* out, int64_t cap, int64_t* len) {
  if (!p) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_blob: null plan");
  if (p->device_mode) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_blob: plan is device-resident (call moe_plan_sync)");
  if (len) *len = p->words;
  if (out) {
    if (cap < p->words) MOE_FAIL(MOE_ERR_CAPACITY, "moe_plan_blob: cap %lld < %lld", (long long)cap, (long long)p->words);
    std::memcpy(out, p->blob.data(), sizeof(int32_t) * p->words);
  }
  return MOE_OK;
}

const int32_t* moe_plan_device_blob(const moe_plan* p) { return p ? p->dev : nullptr; }

void moe_plan_destroy(moe_plan* p) {
  if (!p) return;
  if (p->sk_ws) cudaFreeAsync(p->sk_ws, p->stream);
  if (p->dev) cudaFreeAsync(p->dev, p->stream);
  delete p;
}

}  // extern "C"
