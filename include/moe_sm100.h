/*
 * moe_sm100.h — C ABI of the single-launch, statically batched MoE expert GEMM
 * for NVIDIA B200 (sm_100a).  Method: arXiv 2501.16103 ("P:n" = line n of the
 * paper's LaTeX source, /root/reference/PAPER.md; see DESIGN.md for readings).
 *
 *   moe_route      tokens' top-k expert ids -> per-expert token-index arrays
 *                  (CSR).
 *   moe_plan_*     expert token counts + tile shape -> the compressed mapping:
 *                  TilePrefix over non-empty tasks (Alg. 1; Alg. 4's
 *                  extra stage) plus sigma and task parameters p_i.
 *   moe_gemm       ONE kernel launch computing every (expert, output-tile) task:
 *                  each CTA decodes (task, tile) on device with the warp
 *                  vote/popcount algorithm (Alg. 2), gathers its
 *                  token rows through the token-index array and
 *                  multiplies them by that expert's weight slice.
 *   moe_decode_debug  the device decode alone, for bit-exact parity tests.
 *
 * Conventions (all entry points):
 *   - Plain pointers and sizes only.  "_dev" = device memory, "_host" = host
 *     memory.  All tensors are caller-owned; the library never frees them.
 *   - `stream` is a cudaStream_t (passed as void*).  Device work is enqueued
 *     on it; no entry point synchronises the stream.
 *   - Return codes: moe_status below.  No C++ exception crosses the ABI.  On a
 *     non-OK status nothing has been enqueued and moe_last_error() returns a
 *     thread-local message.  Asynchronous CUDA faults surface at the caller's
 *     next synchronisation, as for any CUDA library.
 *   - Indices are 0-based (reading R1).  Rows of the token-index
 *     array are grouped by expert in ascending expert id; within an expert they
 *     are in ascending token id (reading R3).
 */
#ifndef MOE_SM100_H_
#define MOE_SM100_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t moe_status;
#define MOE_OK               0   /* success                                                     */
#define MOE_OK_EMPTY         1   /* success, nothing to compute (every expert empty): no launch */
#define MOE_ERR_INVALID     (-1) /* bad argument, shape, null or misaligned pointer             */
#define MOE_ERR_UNSUPPORTED (-2) /* H%8, N%8 (TMA needs 16-byte strides), tile shape, non-sm_100 */
#define MOE_ERR_CAPACITY    (-3) /* int32 overflow of rows / tiles, too many tasks, buffer small */
#define MOE_ERR_CUDA        (-4) /* a CUDA runtime/driver call failed (message has the name)     */
#define MOE_ERR_NCCL        (-5) /* reserved for the expert-parallel layer                       */

/* Expert (task) ordering of sigma, §4.2, plan flags; results never depend on it. */
#define MOE_ORDER_ALTERNATING    4u  /* sort non-empty tasks by load (desc, ties: lower id), interleave
                                        the busiest half with the rest: b1, s1, b2, s2, ...          */
#define MOE_ORDER_HALF_INTERVAL  8u  /* same sort; the i-th busiest task takes the i-th slot of the
                                        bit-reversal (van der Corput) sequence over the slots        */
#define MOE_ORDER_LIGHT_LAST  4096u  /* tasks of > MOE_LIGHT_ROWS rows first, then the light ones (each group
                                        in expert order); with the dynamic tile order (CTA-pair tiles)
                                        the kernel then interleaves the light tiles among the others in
                                        proportion, so memory-bound tiles overlap compute-bound ones
                                        instead of streaming W all at once           */
#define MOE_LIGHT_ROWS 64

/* Launch options carried by the plan (moe_gemm reads them from the plan it is given; they never
 * change Y).  Defaults are the measured-fastest choices; these exist for
 * same-box A/B timing and for tests that pin the alternative paths.                                 */
#define MOE_GRID_BALANCED  16u  /* persistent grid over ceil(tiles / ceil(tiles / CTAs)) CTAs (pairs), each
                                   W or W-1 tiles (default for one-CTA tiles only)                    */
#define MOE_GRID_STATIC    32u  /* plain static stride over all CTAs (pairs): no balanced grid, no
                                   dynamic tile order                                                 */
#define MOE_A_GATHER4      64u  /* stage token rows with TMA tile::gather4 (one-CTA tiles) instead of
                                   cp.async                                                           */
#define MOE_EPI_REGISTER  128u  /* bf16 Y through masked register stores only (no TMA tile stores)    */
#define MOE_L2_PREFETCH   512u  /* load/store-path L2 prefetch of W for memory-bound tiles (one-CTA tiles,
                                   swap-AB tiles) ahead of the ring — opt-in: measured slower */
#define MOE_SCHED_DYNAMIC 256u  /* dynamic tile order: after its first tile each persistent CTA (pair)
                                   takes the next virtual tile from a counter in the plan's device
                                   memory (the order the hardware dispatches one block per tile,
                                   P:138) instead of the static stride — the default for CTA-pair
                                   tiles (bm = 256) unless MOE_GRID_STATIC / MOE_GRID_BALANCED is set;
                                   launches on one plan must be stream-ordered (the counter is reset
                                   by the launch's last CTA pair)                                     */

#define MOE_SPLIT_K  1024u      /* one-CTA tiles: when whole tiles would leave SMs idle and every task has
                                   <= 16 rows, split each tile's K blocks into S parts over one CTA per SM
                                   and sum them in K order (opt-in: measured slower than whole tiles on the
                                   balanced grid)                                       */

#define MOE_SCHED_PLAN_ORDER 16384u /* dynamic order of wide tiles strictly in the plan's order (default when N %
                                   bn != 0: every task's narrower last column block after the full-width
                                   ones)                                              */
#define MOE_SCHED_HALF_LAST 2048u /* dynamic order of wide tiles: each task's <= 128-row last row tiles after
                                   all full tiles (LPT-like end of the launch; opt-in: 8x22B +3.4 %, Mix
                                   -1.9 % — a half tile moved away from its column block re-reads W from
                                   HBM)                                                */

/* Output element types of moe_gemm. */
#define MOE_DTYPE_BF16 0
#define MOE_DTYPE_F32  1

/* Plan flags. */
#define MOE_PAD_MAX     0u  /* pad TilePrefix with INT32_MAX ("the maximum possible value") */
#define MOE_PAD_REPEAT  1u  /* pad TilePrefix by repeating its last element                */
#define MOE_SPLIT_TAIL  2u  /* bm = 256, bn = 256 or 512: an expert whose m is not a multiple of 256
                               is kind 1 — the LAST row tile of each column block (its m mod 256 tail
                               rows) runs as a swap-AB pair tile (each 256-column W block as the
                               M = 256 operand, the tail's tokens as N = tail rounded up to 16).
                               Same tile partition; a second tiling strategy in the launch
                               (Alg. 3 with K = 2).                                      */

/* ---- the compressed mapping ("plan blob"), int32 words -------------------
 * Built on the host by moe_plan_build (no GPU needed) and copied once to the
 * device by moe_plan_create ("pre-computed on the host and then copied to the
 * device").  Layout:
 *   [0]  MOE_PLAN_MAGIC          [1] M  = number of non-empty tasks (|eta|)
 *   [2]  total virtual tiles     [3] M_pad = M rounded up to a multiple of 32 (>= 32)
 *   [4]  E (experts)             [5] N (expert output width)   [6] H (hidden = GEMM K)
 *   [7]  BM (tile rows)          [8] BN (tile cols)            [9] n_tasks (tasks incl. empty)
 *   [10] flags                   [11] device planner status (0 = ok, 3 = capacity)
 *   [12..16) the tile-strategy catalog: MOE_MAX_RULES (kind, m_max) pairs (unused: m_max = -1)
 *   [16 .. 16+M_pad)               TilePrefix: inclusive prefix of nu over the
 *                                  non-empty tasks (Alg. 1), padded
 *   [16+M_pad .. 16+2*M_pad)       sigma: non-empty index -> task index,
 *                                  padded with 0
 *   [16+2*M_pad .. +8*n_tasks)     task parameters p_i, 8 words per
 *                                  task i: {expert, row0, rows, kind, bm, bn,
 *                                  row_tiles, col_tiles}; row0 = first CSR row of
 *                                  the task (= row_off[expert] + offset in expert);
 *                                  kind = the catalog's strategy for the task's last
 *                                  row tile (MOE_KIND_SWAP: swap-AB, see below)
 *   [.. +E+1)                      row_off: exclusive prefix of counts (CSR offsets)
 * nu(task) = row_tiles * col_tiles, row_tiles = ceil(rows/BM), col_tiles = ceil(N/BN).
 * Intra-task tile order: row tile fastest, rt = l mod row_tiles, ct = l div
 * row_tiles (reading R5).
 */
#define MOE_PLAN_MAGIC      0x4d4f4531  /* "MOE1" */
#define MOE_PLAN_HEADER     16
#define MOE_PLAN_TASK_WORDS 8

/* ---- per-task tiling strategies ("different tasks inside a batch can have different
 * tiling strategies"; "categorized into several pre-defined tiling strategies ...
 * GEMMs with large input and output sizes prefer large tiles"; Alg. 3 / Alg. 4's per-task
 * dispatch).  With CTA-pair tiles (bm = 256, bn = 256 or 512) each expert's LAST row tile — its
 * r = m mod 256 tail rows, or all its rows when m < 256 — is executed by the strategy the catalog
 * picks for r; every other row tile is a full 256-row tile:
 *   MOE_KIND_WIDE  the bm x bn tile (r <= 128: an M = 128 pair MMA, half the tensor time);
 *   MOE_KIND_SWAP  a swap-AB tile: each 256-column W block is the M = 256 operand, the tile's r
 *                  tokens the N operand rounded up to 16 (tensor time ~ r, not 128 / 256), its W
 *                  blocks also prefetched into L2 ahead of the ring (memory-bound tiles).
 * Rules are tried in order; the first with r <= m_max gives the kind (none matches: WIDE).  The tile
 * partition — hence the mapping and Y — does not depend on the catalog. */
typedef struct { int32_t kind; int32_t m_max; } moe_tile_rule;
#define MOE_KIND_WIDE 0
#define MOE_KIND_SWAP 1
#define MOE_KIND_GEMV 2           /* a whole task of m <= m_max <= MOE_GEMV_MAX_ROWS rows (a single partial row
                                     tile) computed as a GEMV on the CUDA cores by the epilogue warps between
                                     their accumulator drains (wide pair tiles only): the task has no tiles
                                     (nu = 0, outside TilePrefix and sigma), its W streams while the tensor
                                     cores work on the other tasks                       */
#define MOE_KIND_RIDE 3           /* an expert of m = 256 R + r rows (R >= 1, 1 <= r <= m_max <= MOE_RIDE_MAX_ROWS)
                                     in a plan of 256 x 512 pair tiles with N % 512 == 0: its last two row-tile
                                     slots of each column block are the two 256-column halves of its last full
                                     row tile, and each also computes the r tail rows x its 256 columns with a
                                     swap-AB MMA (the staged W block as the M = 256 operand, the tail tokens as
                                     N = r rounded up to 16) on the same staged K blocks — the tail needs no
                                     W stream of its own.  Same tile count (ceil(m / 256) per column block),
                                     same mapping; kernels without the strategy (FP8, gated, contiguous-row A)
                                     run those slots as the plain wide tiles.  Elsewhere the
                                     rule does not match (the catalog's next rule applies).            */
#define MOE_RIDE_MAX_ROWS 32
#define MOE_GEMV_MAX_ROWS 4
#define MOE_GEMV_MIN_SHARE 10     /* ... and only when the GEMV candidates would otherwise take >= this many
                                     percent as many tiles (count x column tiles) as the other tasks have: a
                                     GEMV unit streams all of K for 128 columns on one warp, a tail that a
                                     handful of candidates does not repay              */
#define MOE_GEMV_MIN_TILES 128    /* GEMV rules apply only when the plan's other tasks have >= this many tiles
                                     (their tensor work must cover the GEMV streams); otherwise those tasks
                                     fall through to the catalog's next rule                              */
#define MOE_MAX_RULES 2
#ifndef MOE_DEFAULT_GEMV_MAX
#define MOE_DEFAULT_GEMV_MAX 4    /* built-in catalog of wide pair plans (bm 256, bn > 256): {GEMV, 4};
                                     other shapes: no rules (SWAP is opt-in: measured no faster, §7.5)    */
#endif
#define MOE_DEFAULT_SWAP_MAX 64   /* the swap-AB rule tests and A/B runs use: {SWAP, 64}                   */

/* A plan has work to launch when it has tiles (header word 2 > 0) or GEMV tasks; moe_gemm returns
 * MOE_OK_EMPTY only when it has neither. */

/* Number of int32 words moe_plan_build needs for E experts (upper bound). */
int64_t moe_plan_blob_words(int32_t E);

/*
 * Build the compressed mapping on the host.
 *   counts_host [E]  tokens routed to each expert (m_e >= 0), host memory.
 *   H, N             GEMM K and expert output width; both must be multiples of 8.
 *   bm, bn           tile shape.  bm = 64 (bn = 256): decode tile — one CTA, swap-AB (the
 *                    W block as two M = 128 operands, <= 64 tokens as N), opt-in;
 *                    bm = 128: one CTA per tile (tcgen05 M=128, cta_group::1);
 *                    bm = 256: a CTA pair per tile (tcgen05 M=256, cta_group::2, each
 *                    CTA 128 rows and half of the W block).  16 <= bn <= 256, bn % 16 == 0
 *                    (bn % 32 == 0 when bm = 256), or bn = 512 with bm = 256: a wide pair
 *                    tile (two N = 256 MMA blocks per staged K block, both TMEM accumulators).
 *                    bm = 0: automatic — 256 unless the pair tiles' extra padding rows exceed
 *                    their ~10% per-row speed advantage (sum of ceil(m_e/256)*256 > 1.10 *
 *                    sum of ceil(m_e/128)*128).  bn = 0: automatic — 512 when bm resolves to
 *                    256 and N >= 512, else 256.  The blob records
 *                    the resolved bm and bn.
 *   flags            MOE_PAD_MAX | MOE_PAD_REPEAT, optionally | MOE_SPLIT_TAIL and one of
 *                    MOE_ORDER_ALTERNATING / MOE_ORDER_HALF_INTERVAL (sigma order, §4.2).
 *   blob, blob_cap   caller buffer of blob_cap int32 words (see moe_plan_blob_words).
 *   blob_len         out: words written.
 * Returns MOE_OK, MOE_OK_EMPTY (all experts empty: M = 0, total = 0),
 * MOE_ERR_INVALID, MOE_ERR_UNSUPPORTED or MOE_ERR_CAPACITY (sum of counts or
 * total tiles >= 2^31, blob_cap too small).  Pure host code: never touches CUDA.
 */
moe_status moe_plan_build(const int32_t* counts_host, int32_t E, int64_t H, int64_t N,
                          int32_t bm, int32_t bn, uint32_t flags,
                          int32_t* blob, int64_t blob_cap, int64_t* blob_len);

/*
 * moe_plan_build with an explicit catalog: rules[n_rules] (n_rules <= MOE_MAX_RULES), n_rules = 0 for
 * one strategy per launch (every tile MOE_KIND_WIDE), n_rules < 0 for the built-in catalog
 * (moe_plan_build's behaviour).  MOE_SPLIT_TAIL in flags overrides it with {MOE_KIND_SWAP, bm}.
 * MOE_ERR_UNSUPPORTED: a SWAP rule on a plan whose tiles are not CTA pairs with 256-column blocks.
 */
moe_status moe_plan_build_catalog(const int32_t* counts_host, int32_t E, int64_t H, int64_t N,
                                  int32_t bm, int32_t bn, uint32_t flags, const moe_tile_rule* rules,
                                  int32_t n_rules, int32_t* blob, int64_t blob_cap, int64_t* blob_len);

/* Opaque plan: the host blob plus its device copy (library-owned). */
typedef struct moe_plan moe_plan;

/*
 * moe_plan_build + one stream-ordered H2D copy of the blob into a device buffer
 * owned by the plan (the copy is "very small" — its length is the
 * number of tasks, not the number of blocks).  The plan is bound to `stream`:
 * moe_gemm / moe_decode_debug must be enqueued on the same stream (or after an
 * event on it).  On MOE_OK_EMPTY a valid plan with total = 0 is returned.
 */
moe_status moe_plan_create(const int32_t* counts_host /* NULL: all zero, for moe_plan_device */,
                           int32_t E, int64_t H, int64_t N,
                           int32_t bm, int32_t bn, uint32_t flags, void* stream, moe_plan** out);

/* moe_plan_create with an explicit catalog (as moe_plan_build_catalog); the device planner and
 * moe_plan_update keep it. */
moe_status moe_plan_create_catalog(const int32_t* counts_host, int32_t E, int64_t H, int64_t N,
                                   int32_t bm, int32_t bn, uint32_t flags, const moe_tile_rule* rules,
                                   int32_t n_rules, void* stream, moe_plan** out);

/* Re-plan in place for new counts (same E, H, N, flags; the bm, bn resolved at creation are kept);
 * reuses the device buffer. */
moe_status moe_plan_update(moe_plan* plan, const int32_t* counts_host, void* stream);

/*
 * Device-side planner ("or directly generated on the device", P:144 parallel prefix
 * sum): one single-block kernel on `stream` rebuilds the plan's device blob from
 * device-resident counts (e.g. moe_route's counts_dev) — no host synchronisation, so
 * route -> plan -> moe_gemm can be enqueued (and graph-captured) back to back.  Same
 * arithmetic and layout as moe_plan_build except M_pad = pad32(E) (count-independent).
 * The plan keeps the E, H, N, bm, bn, flags of moe_plan_create (counts_host may be NULL
 * there; bm = 0 then resolves to 256 when bn % 32 == 0, bn = 0 to 512 when N >= 512).  Requires E <= 1024.  Afterwards
 * the host copy is stale: moe_plan_query / moe_plan_blob / moe_decode_debug return
 * MOE_ERR_INVALID until moe_plan_sync; moe_gemm launches one CTA (pair) per SM and reads
 * the tile count from the device blob.  If the counts overflow int32 rows or tiles the
 * device blob gets total = 0 and header word 11 = 3 (reported by moe_plan_sync).
 */
moe_status moe_plan_device(moe_plan* plan, const int32_t* counts_dev, void* stream);

/*
 * The tile shape (bm, bn) moe_plan_build's automatic rule (bm = bn = 0) picks for `rows` routed rows
 * spread evenly over min(E, rows) experts: the expectation for a plan created before its counts exist.
 * Pure host code.
 */
moe_status moe_plan_suggest_tile(int64_t rows, int32_t E, int64_t H, int64_t N, int32_t* bm, int32_t* bn);

/*
 * moe_plan_create(NULL counts, ...) for a device-planned step whose batch has about expected_rows routed
 * rows (T * k): with bm = bn = 0 the tile shape is moe_plan_suggest_tile(expected_rows, ...), so a
 * C-ABI caller gets the shape the automatic rule would choose for its batch (e.g. one-CTA tiles for a
 * decode step) instead of the count-free default.  Other arguments as moe_plan_create.
 */
moe_status moe_plan_create_expected(int64_t expected_rows, int32_t E, int64_t H, int64_t N, int32_t bm, int32_t bn,
                                    uint32_t flags, void* stream, moe_plan** out);

/* Copy a device-planned blob back to the host (synchronises `stream`; NULL = plan's stream). */
moe_status moe_plan_sync(moe_plan* plan, void* stream);

/* Scalars of a plan (any pointer may be NULL). */
moe_status moe_plan_query(const moe_plan* plan, int32_t* M, int32_t* total_tiles, int32_t* M_pad);

/* Copy of the host blob into a caller buffer of cap words; *len = blob words. */
moe_status moe_plan_blob(const moe_plan* plan, int32_t* out, int64_t cap, int64_t* len);

/* Device address of the plan blob (same layout), for debugging and tests. */
const int32_t* moe_plan_device_blob(const moe_plan* plan);

/* Stream-ordered release of the device buffer (safe while work using it is in flight). */
void moe_plan_destroy(moe_plan* plan);

/*
 * Token-index buckets on device, stable: token_idx[row_off[e] + r]
 * is the r-th smallest token id t with e in topk_ids[t, :].
 *   topk_ids_dev [T, k] int32 row-major, expert ids in [0, E); no token may list
 *                an expert twice.  A negative id marks a masked slot (skipped silently;
 *                used by expert parallelism for slots owned by another rank).
 *   counts_dev   [E]   out: m_e.
 *   row_off_dev  [E+1] out: exclusive prefix of counts.
 *   token_idx_dev[T*k] out.
 *   slot_dev     [T*k] out (nullable): the top-k position j of each row.
 *   status_dev   [1]   out (nullable): set to 0, or to 1 if an id was >= E or
 *                      duplicated in a token (those entries are dropped).
 * Three kernel launches on `stream` (chunk histograms, one scan block, chunk x expert stable
 * compaction) plus a stream-ordered scratch allocation (cudaMallocAsync, n_chunks * E int32);
 * T*k < 2^31, 1 <= k <= 32, 1 <= E <= 1024.
 */
moe_status moe_route(const int32_t* topk_ids_dev, int64_t T, int32_t k, int32_t E,
                     int32_t* counts_dev, int32_t* row_off_dev, int32_t* token_idx_dev,
                     int32_t* slot_dev, int32_t* status_dev, void* stream);

/*
 * moe_route fused with moe_plan_device: the scan block that produces counts / row_off also
 * writes `plan`'s device blob (same kernels, no extra launch, no host synchronisation).
 * plan must have been created for the same E (counts_host may have been NULL).
 */
moe_status moe_route_plan(const int32_t* topk_ids_dev, int64_t T, int32_t k, int32_t E,
                          int32_t* counts_dev, int32_t* row_off_dev, int32_t* token_idx_dev,
                          int32_t* slot_dev, int32_t* status_dev, moe_plan* plan, void* stream);

/*
 * moe_route / moe_route_plan with explicit kernel-path options (same results on every path; for
 * same-box timing and for tests that pin each path):
 *   MOE_ROUTE_NO_SMALL       never the single-block small-batch kernel (T <= 1024, E <= 16, k <= 8)
 *   MOE_ROUTE_THREE_KERNELS  histogram + scan block + compaction instead of the fused two-kernel form
 * plan: NULL (moe_route) or a plan to fill on the device (moe_route_plan).
 */
#define MOE_ROUTE_NO_SMALL       1u
#define MOE_ROUTE_THREE_KERNELS  2u
moe_status moe_route_ex(const int32_t* topk_ids_dev, int64_t T, int32_t k, int32_t E,
                        int32_t* counts_dev, int32_t* row_off_dev, int32_t* token_idx_dev,
                        int32_t* slot_dev, int32_t* status_dev, moe_plan* plan, uint32_t route_flags,
                        void* stream);

/*
 * The hot path: Y[row0 + r, n] = sum_h X[token_idx[row0 + r], h] * W[e, h, n]
 * for every task of the plan, in ONE persistent kernel launch (sm_100a: token rows
 * gathered by cp.async (or TMA gather4), TMA tiles of W, tcgen05.mma with fp32
 * accumulation in TMEM, warp-specialised pipeline).
 *   X_dev         [T, H] bf16 row-major (token activations), 16-byte aligned.
 *   token_idx_dev [sum m_e] int32, the CSR of moe_route, consistent with the
 *                 plan's counts (not re-checked on device).  NULL: the rows of X are
 *                 already in the plan's CSR order (X row i = CSR row i, T >= sum m_e;
 *                 e.g. the intermediate activations of the FFN layer) and are staged
 *                 with one 128-row tile TMA per stage instead of a gather.
 *   W_dev         [E, H, N] bf16 row-major (expert weights), 16-byte aligned.
 *   Y_dev         [sum m_e, N] of y_dtype (MOE_DTYPE_BF16: fp32 accumulate, RNE
 *                 to bf16; MOE_DTYPE_F32: the fp32 accumulator), 16-byte aligned.
 * Returns MOE_OK_EMPTY without launching when the plan has no tiles.
 */
moe_status moe_gemm(const moe_plan* plan, const void* X_dev, int64_t T, const int32_t* token_idx_dev,
                    const void* W_dev, void* Y_dev, int32_t y_dtype, void* stream);

/*
 * moe_gemm with the output rows scattered: the result row of CSR row i is written to
 * Y_dev[y_row_map_dev[i]] (Y_dev has at least max(map)+1 rows of N).  Used by expert
 * parallelism to write results straight into the combine send buffer (no Y gather copy).
 */
moe_status moe_gemm_rowmap(const moe_plan* plan, const void* X_dev, int64_t T, const int32_t* token_idx_dev,
                           const void* W_dev, void* Y_dev, int32_t y_dtype, const int32_t* y_row_map_dev,
                           void* stream);

/*
 * Device decode of every virtual tile B in [0, total) with the same device
 * function moe_gemm uses: out_dev[5*B .. 5*B+5) = {h, task, l, rt, ct}
 * (h = non-empty task index, task = sigma(h), l = tile index in the task).
 */
moe_status moe_decode_debug(const moe_plan* plan, int32_t* out_dev, void* stream);

/* Number of SMs of the current device, and a check that it is sm_100 (MOE_OK) or not. */
moe_status moe_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* Thread-local message describing the last non-OK status ("" if none). */
const char* moe_last_error(void);

/* Library version string. */
const char* moe_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MOE_SM100_H_ */
