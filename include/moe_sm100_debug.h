/*
 * moe_sm100_debug.h — diagnostic entry points of libmoe_sm100 (not on the hot path).
 * Same conventions as moe_sm100.h.
 */
#ifndef MOE_SM100_DEBUG_H_
#define MOE_SM100_DEBUG_H_

#include "moe_sm100.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 * TMA tile::gather4 probe (the token-row staging step of moe_gemm).
 * One CTA gathers rows rows_dev[0..128) of X[T, H] (bf16), columns
 * [col0, col0 + 64), into a 1024-byte-aligned shared-memory buffer with the
 * 128-byte swizzle moe_gemm uses, and copies the raw 16 KB buffer to out_dev.
 * Expected byte layout: row r occupies bytes [128 r, 128 r + 128); its 16-byte
 * chunk c (columns 8c..8c+7) sits at chunk position c XOR (r mod 8).
 * Columns >= H read as zero.
 */
moe_status moe_probe_gather4(const void* X_dev, int64_t T, int64_t H, const int32_t* rows_dev, int32_t col0,
                             void* out_dev, void* stream);

/*
 * moe_gemm with per-CTA cycle counters (an instrumented build of the same
 * kernel; clock64() around every mbarrier wait).  prof_dev: device int64 array of
 * grid * 16 words, grid = CTAs launched (min(total tiles, SMs) for bm=128; 2*min(total, SMs/2)
 * for bm=256; 4*min(total, SMs/4) for bm=256, bn=512); per CTA:
 *   [0] MMA warp cycles waiting for a free TMEM accumulator (epilogue-bound time)
 *   [1] MMA warp cycles waiting for TMA bytes (load-bound time)
 *   [2] MMA warp cycles in its tile loop
 *   [3] producer warp 0 cycles waiting for a free stage
 *   [4] epilogue warp (TMEM lanes 0-31) cycles waiting for an accumulator
 *   [5] the same warp's cycles draining TMEM and storing Y
 *   [6] tiles processed by the CTA
 *   [7] producer warp 0 cycles in its tile loop
 *   [8] MMA warp cycles from "stage full" observed to the stage's commit issued
 *   [9] MMA warp cycles between tiles (decode + waiting for the accumulator)
 *   [10] B warp cycles waiting for a free stage    [11] B warp cycles in its tile loop
 *   [12] sum over stages of (MMA warp sees the stage full) - (B warp issued its TMA)
 *   [13] the same from A warp 0's issue of its row copies
 *   [14] sum over stages of (B warp re-issues into a slot) - (MMA committed that slot)
 *   [15] stages counted by the MMA warp
 * Results (Y) are identical to moe_gemm.
 */
moe_status moe_gemm_profile(const moe_plan* plan, const void* X_dev, int64_t T, const int32_t* token_idx_dev,
                            const void* W_dev, void* Y_dev, int32_t y_dtype, long long* prof_dev, void* stream);

/* The same counters for moe_gemm_fp8 (include/moe_sm100_fp8.h) on wide pair tiles (bm 256, bn 512);
 * other tiles: MOE_ERR_UNSUPPORTED.  Y identical to moe_gemm_fp8. */
moe_status moe_gemm_fp8_profile(const moe_plan* plan, const void* X_dev, int64_t T, const int32_t* token_idx_dev,
                                const void* W_dev, const float* scale_dev, void* Y_dev, int32_t y_dtype,
                                long long* prof_dev, void* stream);

/* Test transport for the library's expert-parallel step (include/moe_sm100_ep.h): `world`
 * handles (eps_out[world]) of one process and device that exchange rows with device copies
 * instead of NCCL, so the multi-rank orchestration of moe_ep_forward runs on one GPU.  Rank r's
 * moe_ep_forward must be called from its own host thread with its own stream, all ranks
 * concurrently (each exchange is a rendezvous of all `world` threads).  fused != 0: the GEMM
 * epilogue stores result rows straight into the owners' receive buffers (the peer-memory combine)
 * instead of a send buffer + exchange.  moe_ep_destroy each. */
typedef struct moe_ep moe_ep;
moe_status moe_ep_create_loopback(int32_t world, int32_t E, int32_t bm, int32_t bn, int32_t fused, moe_ep** eps_out);

#ifdef __cplusplus
}
#endif
#endif /* MOE_SM100_DEBUG_H_ */
