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

#ifdef __cplusplus
}
#endif
#endif /* MOE_SM100_DEBUG_H_ */
