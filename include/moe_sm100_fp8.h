/*
 * moe_sm100_fp8.h — the statically batched MoE expert GEMM on FP8 E4M3 operands (SURVEY §8(f)
 * row 4, "optionally FP8"; reading R15).
 *
 * The computation is the paper's per-expert product on 8-bit inputs:
 * for every CSR row i of expert e in the plan (token t = token_idx[i]),
 *     Y[i, n] = s_e * sum_h X[t, h] * W[e, h, n]          n < N,
 * where X and W hold FP8 E4M3 codes (OCP FP8: 1 sign, 4 exponent bits with bias 7, 3 mantissa bits,
 * no infinities, S.1111.111 = NaN), the products and the sum are accumulated in fp32 by
 * tcgen05.mma kind::f8f6f4 in TMEM, and s_e = scale[e] (1 if scale is NULL) multiplies the fp32
 * accumulator before the bf16 (RNE) or fp32 store.  A per-tensor activation scale is folded into
 * scale[] by the caller.  Same plan, mapping, decode and tile schedule as moe_gemm (one launch for
 * all tasks); same conventions as moe_sm100.h (plain pointers, row-major, `stream` a cudaStream_t).
 */
#ifndef MOE_SM100_FP8_H
#define MOE_SM100_FP8_H

#include "moe_sm100.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 *   plan       from moe_plan_create / moe_plan_device (host or device planned), built for (H, N).
 *              Tile shapes: 1-CTA bm = 128 with bn % 128 == 0, CTA pair bm = 256 with bn = 256, or
 *              the wide pair tile bn = 512 (the automatic choices for decode and large batches).
 *   X          [T, H] FP8 E4M3 bytes, device, 16-byte aligned, H % 16 == 0.
 *   token_idx  [sum m_e] int32 CSR token-index array (moe_route), or NULL when X's rows already are
 *              the plan's CSR rows (X then has >= sum m_e rows).
 *   W          [E, H, N] FP8 E4M3 bytes, device, 16-byte aligned, N % 128 == 0.
 *   scale      [E] fp32 device array or NULL.
 *   Y          [sum m_e, N] bf16 or fp32 (y_dtype), device, caller-owned; every valid element is
 *              written once.
 * Returns MOE_OK, MOE_OK_EMPTY (no tiles, nothing launched), MOE_ERR_INVALID (null / misaligned
 * pointer, bad T or y_dtype), MOE_ERR_UNSUPPORTED (tile shape, bm = 64 decode tiles, MOE_SPLIT_TAIL
 * plans, N % 128, H % 16), MOE_ERR_CAPACITY, MOE_ERR_CUDA.  Asynchronous: no stream synchronisation.
 */
moe_status moe_gemm_fp8(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx, const void* W,
                        const float* scale, void* Y, int32_t y_dtype, void* stream);

/*
 * As moe_gemm_fp8, but CSR row i of the plan is stored at Y row y_row_map[i] (device int32
 * [sum m_e], a permutation into Y's rows) — the expert-parallel combine send buffer
 * (include/moe_sm100_ep.h, moe_ep_combine_map), as moe_gemm_rowmap does for bf16.
 * Errors as moe_gemm_fp8, plus MOE_ERR_INVALID for a null y_row_map.
 */
moe_status moe_gemm_fp8_rowmap(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx,
                               const void* W, const float* scale, void* Y, int32_t y_dtype, const int32_t* y_row_map,
                               void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MOE_SM100_FP8_H */
