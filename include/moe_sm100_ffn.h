/*
 * moe_sm100_ffn.h — the full MoE FFN layer around the expert GEMM.
 *
 * The paper's MoE layer "selects the subset of experts for a token, then computes the products
 * of the token tensor and each selected expert weight tensor, and finally sums them up as the
 * output".  For the Mixtral-shaped expert FFN (reading R14):
 *   h   = silu(x W_gate[e]) * (x W_up[e])         moe_gemm_swiglu  (one launch, all experts)
 *   y   = h W_down[e]                             moe_gemm          (one launch, rows in CSR order)
 *   out = sum_j w[t, j] y(t, j)                   moe_combine
 * Same conventions as moe_sm100.h: plain pointers (device memory unless stated), row-major,
 * `stream` is a cudaStream_t, status codes as there.
 */
#ifndef MOE_SM100_FFN_H
#define MOE_SM100_FFN_H

#include "moe_sm100.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 * Gated first GEMM of the expert FFN: for every CSR row i of expert e (the plan's rows, token
 * token_idx[i]), Y[i, n] = silu(X[token] . W_gate[e][:, n]) * (X[token] . W_up[e][:, n]),
 * n < N, accumulated in fp32 in TMEM, silu and the product in fp32, stored bf16 (RNE) or fp32.
 * One launch of the wide pair-tile kernel: the two N = 256 accumulator blocks of a tile are the
 * same 256 columns of W_gate and W_up, and the epilogue multiplies them.
 *   plan         built for N (the FFN width I) with bm = 256, bn = 256 (else MOE_ERR_UNSUPPORTED).
 *   X [T, H], W_gate / W_up [E, H, N] bf16 row-major, 16-byte aligned; Y [sum m_e, N].
 * Errors as moe_gemm.
 */
moe_status moe_gemm_swiglu(const moe_plan* plan, const void* X, int64_t T, const int32_t* token_idx,
                           const void* W_gate, const void* W_up, void* Y, int32_t y_dtype, void* stream);

/*
 * Weighted combine ("sums them up"): out[t, :] = sum over j < k with a CSR row r(t, j) of
 * topk_w[t, j] * Y[r(t, j), :], in fp32 in ascending j (deterministic), stored bf16 (RNE) or fp32.
 * r(t, j) is recovered from moe_route's outputs: CSR row r holds token token_idx[r], slot slot[r],
 * for r < row_off[E] (read on the device; the routing need not be synchronised to the host).
 * Slots without a row (masked / invalid ids) contribute nothing; a token with none gets zeros.
 *   Y [>= row_off[E], N] bf16 or fp32 (y_dtype); topk_w [T, k] fp32; out [T, N] (out_dtype).
 *   N % 8 == 0.  Scratch: T*k int32, stream-ordered (cudaMallocAsync).
 * Returns MOE_OK, MOE_ERR_INVALID (null pointer, T < 0, k outside [1, 32], N % 8), MOE_ERR_CUDA.
 */
moe_status moe_combine(const void* Y, int32_t y_dtype, int64_t T, int32_t k, int64_t N, const int32_t* token_idx,
                       const int32_t* slot, const int32_t* row_off, int32_t E, const float* topk_w, void* out,
                       int32_t out_dtype, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MOE_SM100_FFN_H */
