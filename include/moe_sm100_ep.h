/*
 * moe_sm100_ep.h — expert-parallel (EP) bookkeeping kernels of libmoe_sm100.
 *
 * Expert parallelism is background in the paper ("a subset of experts reside on
 * each GPU"; the per-GPU work remains an irregular batch).  Sharding (R8): G ranks,
 * rank g owns experts [g*E/G, (g+1)*E/G) and its own tokens.  One EP step:
 *   1. moe_ep_dispatch_plan  per destination d: the owned tokens with >= 1 expert on d
 *                            (deduplicated, ascending token), their d-local expert ids;
 *   2. NCCL all-to-all of the counts (caller), moe_gather_rows + all-to-all of the rows;
 *   3. on every rank: moe_route over the received rows' local ids (-1 = masked slot),
 *      moe_plan_device, moe_gemm_rowmap writing each result row straight into the combine
 *      send buffer at the position moe_ep_combine_map chose;
 *   4. all-to-all of the result rows back (caller), moe_ep_unpack into (token, slot) order.
 * Same conventions as moe_sm100.h (device pointers, void* stream, no synchronisation).
 */
#ifndef MOE_SM100_EP_H_
#define MOE_SM100_EP_H_

#include "moe_sm100.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 * topk_dev [T, k] int32 global expert ids of this rank's tokens (negative = masked), E % G == 0.
 * Out (device):
 *   counts2_dev [G][2]   {rows sent to d, result rows d will return} — exchanged by the caller
 *                        with one all-to-all of 2 ints per peer;
 *   send_off_dev [G+1]   exclusive prefix of rows sent per destination;
 *   send_tok_dev [<= G*T] local token index of each send row (destination-major, ascending t);
 *   send_meta_dev [<= G*T, k] the row's k ids mapped to destination-local expert ids, -1 where
 *                        another rank owns the slot.
 * Two kernel launches.
 */
moe_status moe_ep_dispatch_plan(const int32_t* topk_dev, int64_t T, int32_t k, int32_t E, int32_t G,
                                int32_t* counts2_dev, int32_t* send_off_dev, int32_t* send_tok_dev,
                                int32_t* send_meta_dev, void* stream);

/* dst_dev[i, :] = src_dev[idx_dev[i], :] for n rows of row_bytes (a multiple of 16, 16-byte aligned). */
moe_status moe_gather_rows(const void* src_dev, const int32_t* idx_dev, int64_t n, int64_t row_bytes,
                           void* dst_dev, void* stream);

/*
 * Expert side.  For the n CSR rows of moe_route over the received rows (token_idx_dev: received
 * row r, slot_dev: top-k slot j), recv_off_dev [G+1]: segment of received rows per source,
 * ret_off_dev [G+1]: segment of the combine send buffer per source.  Out: row_map_dev[i] =
 * position of CSR row i in the combine send buffer (any order within a source's segment;
 * pass it to moe_gemm_rowmap), ret_meta_dev[pos] = (r - recv_off[s]) * k + j.  cursor_dev:
 * [G] int32 scratch.
 */
moe_status moe_ep_combine_map(const int32_t* token_idx_dev, const int32_t* slot_dev, int64_t n,
                              const int32_t* recv_off_dev, const int32_t* ret_off_dev, int32_t G, int32_t k,
                              int32_t* cursor_dev, int32_t* row_map_dev, int32_t* ret_meta_dev, void* stream);

/*
 * Fused combine (the GEMM epilogue writes each result row straight into the token owner's receive
 * buffer, over NVLink peer memory between GPUs).  For the n CSR rows (token_idx_dev / slot_dev as
 * moe_ep_combine_map, recv_off_dev [G+1]): with source s = the segment of row r, and pos = a slot
 * among s's rows (any order) plus peer_off_dev[s], row_ptr_dev[i] = peer_rows_dev[s] + pos * row_bytes
 * and ((int32_t*)peer_meta_dev[s])[pos] = (r - recv_off[s]) * k + j.  peer_rows_dev / peer_meta_dev:
 * [G] device arrays of the owners' row / tag buffer addresses; peer_off_dev [G] int32: where this
 * rank's segment starts in owner s's buffers.
 * cursor_dev: [G] int32 scratch.  Pass row_ptr_dev to moe_gemm_rowptr.
 */
moe_status moe_ep_combine_ptr(const int32_t* token_idx_dev, const int32_t* slot_dev, int64_t n,
                              const int32_t* recv_off_dev, int32_t G, int32_t k, int32_t* cursor_dev,
                              const unsigned long long* peer_rows_dev, const unsigned long long* peer_meta_dev,
                              const int32_t* peer_off_dev, int64_t row_bytes, unsigned long long* row_ptr_dev,
                              void* stream);

/*
 * The expert GEMM (moe_gemm / moe_gemm_fp8 by x_dtype: MOE_DTYPE_BF16 or MOE_DTYPE_E4M3 (2), with
 * the optional per-expert scale for E4M3) storing CSR row i at the device address y_row_ptr_dev[i]
 * (N values of y_dtype, 16-byte aligned; any memory the GPU can write, e.g. a peer's buffer).
 * Plain, pair and wide tiles; MOE_ERR_UNSUPPORTED for bm = 64 and MOE_SPLIT_TAIL plans.
 */
moe_status moe_gemm_rowptr(const moe_plan* plan, const void* X_dev, int64_t T, const int32_t* token_idx_dev,
                           const void* W_dev, int32_t x_dtype, const float* scale_dev,
                           const unsigned long long* y_row_ptr_dev, int32_t y_dtype, void* stream);

/*
 * Source side.  rows_dev: n returned result rows (segment per destination given by
 * ret_off_dev [G+1]) with their ret_meta_dev; send_off_dev / send_tok_dev from
 * moe_ep_dispatch_plan.  out_dev[t * k + j, :] = the returned row of (token t, slot j).
 */
moe_status moe_ep_unpack(const void* rows_dev, const int32_t* ret_meta_dev, int64_t n, const int32_t* ret_off_dev,
                         const int32_t* send_off_dev, const int32_t* send_tok_dev, int32_t G, int32_t k,
                         int64_t row_bytes, void* out_dev, void* stream);

/* ------------------------------------------------------------------------------------------
 * The whole expert-parallel step in the library (SURVEY §8(b) moe_ep_*): NCCL is called from
 * C++ (libnccl.so.2 resolved at run time with dlopen — the one the process already loaded, e.g.
 * PyTorch's; no link-time dependency); the host only bootstraps the 128-byte unique id.
 * Per step, on `stream`: moe_ep_dispatch_plan -> grouped ncclSend/ncclRecv of the 2-int counts
 * -> ONE stream synchronisation (the split sizes, as the all-to-all-v needs them on the host) ->
 * moe_gather_rows + grouped send/recv of rows and local-id metadata -> moe_route + moe_plan_device
 * on the received rows -> moe_ep_combine_map -> moe_gemm_rowmap / moe_gemm_fp8_rowmap into the
 * combine send buffer -> grouped send/recv of result rows + metadata -> moe_ep_unpack.
 * Scratch is stream-ordered (cudaMallocAsync / cudaFreeAsync); the handle owns the NCCL
 * communicator, a device plan for the local experts and pinned host staging.
 * ------------------------------------------------------------------------------------------ */
#define MOE_DTYPE_E4M3 2          /* x_dtype of moe_ep_forward: FP8 E4M3 rows and weights */

typedef struct moe_ep moe_ep;     /* opaque, library-owned */

/* Writes a fresh NCCL unique id (128 bytes) to id_out (host); rank 0 calls it, the caller
 * broadcasts it.  MOE_ERR_NCCL when libnccl.so.2 cannot be loaded or fails. */
moe_status moe_ep_unique_id(void* id_out);

/* moe_ep_create flags. */
#define MOE_EP_UNFUSED 1u   /* one rank: return result rows through the send buffer + exchange instead
                               of storing them from the GEMM epilogue into the receive buffer (A/B) */

/* Collective over `world` ranks (blocking until all joined): communicator for this rank.
 * E % world == 0 experts; rank g owns experts [g E/world, (g+1) E/world).  bm / bn: the local
 * GEMM's tile shape (0: the planner's choice).  flags: MOE_EP_* above.  The calling thread's
 * current CUDA device is used.  Step scratch comes from a memory pool owned by the handle. */
moe_status moe_ep_create(const void* unique_id, int32_t rank, int32_t world, int32_t E, int32_t bm, int32_t bn,
                         uint32_t flags, moe_ep** out);

/*
 * One step.  topk_dev [T, k] int32 global expert ids of this rank's T tokens (negative = masked);
 * X_dev [T, H] (x_dtype MOE_DTYPE_BF16 or MOE_DTYPE_E4M3); W_dev [E/world, H, N] of the same
 * type (this rank's experts); w_scale_dev [E/world] fp32 (E4M3 only, nullable);
 * out_dev [T k, N] of out_dtype (MOE_DTYPE_BF16 / MOE_DTYPE_F32): out[t k + j] = the product of
 * token t with expert topk[t, j] (rows of masked slots are not written).
 * Returns MOE_OK, MOE_ERR_INVALID, MOE_ERR_UNSUPPORTED (as the GEMMs), MOE_ERR_CUDA, MOE_ERR_NCCL.
 */
moe_status moe_ep_forward(moe_ep* ep, const int32_t* topk_dev, int64_t T, int32_t k, const void* X_dev, int64_t H,
                          int32_t x_dtype, const void* W_dev, int64_t N, const float* w_scale_dev, void* out_dev,
                          int32_t out_dtype, void* stream);

/* Row counts of the last step: sent (dispatch), received (dispatch), local expert rows (GEMM). */
moe_status moe_ep_last_rows(const moe_ep* ep, int64_t* sent, int64_t* received, int64_t* local_rows);

/* Device time of the last step's GEMM launch (CUDA events recorded around it on the step's
 * stream; waits for the second one).  MOE_OK_EMPTY (0 ms) when the rank had no local rows. */
moe_status moe_ep_last_gemm_ms(const moe_ep* ep, float* ms);

/* Releases the handle (either transport).  Peer handles: every rank must have finished its last step
 * (synchronise, then a barrier of the caller's) before any rank destroys, since peers store into
 * this rank's region. */
void moe_ep_destroy(moe_ep* ep);

/* ------------------------------------------------------------------------------------------
 * The same step over symmetric peer memory (no collective library, no host synchronisation).
 * Each rank allocates one device region: receive buffers for max_tokens rows from every rank
 * (fixed segment per source), its output rows in (token, slot) order, epoch flags.  The region is
 * exported as a CUDA IPC handle inside a MOE_EP_PEER_BLOB_BYTES blob; the caller all-gathers the
 * blobs (plumbing, e.g. torch.distributed) and every rank maps every peer's region once
 * (moe_ep_peer_connect; ranks of one process on one device use the pointers directly).  A step on
 * `stream` (moe_ep_forward on a peer handle):
 *   moe_ep_dispatch_plan -> each token row stored once into each owning rank's receive buffer
 *   (NVLink peer stores between GPUs) -> release/acquire epoch flags at system scope -> moe_route_plan
 *   over the received ids -> the single-launch GEMM whose epilogue stores every result row straight
 *   into its token owner's output (moe_gemm_rowptr: the combine overlaps the GEMM tile by tile) ->
 *   epoch flags -> a copy of the computed rows into out_dev (skipped when out_dev is the handle's own
 *   output, moe_ep_peer_output: zero copy; its rows stay valid until the next step).
 * Every call is stream-ordered and host-synchronisation-free (CUDA-graph capturable).  All ranks run
 * the same number of steps with the same k, H, N, dtypes; T <= max_tokens per rank and step.  Ranks
 * driven from one process need one stream each (a rank's step waits on the device for its peers').
 * A rank whose peer never signals does not hang: its waits give up after the timeout (default 60 s,
 * moe_ep_peer_set_timeout) and moe_ep_peer_status reports 2.  P:94-98 (EP background), DESIGN.md §9.
 * ------------------------------------------------------------------------------------------ */
#define MOE_EP_PEER_BLOB_BYTES 256

/* Collective-free local part of the setup.  E % world == 0 (world <= 64); bm / bn: the local GEMM's
 * tile shape (0: the planner's choice for max_tokens * k expected rows); max_x_row_bytes /
 * max_y_row_bytes: capacities of a token row (H * 2 bf16, H E4M3) and a result row (N * 2 bf16,
 * N * 4 fp32), multiples of 16.  Writes this rank's blob (MOE_EP_PEER_BLOB_BYTES, host) to blob_out.
 * The region (world * max_tokens * (max_x_row_bytes + 4 k + 4) + max_tokens * k * max_y_row_bytes bytes)
 * is initialised before the call returns.  The calling thread's current device is used. */
moe_status moe_ep_peer_create(int32_t rank, int32_t world, int32_t E, int32_t bm, int32_t bn, int64_t max_tokens,
                              int32_t k, int64_t max_x_row_bytes, int64_t max_y_row_bytes, moe_ep** out,
                              void* blob_out);

/* blobs: world * MOE_EP_PEER_BLOB_BYTES bytes (host), rank order (the all-gather of every rank's blob).
 * Maps the peers' regions (cudaIpcOpenMemHandle, peer access enabled lazily).  MOE_ERR_INVALID when a
 * blob does not belong to this group. */
moe_status moe_ep_peer_connect(moe_ep* ep, const void* blobs);

/* The handle's output rows (device; row t * k + j of the step's result row bytes) and their capacity. */
moe_status moe_ep_peer_output(const moe_ep* ep, void** out_dev, int64_t* bytes);

/* Timeout of the device-side waits, in ns (default 60 s). */
moe_status moe_ep_peer_set_timeout(moe_ep* ep, int64_t timeout_ns);

/* Synchronises the last step's stream; *status = 0, or 2 if a wait timed out (results invalid). */
moe_status moe_ep_peer_status(moe_ep* ep, int32_t* status);

#ifdef __cplusplus
}
#endif
#endif /* MOE_SM100_EP_H_ */
