// Expert-parallel (EP) bookkeeping kernels: dispatch of token rows to the ranks that own
// their experts, and combine of expert outputs back to the tokens' owners.
//
// The paper gives EP only as background ("a subset of experts reside on each
// GPU"; per-GPU work stays irregular).  Sharding (R8): G ranks, rank g owns
// experts [g*El, (g+1)*El) and its own tokens.  A token is sent ONCE to every rank that
// owns at least one of its experts (deduplicated per destination — the token-copy
// argument of §4.3 applied across GPUs); the receiving rank runs the ordinary single-launch
// GEMM over its local experts; each (token, slot) result row returns to the token's owner.
// The collectives themselves are NCCL all-to-alls issued by the caller (torch.distributed);
// these kernels produce and consume the packed, variable-split buffers.
#include <cuda_runtime.h>

#include <climits>

#include "common.h"
#include "ep_internal.h"

namespace {

constexpr int kThreads = 1024;

__device__ __forceinline__ bool owns(int e, int d, int El) { return e >= 0 && e / El == d; }

// Slot j of a token's top-k row counts only at the first occurrence of its expert id: a repeated
// id is an invalid input that moe_route drops (R10), so dispatch must neither count nor
// forward it (the receiving rank's route would drop it and the return-row totals would disagree).
__device__ __forceinline__ bool first_slot(const int32_t* __restrict__ row, int j) {
  const int e = row[j];
  for (int i = 0; i < j; ++i)
    if (row[i] == e) return false;
  return true;
}

// Block d: rows to send to d (tokens with >= 1 slot owned by d) and result rows d returns
// (slots owned by d).
__global__ void __launch_bounds__(kThreads)
    ep_count_kernel(const int32_t* __restrict__ topk, int T, int k, int El, int32_t* __restrict__ counts2) {
  const int d = blockIdx.x;
  int rows = 0, slots = 0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    int n = 0;
    const int32_t* row = topk + (int64_t)t * k;
    for (int j = 0; j < k; ++j) n += owns(row[j], d, El) && first_slot(row, j);
    rows += n > 0;
    slots += n;
  }
  __shared__ int s_r[32], s_s[32];
  for (int o = 16; o > 0; o >>= 1) {
    rows += __shfl_xor_sync(0xffffffffu, rows, o);
    slots += __shfl_xor_sync(0xffffffffu, slots, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_r[threadIdx.x >> 5] = rows;
    s_s[threadIdx.x >> 5] = slots;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += s_r[w];
      b += s_s[w];
    }
    counts2[2 * d] = a;       // send rows to d
    counts2[2 * d + 1] = b;   // result rows d returns to me
  }
}

// Block d: stable (ascending t) compaction of the tokens sent to d into the send segment
// [send_off[d], send_off[d+1]); send_meta row = the token's k ids mapped to d-local expert
// ids (or -1 where another rank owns the slot).
__global__ void __launch_bounds__(kThreads)
    ep_scatter_kernel(const int32_t* __restrict__ topk, int T, int k, int El, int G,
                      const int32_t* __restrict__ counts2, int32_t* __restrict__ send_off,
                      int32_t* __restrict__ send_tok, int32_t* __restrict__ send_meta) {
  const int d = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  __shared__ int s_base;
  __shared__ int s_warp[32];
  if (threadIdx.x == 0) {
    int b = 0;
    for (int i = 0; i < d; ++i) b += counts2[2 * i];
    s_base = b;
    send_off[d] = b;
    if (d == G - 1) send_off[G] = b + counts2[2 * d];
  }
  __syncthreads();
  int base = s_base;
  const unsigned lt = (1u << lane) - 1u;
  for (int t0 = 0; t0 < T; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    bool hit = false;
    if (t < T)
      for (int j = 0; j < k; ++j) hit |= owns(topk[(int64_t)t * k + j], d, El);
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    int woff = 0, tot = 0;
    for (int w = 0; w < nwarps; ++w) {
      woff += w < warp ? s_warp[w] : 0;
      tot += s_warp[w];
    }
    if (hit) {
      const int pos = base + woff + __popc(m & lt);
      send_tok[pos] = t;
      const int32_t* row = topk + (int64_t)t * k;
      for (int j = 0; j < k; ++j) {
        const int e = row[j];
        send_meta[(int64_t)pos * k + j] = owns(e, d, El) && first_slot(row, j) ? e - d * El : -1;
      }
    }
    base += tot;
    __syncthreads();
  }
}

// Chunked form (round 2): block (c, d) covers tokens [c kChunkT, (c+1) kChunkT) for destination d, so the
// dispatch plan uses chunks x G blocks instead of G (one block per destination scanned every token: 22 us
// of a 0.78 ms world-1 step).  Pass 1 counts rows / slots per (chunk, destination); pass 2 derives each
// block's first send row from those counts (destinations before d, then chunks before c) and compacts its
// tokens in ascending order, exactly as ep_scatter_kernel.
constexpr int kChunkT = 1024;

__global__ void __launch_bounds__(kChunkT)
    ep_count_chunk_kernel(const int32_t* __restrict__ topk, int T, int k, int El, int G, int2* __restrict__ cc) {
  const int c = blockIdx.x, d = blockIdx.y;
  const int t = c * kChunkT + threadIdx.x;
  int rows = 0, slots = 0;
  if (t < T) {
    int n = 0;
    const int32_t* row = topk + (int64_t)t * k;
    for (int j = 0; j < k; ++j) n += owns(row[j], d, El) && first_slot(row, j);
    rows = n > 0;
    slots = n;
  }
  rows = __reduce_add_sync(0xffffffffu, rows);
  slots = __reduce_add_sync(0xffffffffu, slots);
  __shared__ int s_r[32], s_s[32];
  if ((threadIdx.x & 31) == 0) {
    s_r[threadIdx.x >> 5] = rows;
    s_s[threadIdx.x >> 5] = slots;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += s_r[w];
      b += s_s[w];
    }
    cc[(int64_t)c * G + d] = make_int2(a, b);
  }
}

__global__ void __launch_bounds__(kChunkT)
    ep_scatter_chunk_kernel(const int32_t* __restrict__ topk, int T, int k, int El, int G, int n_chunks,
                            const int2* __restrict__ cc, int32_t* __restrict__ counts2, int32_t* __restrict__ send_off,
                            int32_t* __restrict__ send_tok, int32_t* __restrict__ send_meta) {
  const int c = blockIdx.x, d = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  __shared__ int s_base, s_warp[32];
  if (warp == 0) {
    // rows of every destination < d (all chunks) + rows of d in chunks < c; totals of d for counts2
    int before = 0, tot_r = 0, tot_s = 0;
    for (int i = lane; i < n_chunks * G; i += 32) {
      const int2 v = cc[i];
      const int ci = i / G, di = i - ci * G;
      if (di < d || (di == d && ci < c)) before += v.x;
      if (di == d) {
        tot_r += v.x;
        tot_s += v.y;
      }
    }
    before = __reduce_add_sync(0xffffffffu, before);
    tot_r = __reduce_add_sync(0xffffffffu, tot_r);
    tot_s = __reduce_add_sync(0xffffffffu, tot_s);
    if (lane == 0) {
      s_base = before;
      if (c == 0) {
        send_off[d] = before;                       // chunk 0: no rows of d before it
        counts2[2 * d] = tot_r;
        counts2[2 * d + 1] = tot_s;
        if (d == G - 1) send_off[G] = before + tot_r;
      }
    }
  }
  __syncthreads();
  const int t = c * kChunkT + threadIdx.x;
  bool hit = false;
  if (t < T)
    for (int j = 0; j < k; ++j) hit |= owns(topk[(int64_t)t * k + j], d, El);
  const unsigned m = __ballot_sync(0xffffffffu, hit);
  if (lane == 0) s_warp[warp] = __popc(m);
  __syncthreads();
  int woff = 0;
  for (int w = 0; w < warp; ++w) woff += s_warp[w];
  if (hit) {
    const int pos = s_base + woff + __popc(m & ((1u << lane) - 1u));
    send_tok[pos] = t;
    const int32_t* row = topk + (int64_t)t * k;
    for (int j = 0; j < k; ++j) {
      const int e = row[j];
      send_meta[(int64_t)pos * k + j] = owns(e, d, El) && first_slot(row, j) ? e - d * El : -1;
    }
  }
  (void)nwarps;
}

// dst[i] = src[idx[i]] for rows of row_bytes (multiple of 16), one warp per row.
__global__ void gather_rows_kernel(const uint4* __restrict__ src, const int32_t* __restrict__ idx, int n,
                                   int row_vec, uint4* __restrict__ dst) {
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const uint4* s = src + (int64_t)idx[i] * row_vec;
    uint4* o = dst + (int64_t)i * row_vec;
    for (int c = threadIdx.x & 31; c < row_vec; c += 32) o[c] = s[c];
  }
}

__device__ __forceinline__ int segment_of(const int32_t* off, int G, int r) {
  int s = 0;
  while (s + 1 < G && off[s + 1] <= r) ++s;
  return s;
}

// Expert side: CSR row i (received row r = token_idx[i], slot j = slot[i]) returns to the
// source s owning r's segment of the receive buffer.  Position in the combine send buffer:
// ret_off[s] + (running count within s, any order); meta = (r - recv_off[s]) * k + j lets the
// source put the row back at (token, slot) whatever the order.
__global__ void ep_combine_map_kernel(const int32_t* __restrict__ token_idx, const int32_t* __restrict__ slot,
                                      int n, const int32_t* __restrict__ recv_off, const int32_t* __restrict__ ret_off,
                                      int G, int k, int32_t* __restrict__ cursor, int32_t* __restrict__ row_map,
                                      int32_t* __restrict__ ret_meta) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = token_idx[i];
    const int s = segment_of(recv_off, G, r);
    const int pos = ret_off[s] + atomicAdd(cursor + s, 1);
    row_map[i] = pos;
    ret_meta[pos] = (r - recv_off[s]) * k + slot[i];
  }
}

// Source side: returned row i (from destination d = segment of i in ret_off) goes to
// out[t * k + j] with t = send_tok[send_off[d] + meta / k], j = meta % k.  One warp per row.
// Fused combine (moe_ep_combine_ptr): the row's destination is a row of the token owner's receive
// buffer (peer memory), so the GEMM epilogue stores it there directly.
__global__ void ep_combine_ptr_kernel(const int32_t* __restrict__ token_idx, const int32_t* __restrict__ slot,
                                      int n, const int32_t* __restrict__ recv_off, int G, int k,
                                      int32_t* __restrict__ cursor, const unsigned long long* __restrict__ peer_rows,
                                      const unsigned long long* __restrict__ peer_meta,
                                      const int32_t* __restrict__ peer_off, long long row_bytes,
                                      unsigned long long* __restrict__ row_ptr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = token_idx[i];
    const int s = segment_of(recv_off, G, r);
    const int pos = peer_off[s] + atomicAdd(cursor + s, 1);
    row_ptr[i] = peer_rows[s] + (unsigned long long)pos * row_bytes;
    reinterpret_cast<int32_t*>(peer_meta[s])[pos] = (r - recv_off[s]) * k + slot[i];
  }
}

__global__ void ep_unpack_kernel(const uint4* __restrict__ rows, const int32_t* __restrict__ ret_meta, int n,
                                 const int32_t* __restrict__ ret_off, const int32_t* __restrict__ send_off,
                                 const int32_t* __restrict__ send_tok, int G, int k, int row_vec,
                                 uint4* __restrict__ out) {
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const int d = segment_of(ret_off, G, i);
    const int m = ret_meta[i];
    const int t = send_tok[send_off[d] + m / k];
    const uint4* s = rows + (int64_t)i * row_vec;
    uint4* o = out + ((int64_t)t * k + m % k) * row_vec;
    for (int c = threadIdx.x & 31; c < row_vec; c += 32) o[c] = s[c];
  }
}


// ---------------------------------------------------------------------------------------------
// Peer-memory transport (ep_peer.cpp): every rank's symmetric buffers are mapped in
// every process (CUDA IPC), so dispatch rows are stored straight into the owners' receive buffers
// (NVLink peer stores between GPUs), the GEMM epilogue stores result rows straight into the token
// owners' output buffers, and ranks order those stores with epoch flags (release / acquire at
// system scope) instead of host synchronisation.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Send row i (destination d = segment of i in send_off) -> row rank * T_max + (i - send_off[d]) of d's
// receive buffers: the token row (one warp, 16-byte vectors, four loads in flight per lane), its k
// destination-local ids and its source-local token index.  Block 0 also stores the row count per
// destination into the destination's count word for this source.
__global__ void __launch_bounds__(256)
    ep_peer_dispatch_kernel(const uint4* __restrict__ X, int row_vec, const int32_t* __restrict__ send_off,
                            const int32_t* __restrict__ send_tok, const int32_t* __restrict__ send_meta, int G, int k,
                            int rank, long long T_max, const moe::PeerPtrs* __restrict__ peers) {
  if (blockIdx.x == 0)
    for (int d = threadIdx.x; d < G; d += blockDim.x)
      reinterpret_cast<int32_t*>(peers[d].flags)[moe::kCountWord + rank] = send_off[d + 1] - send_off[d];
  const int S = send_off[G];
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < S; i += warps) {
    const int d = segment_of(send_off, G, i);
    const long long row = rank * T_max + (i - send_off[d]);
    const moe::PeerPtrs p = peers[d];
    const int t = send_tok[i];
    const uint4* src = X + (long long)t * row_vec;
    uint4* dst = reinterpret_cast<uint4*>(p.x) + row * row_vec;
    int c = lane;
    for (; c + 96 < row_vec; c += 128) {
      const uint4 v0 = src[c], v1 = src[c + 32], v2 = src[c + 64], v3 = src[c + 96];
      dst[c] = v0;
      dst[c + 32] = v1;
      dst[c + 64] = v2;
      dst[c + 96] = v3;
    }
    for (; c < row_vec; c += 32) dst[c] = src[c];
    if (lane < k) reinterpret_cast<int32_t*>(p.meta)[row * k + lane] = send_meta[(long long)i * k + lane];
    if (lane == 0) reinterpret_cast<int32_t*>(p.tok)[row] = t;
  }
}

// Epoch signal to every rank d: flags_d[word0 + rank] = epoch (bump: this step's new epoch).  The
// stores of the kernels before it on the stream happen-before this kernel; the system-scope fence
// and release make them visible to d before d observes the flag.
__global__ void ep_peer_signal_kernel(const moe::PeerPtrs* __restrict__ peers, int G, int rank, int word0,
                                      uint32_t* epoch, int bump) {
  __shared__ uint32_t e;
  if (threadIdx.x == 0) {
    uint32_t v = *epoch;
    if (bump) *epoch = ++v;
    e = v;
  }
  __syncthreads();
  __threadfence_system();
  for (int d = threadIdx.x; d < G; d += blockDim.x)
    st_release_sys(reinterpret_cast<uint32_t*>(peers[d].flags) + word0 + rank, e);
}

// Wait until every source s has signalled this step's epoch on flags[word0 + s] (acquire, system
// scope; wrap-safe comparison).  A peer that never signals cannot hang the stream: after timeout_ns
// the wait gives up and sets *status = 2 (moe_ep_peer_status reports it).
__global__ void ep_peer_wait_kernel(const uint32_t* flags, int G, int word0, const uint32_t* epoch, int32_t* status,
                                    long long timeout_ns) {
  const uint32_t e = *epoch;
  for (int s = threadIdx.x; s < G; s += blockDim.x) {
    const unsigned long long t0 = globaltimer_ns();
    while ((int32_t)(ld_acquire_sys(flags + word0 + s) - e) < 0) {
      if ((long long)(globaltimer_ns() - t0) > timeout_ns) {
        atomicExch(status, 2);
        break;
      }
      __nanosleep(256);
    }
  }
}

// Local CSR row i (received row r = tok_l[i], slot j = slot_l[i]) -> the address of row
// (t * k + j) in source s's output buffer, s = r / T_max, t = the source's token index of r.
__global__ void ep_peer_combine_ptr_kernel(const int32_t* __restrict__ row_off_l, int El,
                                           const int32_t* __restrict__ tok_l, const int32_t* __restrict__ slot_l,
                                           const int32_t* __restrict__ recv_tok, long long T_max, int k,
                                           const moe::PeerPtrs* __restrict__ peers, long long y_row, long long n_cap,
                                           unsigned long long* __restrict__ row_ptr) {
  const long long n = min((long long)row_off_l[El], n_cap);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = tok_l[i];
    const int s = (int)(r / T_max);
    const long long t = recv_tok[r];
    row_ptr[i] = peers[s].out + (unsigned long long)((t * k + slot_l[i]) * y_row);
  }
}

// out[t k + j] = src[t k + j] for every slot the step computed (valid id, first occurrence in the row):
// the rows of masked slots are left as the caller had them (moe_ep_forward's contract).
__global__ void ep_peer_copy_out_kernel(const uint4* __restrict__ src, const int32_t* __restrict__ topk, int n, int k,
                                        int row_vec, uint4* __restrict__ out) {
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const int32_t* row = topk + (long long)(i / k) * k;
    const int j = i % k;
    if (row[j] < 0 || !first_slot(row, j)) continue;
    const uint4* s = src + (long long)i * row_vec;
    uint4* o = out + (long long)i * row_vec;
    for (int c = threadIdx.x & 31; c < row_vec; c += 32) o[c] = s[c];
  }
}

int grid_for(int64_t warps_needed) {
  const int64_t b = (warps_needed + 7) / 8;
  return (int)(b < 1 ? 1 : (b > 4 * 148 ? 4 * 148 : b));
}

}  // namespace

namespace moe {

cudaError_t ep_peer_dispatch(const void* X, int64_t x_row, const int32_t* send_off, const int32_t* send_tok,
                             const int32_t* send_meta, int G, int k, int rank, int64_t T_max, const PeerPtrs* peers,
                             cudaStream_t s) {
  ep_peer_dispatch_kernel<<<2 * 148, 256, 0, s>>>((const uint4*)X, (int)(x_row / 16), send_off, send_tok, send_meta,
                                                   G, k, rank, T_max, peers);
  return cudaGetLastError();
}

cudaError_t ep_peer_signal(const PeerPtrs* peers, int G, int rank, int word0, uint32_t* epoch, bool bump,
                           cudaStream_t s) {
  ep_peer_signal_kernel<<<1, 64, 0, s>>>(peers, G, rank, word0, epoch, bump ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t ep_peer_wait(const uint32_t* flags, int G, int word0, const uint32_t* epoch, int32_t* status,
                         long long timeout_ns, cudaStream_t s) {
  ep_peer_wait_kernel<<<1, 64, 0, s>>>(flags, G, word0, epoch, status, timeout_ns);
  return cudaGetLastError();
}

cudaError_t ep_peer_combine_ptr(const int32_t* row_off_l, int El, const int32_t* tok_l, const int32_t* slot_l,
                                const int32_t* recv_tok, int64_t T_max, int k, const PeerPtrs* peers, int64_t y_row,
                                int64_t n_cap, unsigned long long* row_ptr, cudaStream_t s) {
  ep_peer_combine_ptr_kernel<<<2 * 148, 256, 0, s>>>(row_off_l, El, tok_l, slot_l, recv_tok, T_max, k, peers, y_row,
                                                      n_cap, row_ptr);
  return cudaGetLastError();
}

cudaError_t ep_peer_copy_out(const void* src, const int32_t* topk, int64_t T, int k, int64_t y_row, void* out,
                             cudaStream_t s) {
  if (T * k == 0) return cudaSuccess;
  ep_peer_copy_out_kernel<<<grid_for(T * k), 256, 0, s>>>((const uint4*)src, topk, (int)(T * k), k, (int)(y_row / 16),
                                                          (uint4*)out);
  return cudaGetLastError();
}

}  // namespace moe

extern "C" {

moe_status moe_ep_dispatch_plan(const int32_t* topk, int64_t T, int32_t k, int32_t E, int32_t G,
                                int32_t* counts2, int32_t* send_off, int32_t* send_tok, int32_t* send_meta,
                                void* stream) {
  moe::clear_error();
  if (G < 1 || E < 1 || E % G || k < 1 || k > 32 || T < 0 || T * k >= INT_MAX)
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_dispatch_plan: E=%d G=%d k=%d T=%lld", E, G, k, (long long)T);
  if (!counts2 || !send_off || (T > 0 && (!topk || !send_tok || !send_meta)))
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_dispatch_plan: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int El = E / G;
  cudaError_t e;
  if (T > kChunkT) {
    // chunks x G blocks (stream-ordered scratch of 2 ints per chunk and destination)
    const int n_chunks = (int)((T + kChunkT - 1) / kChunkT);
    int2* cc = nullptr;
    e = cudaMallocAsync((void**)&cc, sizeof(int2) * (size_t)n_chunks * G, s);
    if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_ep_dispatch_plan scratch: %s", cudaGetErrorString(e));
    ep_count_chunk_kernel<<<dim3(n_chunks, G), kChunkT, 0, s>>>(topk, (int)T, k, El, G, cc);
    ep_scatter_chunk_kernel<<<dim3(n_chunks, G), kChunkT, 0, s>>>(topk, (int)T, k, El, G, n_chunks, cc, counts2,
                                                                  send_off, send_tok, send_meta);
    cudaFreeAsync(cc, s);
  } else {
    ep_count_kernel<<<G, kThreads, 0, s>>>(topk, (int)T, k, El, counts2);
    ep_scatter_kernel<<<G, kThreads, 0, s>>>(topk, (int)T, k, El, G, counts2, send_off, send_tok, send_meta);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_ep_dispatch_plan launch: %s", cudaGetErrorString(e));
  return MOE_OK;
}

moe_status moe_gather_rows(const void* src, const int32_t* idx, int64_t n, int64_t row_bytes, void* dst,
                           void* stream) {
  moe::clear_error();
  if (n == 0) return MOE_OK;
  if (!src || !idx || !dst || n < 0 || n >= INT_MAX) MOE_FAIL(MOE_ERR_INVALID, "moe_gather_rows: bad argument");
  if (row_bytes <= 0 || row_bytes % 16 || (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    MOE_FAIL(MOE_ERR_INVALID, "moe_gather_rows: rows and pointers must be 16-byte multiples/aligned");
  gather_rows_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      (const uint4*)src, idx, (int)n, (int)(row_bytes / 16), (uint4*)dst);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_gather_rows launch: %s", cudaGetErrorString(e));
  return MOE_OK;
}

moe_status moe_ep_combine_map(const int32_t* token_idx, const int32_t* slot, int64_t n, const int32_t* recv_off,
                              const int32_t* ret_off, int32_t G, int32_t k, int32_t* cursor, int32_t* row_map,
                              int32_t* ret_meta, void* stream) {
  moe::clear_error();
  if (n == 0) return MOE_OK;
  if (!token_idx || !slot || !recv_off || !ret_off || !cursor || !row_map || !ret_meta || G < 1 || k < 1 ||
      n < 0 || n >= INT_MAX)
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_combine_map: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(cursor, 0, sizeof(int32_t) * G, s);
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_ep_combine_map memset: %s", cudaGetErrorString(e));
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 4 * 148);
  ep_combine_map_kernel<<<blocks, 256, 0, s>>>(token_idx, slot, (int)n, recv_off, ret_off, G, k, cursor, row_map,
                                               ret_meta);
  e = cudaGetLastError();
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_ep_combine_map launch: %s", cudaGetErrorString(e));
  return MOE_OK;
}

moe_status moe_ep_combine_ptr(const int32_t* token_idx, const int32_t* slot, int64_t n, const int32_t* recv_off,
                              int32_t G, int32_t k, int32_t* cursor, const unsigned long long* peer_rows,
                              const unsigned long long* peer_meta, const int32_t* peer_off, int64_t row_bytes,
                              unsigned long long* row_ptr, void* stream) {
  moe::clear_error();
  if (n == 0) return MOE_OK;
  if (!token_idx || !slot || !recv_off || !cursor || !peer_rows || !peer_meta || !peer_off || !row_ptr || G < 1 || k < 1 ||
      n < 0 || n >= INT_MAX || row_bytes <= 0 || row_bytes % 16)
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_combine_ptr: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(cursor, 0, sizeof(int32_t) * G, s);
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_ep_combine_ptr memset: %s", cudaGetErrorString(e));
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 4 * 148);
  ep_combine_ptr_kernel<<<blocks, 256, 0, s>>>(token_idx, slot, (int)n, recv_off, G, k, cursor, peer_rows, peer_meta,
                                               peer_off, row_bytes, row_ptr);
  e = cudaGetLastError();
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_ep_combine_ptr launch: %s", cudaGetErrorString(e));
  return MOE_OK;
}

moe_status moe_ep_unpack(const void* rows, const int32_t* ret_meta, int64_t n, const int32_t* ret_off,
                         const int32_t* send_off, const int32_t* send_tok, int32_t G, int32_t k, int64_t row_bytes,
                         void* out, void* stream) {
  moe::clear_error();
  if (n == 0) return MOE_OK;
  if (!rows || !ret_meta || !ret_off || !send_off || !send_tok || !out || G < 1 || k < 1 || n < 0 || n >= INT_MAX)
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_unpack: bad argument");
  if (row_bytes <= 0 || row_bytes % 16 || (reinterpret_cast<uintptr_t>(rows) | reinterpret_cast<uintptr_t>(out)) & 15)
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_unpack: rows and pointers must be 16-byte multiples/aligned");
  ep_unpack_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      (const uint4*)rows, ret_meta, (int)n, ret_off, send_off, send_tok, G, k, (int)(row_bytes / 16), (uint4*)out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_ep_unpack launch: %s", cudaGetErrorString(e));
  return MOE_OK;
}

}  // extern "C"

cudaError_t moe::preload_ep_kernels() {
  cudaFuncAttributes fa;
  const void* ks[] = {(const void*)ep_count_kernel, (const void*)ep_scatter_kernel, (const void*)ep_count_chunk_kernel,
                      (const void*)ep_scatter_chunk_kernel, (const void*)gather_rows_kernel,
                      (const void*)ep_combine_map_kernel, (const void*)ep_combine_ptr_kernel, (const void*)ep_unpack_kernel,
                      (const void*)ep_peer_dispatch_kernel, (const void*)ep_peer_signal_kernel,
                      (const void*)ep_peer_wait_kernel, (const void*)ep_peer_combine_ptr_kernel,
                      (const void*)ep_peer_copy_out_kernel};
  for (const void* k : ks) {
    const cudaError_t e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
