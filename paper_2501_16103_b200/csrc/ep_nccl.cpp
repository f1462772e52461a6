// The expert-parallel step in the library (include/moe_sm100_ep.h, moe_ep_*).
//
// Experts are partitioned across ranks (R8: rank g owns experts
// [g E/G, (g+1) E/G) and its own tokens).  One step moves each token row once to every rank
// owning one of its experts (deduplicated per destination), runs the single-launch expert GEMM
// there, and returns the result rows.  NCCL point-to-point calls inside ncclGroupStart/End form
// the all-to-all-v exchanges; libnccl.so.2 is resolved with dlopen so the library has no
// link-time NCCL dependency and shares the process's NCCL (PyTorch's when it is loaded).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <memory>
#include <type_traits>
#include <vector>

#include "common.h"
#include "ep_internal.h"
#include "moe_sm100_debug.h"
#include "moe_sm100_fp8.h"

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(h, name)); };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
             api.GroupEnd && api.GetErrorString;
  });
  return api;
}

#define NCCL_TRY(expr)                                                                        \
  do {                                                                                        \
    ncclResult_t r_ = (expr);                                                                 \
    if (r_ != ncclSuccess) MOE_FAIL(MOE_ERR_NCCL, "%s: %s", #expr, nccl().GetErrorString(r_)); \
  } while (0)
#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_));  \
  } while (0)
#define MOE_TRY(expr)                     \
  do {                                    \
    moe_status s_ = (expr);               \
    if (s_ < 0) return s_;                \
  } while (0)

// Stream-ordered scratch from the handle's private memory pool, released on the same stream when
// the step returns (the pool keeps the blocks: no trip to the OS at the step's synchronisation).
struct Scratch {
  cudaStream_t s;
  cudaMemPool_t pool;
  std::vector<void*> bufs;
  Scratch(cudaStream_t st, cudaMemPool_t p) : s(st), pool(p) {}
  ~Scratch() {
    for (void* p : bufs) cudaFreeAsync(p, s);
  }
  template <class T>
  T* get(size_t n, cudaError_t* err) {
    void* p = nullptr;
    *err = cudaMallocFromPoolAsync(&p, n ? n * sizeof(T) : 16, pool, s);
    if (*err == cudaSuccess) bufs.push_back(p);
    return static_cast<T*>(p);
  }
};

// A device memory pool private to one moe_ep handle, never trimmed (release threshold = max).
cudaError_t make_pool(cudaMemPool_t* pool) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  e = cudaMemPoolCreate(pool, &props);
  if (e != cudaSuccess) return e;
  uint64_t keep = UINT64_MAX;
  return cudaMemPoolSetAttribute(*pool, cudaMemPoolAttrReleaseThreshold, &keep);
}

}  // namespace

namespace moe {
// Test transport (moe_ep_create_loopback): G virtual ranks of one process on one device, each
// driven by its own host thread and stream; an exchange publishes the source buffer and its
// per-peer row counts, every rank copies its segments from the peers' buffers (after their
// "ready" events), and no rank reuses its source before every peer's copies are done.
struct Loopback {
  int G = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<const void*> src;
  std::vector<std::vector<int64_t>> send;
  std::vector<cudaEvent_t> ready, done;
  std::vector<void*> rows_base, meta_base;       // fused combine: every rank's receive buffers
  ~Loopback() {
    for (cudaEvent_t e : ready)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : done)
      if (e) cudaEventDestroy(e);
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const int64_t g = gen;
    if (++arrived == G) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
}  // namespace moe

namespace {
using moe::Loopback;

// All-to-all-v of rows: peer p gets rows [send_off[p], send_off[p] + send[p]) of `src`, this rank
// receives recv[p] rows from p at recv_off[p] of `dst` (row_bytes each).
moe_status exchange_loopback(Loopback* lb, int rank, const void* src, const std::vector<int64_t>& send, void* dst,
                             const std::vector<int64_t>& recv, int64_t row_bytes, cudaStream_t s) {
  lb->src[rank] = src;
  lb->send[rank] = send;
  CUDA_TRY(cudaEventRecord(lb->ready[rank], s));
  lb->barrier();
  int64_t ro = 0;
  for (int p = 0; p < lb->G; ++p) {
    if (recv[p]) {
      int64_t off = 0;                                 // peer p's rows for ranks before me
      for (int q = 0; q < rank; ++q) off += lb->send[p][q];
      if (lb->send[p][rank] != recv[p]) MOE_FAIL(MOE_ERR_NCCL, "loopback: size mismatch");
      CUDA_TRY(cudaStreamWaitEvent(s, lb->ready[p], 0));
      CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(dst) + ro * row_bytes,
                               static_cast<const char*>(lb->src[p]) + off * row_bytes, (size_t)(recv[p] * row_bytes),
                               cudaMemcpyDeviceToDevice, s));
    }
    ro += recv[p];
  }
  CUDA_TRY(cudaEventRecord(lb->done[rank], s));
  lb->barrier();
  for (int p = 0; p < lb->G; ++p) CUDA_TRY(cudaStreamWaitEvent(s, lb->done[p], 0));
  return MOE_OK;
}

// Every rank's stream waits for every rank's work enqueued so far (fused combine: the peers'
// GEMMs have written this rank's receive buffer).
moe_status sync_loopback(Loopback* lb, int rank, cudaStream_t s) {
  CUDA_TRY(cudaEventRecord(lb->done[rank], s));
  lb->barrier();
  for (int p = 0; p < lb->G; ++p) CUDA_TRY(cudaStreamWaitEvent(s, lb->done[p], 0));
  lb->barrier();                                   // done[] may be re-recorded only after everyone waited
  return MOE_OK;
}

moe_status exchange(const void* src, const std::vector<int64_t>& send, void* dst, const std::vector<int64_t>& recv,
                    int64_t row_bytes, void* comm_, cudaStream_t s, Loopback* lb = nullptr, int rank = 0) {
  ncclComm_t comm = static_cast<ncclComm_t>(comm_);
  if (lb) return exchange_loopback(lb, rank, src, send, dst, recv, row_bytes, s);
  const NcclApi& n = nccl();
  NCCL_TRY(n.GroupStart());
  int64_t so = 0, ro = 0;
  for (size_t p = 0; p < send.size(); ++p) {
    if (send[p])
      NCCL_TRY(n.Send(static_cast<const char*>(src) + so * row_bytes, (size_t)(send[p] * row_bytes), ncclUint8, (int)p,
                      comm, s));
    if (recv[p])
      NCCL_TRY(n.Recv(static_cast<char*>(dst) + ro * row_bytes, (size_t)(recv[p] * row_bytes), ncclUint8, (int)p, comm,
                      s));
    so += send[p];
    ro += recv[p];
  }
  NCCL_TRY(n.GroupEnd());
  return MOE_OK;
}

}  // namespace

// Pinned host staging per rank: counts [G][2], recv [G][2], recv / ret / back offsets 3 (G+1),
// back prefix [G] (int32), then peer row / tag buffer addresses [2][G] (uint64, 8-byte aligned).
inline size_t host_staging_bytes(int G) { return (size_t)4 * (4 * G + 3 * (G + 1) + G + 2) + (size_t)16 * G; }


extern "C" {

moe_status moe_ep_unique_id(void* id_out) {
  moe::clear_error();
  if (!id_out) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_unique_id: null output");
  if (!nccl().ok) MOE_FAIL(MOE_ERR_NCCL, "moe_ep_unique_id: libnccl.so.2 not loadable");
  ncclUniqueId id;
  NCCL_TRY(nccl().GetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return MOE_OK;
}

moe_status moe_ep_create(const void* unique_id, int32_t rank, int32_t world, int32_t E, int32_t bm, int32_t bn,
                         uint32_t flags, moe_ep** out) {
  moe::clear_error();
  if (!unique_id || !out) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_create: null argument");
  if (world < 1 || rank < 0 || rank >= world || E < 1 || E % world)
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_create: rank %d, world %d, E %d (E %% world must be 0)", rank, world, E);
  if (flags & ~MOE_EP_UNFUSED) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_create: unknown flags 0x%x", flags);
  if (!nccl().ok) MOE_FAIL(MOE_ERR_NCCL, "moe_ep_create: libnccl.so.2 not loadable");
  moe_ep* ep = new moe_ep;
  ep->rank = rank;
  ep->world = world;
  ep->E = E;
  ep->bm = bm;
  ep->bn = bn;
  // With one rank the combine never leaves the device: fuse it into the GEMM epilogue (moe_gemm_rowptr,
  // which has no bm = 64 decode-tile form: those tiles keep the send buffer + exchange).  Between GPUs
  // this NCCL transport exchanges result rows; the peer transport (ep_peer.cpp) maps the peers' buffers
  // and fuses the combine at every world size.
  ep->fused = world == 1 && !(flags & MOE_EP_UNFUSED) && bm != 64;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  ncclResult_t r = nccl().CommInitRank(&comm, world, id, rank);
  ep->comm = comm;
  if (r != ncclSuccess) {
    delete ep;
    MOE_FAIL(MOE_ERR_NCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r));
  }
  if (make_pool(&ep->pool) != cudaSuccess || cudaMallocHost((void**)&ep->host, host_staging_bytes(world)) != cudaSuccess ||
      cudaEventCreate(&ep->gemm_ev[0]) != cudaSuccess || cudaEventCreate(&ep->gemm_ev[1]) != cudaSuccess) {
    nccl().CommDestroy(static_cast<ncclComm_t>(ep->comm));
    if (ep->pool) cudaMemPoolDestroy(ep->pool);
    delete ep;
    MOE_FAIL(MOE_ERR_CUDA, "moe_ep_create: memory pool / pinned staging");
  }
  *out = ep;
  return MOE_OK;
}

moe_status moe_ep_forward(moe_ep* ep, const int32_t* topk, int64_t T, int32_t k, const void* X, int64_t H,
                          int32_t x_dtype, const void* W, int64_t N, const float* w_scale, void* out,
                          int32_t out_dtype, void* stream) {
  moe::NvtxRange nvtx("moe_ep_forward");
  moe::clear_error();
  if (!ep || (T > 0 && (!topk || !X || !out)) || !W) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_forward: null argument");
  if (x_dtype != MOE_DTYPE_BF16 && x_dtype != MOE_DTYPE_E4M3)
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_forward: x_dtype %d", x_dtype);
  if (out_dtype != MOE_DTYPE_BF16 && out_dtype != MOE_DTYPE_F32)
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_forward: out_dtype %d", out_dtype);
  if (T < 0 || k < 1 || k > 32 || H < 1 || N < 1) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_forward: T, k, H or N out of range");
  if (ep->peer) return moe::ep_peer_forward(ep, topk, T, k, X, H, x_dtype, W, N, w_scale, out, out_dtype,
                                            (cudaStream_t)stream);
  const int G = ep->world, El = ep->E / G;
  const int64_t x_row = H * (x_dtype == MOE_DTYPE_E4M3 ? 1 : 2);
  const int64_t y_row = N * (out_dtype == MOE_DTYPE_F32 ? 4 : 2);
  if (x_row % 16 || y_row % 16) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_forward: rows must be multiples of 16 bytes");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc(s, ep->pool);
  cudaError_t err = cudaSuccess;
  auto chk = [&]() -> moe_status {
    if (err != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_ep_forward scratch: %s", cudaGetErrorString(err));
    return MOE_OK;
  };

  // 1. dispatch plan: per-destination deduplicated rows, destination-local ids
  int32_t* counts2 = sc.get<int32_t>(2 * G, &err);
  int32_t* recv2 = sc.get<int32_t>(2 * G, &err);
  int32_t* send_off = sc.get<int32_t>(G + 1, &err);
  int32_t* send_tok = sc.get<int32_t>((size_t)G * T, &err);
  int32_t* send_meta = sc.get<int32_t>((size_t)G * T * k, &err);
  MOE_TRY(chk());
  MOE_TRY(moe_ep_dispatch_plan(topk, T, k, ep->E, G, counts2, send_off, send_tok, send_meta, s));
  // 2. counts all-to-all (2 ints per peer), one host read of the split sizes
  {
    std::vector<int64_t> two(G, 1);
    MOE_TRY(exchange(counts2, two, recv2, two, 8, ep->comm, s, ep->lb.get(), ep->rank));
  }
  int32_t* h = ep->host;
  CUDA_TRY(cudaMemcpyAsync(h, counts2, sizeof(int32_t) * 2 * G, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(h + 2 * G, recv2, sizeof(int32_t) * 2 * G, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  std::vector<int64_t> send_rows(G), back_rows(G), recv_rows(G), ret_rows(G);
  int64_t S = 0, R = 0, Rr = 0, B = 0;
  for (int p = 0; p < G; ++p) {
    send_rows[p] = h[2 * p];
    back_rows[p] = h[2 * p + 1];
    recv_rows[p] = h[2 * G + 2 * p];
    ret_rows[p] = h[2 * G + 2 * p + 1];
    S += send_rows[p];
    B += back_rows[p];
    R += recv_rows[p];
    Rr += ret_rows[p];
  }
  // 3. rows and their local ids to the owners
  char* Xs = sc.get<char>((size_t)(S * x_row), &err);
  char* Xr = sc.get<char>((size_t)(R * x_row), &err);
  int32_t* Mr = sc.get<int32_t>((size_t)(R * k), &err);
  MOE_TRY(chk());
  if (S) MOE_TRY(moe_gather_rows(X, send_tok, S, x_row, Xs, s));
  MOE_TRY(exchange(Xs, send_rows, Xr, recv_rows, x_row, ep->comm, s, ep->lb.get(), ep->rank));
  MOE_TRY(exchange(send_meta, send_rows, Mr, recv_rows, 4 * (int64_t)k, ep->comm, s, ep->lb.get(), ep->rank));
  // 4. local experts: buckets over the received rows (masked slots skipped), device plan
  int32_t* counts_l = sc.get<int32_t>(El, &err);
  int32_t* row_off_l = sc.get<int32_t>(El + 1, &err);
  int32_t* tok_l = sc.get<int32_t>((size_t)(R * k), &err);
  int32_t* slot_l = sc.get<int32_t>((size_t)(R * k), &err);
  MOE_TRY(chk());
  if (!ep->plan || ep->plan_H != H || ep->plan_N != N) {
    if (ep->plan) moe_plan_destroy(ep->plan);
    ep->plan = nullptr;
    MOE_TRY(moe_plan_create(nullptr, El, H, N, ep->bm, ep->bn, 0, s, &ep->plan));
    ep->plan_H = H;
    ep->plan_N = N;
  }
  MOE_TRY(moe_route_plan(Mr, R, k, El, counts_l, row_off_l, tok_l, slot_l, nullptr, ep->plan, s));
  // 5. where each local result row goes in the combine send buffer
  int32_t* off_h = h + 4 * G;                       // recv_off, ret_off, back_off (host, pinned)
  off_h[0] = off_h[G + 1] = off_h[2 * (G + 1)] = 0;
  for (int p = 0; p < G; ++p) {
    off_h[p + 1] = off_h[p] + (int32_t)recv_rows[p];
    off_h[G + 1 + p + 1] = off_h[G + 1 + p] + (int32_t)ret_rows[p];
    off_h[2 * (G + 1) + p + 1] = off_h[2 * (G + 1) + p] + (int32_t)back_rows[p];
  }
  int32_t* offs = sc.get<int32_t>(3 * (G + 1), &err);
  int32_t* cursor = sc.get<int32_t>(G, &err);
  if (ep->fused) {
    // 5'. fused combine: each result row goes straight into its owner's receive buffer.
    if (!ep->rows_buf || B * y_row > ep->cap_bytes || B > ep->cap_rows) {   // grow-only (stream idle here)
      if (ep->rows_buf) cudaFree(ep->rows_buf);
      if (ep->meta_buf) cudaFree(ep->meta_buf);
      ep->rows_buf = nullptr;
      ep->meta_buf = nullptr;
      ep->cap_bytes = std::max<int64_t>({B * y_row, 2 * ep->cap_bytes, 16});
      ep->cap_rows = std::max<int64_t>({B, 2 * ep->cap_rows, 4});
      CUDA_TRY(cudaMalloc((void**)&ep->rows_buf, (size_t)ep->cap_bytes));
      CUDA_TRY(cudaMalloc((void**)&ep->meta_buf, sizeof(int32_t) * (size_t)ep->cap_rows));
    }
    Loopback* lb = ep->lb.get();
    if (lb) {                                        // published before the offsets exchange (a rendezvous)
      lb->rows_base[ep->rank] = ep->rows_buf;
      lb->meta_base[ep->rank] = ep->meta_buf;
    }
    // where this rank's rows start in each owner's buffer: owner s's prefix over its sources
    int32_t* pre_h = off_h + 3 * (G + 1);
    for (int p = 0; p < G; ++p) pre_h[p] = off_h[2 * (G + 1) + p];
    int32_t* pre_d = sc.get<int32_t>(G, &err);
    int32_t* at_d = sc.get<int32_t>(G, &err);
    unsigned long long* peer_d = sc.get<unsigned long long>(2 * (size_t)G, &err);
    unsigned long long* row_ptr = sc.get<unsigned long long>((size_t)Rr, &err);
    MOE_TRY(chk());
    CUDA_TRY(cudaMemcpyAsync(offs, off_h, sizeof(int32_t) * 3 * (G + 1), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(pre_d, pre_h, sizeof(int32_t) * G, cudaMemcpyHostToDevice, s));
    {
      std::vector<int64_t> one(G, 1);
      MOE_TRY(exchange(pre_d, one, at_d, one, 4, ep->comm, s, lb, ep->rank));
    }
    unsigned long long* peer_h = reinterpret_cast<unsigned long long*>(
        (reinterpret_cast<uintptr_t>(pre_h + G) + 7) & ~uintptr_t(7));
    for (int p = 0; p < G; ++p) {
      peer_h[p] = (unsigned long long)(lb ? lb->rows_base[p] : (void*)ep->rows_buf);
      peer_h[G + p] = (unsigned long long)(lb ? lb->meta_base[p] : (void*)ep->meta_buf);
    }
    CUDA_TRY(cudaMemcpyAsync(peer_d, peer_h, sizeof(unsigned long long) * 2 * G, cudaMemcpyHostToDevice, s));
    if (Rr) {
      MOE_TRY(moe_ep_combine_ptr(tok_l, slot_l, Rr, offs, G, k, cursor, peer_d, peer_d + G, at_d, y_row, row_ptr, s));
      // 6'. the single-launch expert GEMM; its epilogue stores every row at its owner
      CUDA_TRY(cudaEventRecord(ep->gemm_ev[0], s));
      MOE_TRY(moe_gemm_rowptr(ep->plan, Xr, R, tok_l, W, x_dtype, w_scale, row_ptr, out_dtype, s));
      CUDA_TRY(cudaEventRecord(ep->gemm_ev[1], s));
    }
    ep->gemm_timed = Rr > 0;
    if (lb) MOE_TRY(sync_loopback(lb, ep->rank, s));   // the peers' GEMMs have written this rank's rows
    if (B) MOE_TRY(moe_ep_unpack(ep->rows_buf, ep->meta_buf, B, offs + 2 * (G + 1), send_off, send_tok, G, k, y_row,
                                 out, s));
    ep->sent = S;
    ep->received = R;
    ep->local_rows = Rr;
    return MOE_OK;
  }
  int32_t* row_map = sc.get<int32_t>((size_t)Rr, &err);
  int32_t* ret_meta = sc.get<int32_t>((size_t)Rr, &err);
  char* Ysend = sc.get<char>((size_t)(Rr * y_row), &err);
  MOE_TRY(chk());
  CUDA_TRY(cudaMemcpyAsync(offs, off_h, sizeof(int32_t) * 3 * (G + 1), cudaMemcpyHostToDevice, s));
  if (Rr) {
    MOE_TRY(moe_ep_combine_map(tok_l, slot_l, Rr, offs, offs + (G + 1), G, k, cursor, row_map, ret_meta, s));
    // 6. the single-launch expert GEMM, epilogue writing straight into the combine buffer
    CUDA_TRY(cudaEventRecord(ep->gemm_ev[0], s));
    if (x_dtype == MOE_DTYPE_E4M3)
      MOE_TRY(moe_gemm_fp8_rowmap(ep->plan, Xr, R, tok_l, W, w_scale, Ysend, out_dtype, row_map, s));
    else
      MOE_TRY(moe_gemm_rowmap(ep->plan, Xr, R, tok_l, W, Ysend, out_dtype, row_map, s));
    CUDA_TRY(cudaEventRecord(ep->gemm_ev[1], s));
  }
  ep->gemm_timed = Rr > 0;
  // 7. result rows (+ their (row, slot) tags) back to the token owners, then (token, slot) order
  char* Yb = sc.get<char>((size_t)(B * y_row), &err);
  int32_t* Mb = sc.get<int32_t>((size_t)B, &err);
  MOE_TRY(chk());
  MOE_TRY(exchange(Ysend, ret_rows, Yb, back_rows, y_row, ep->comm, s, ep->lb.get(), ep->rank));
  MOE_TRY(exchange(ret_meta, ret_rows, Mb, back_rows, 4, ep->comm, s, ep->lb.get(), ep->rank));
  if (B) MOE_TRY(moe_ep_unpack(Yb, Mb, B, offs + 2 * (G + 1), send_off, send_tok, G, k, y_row, out, s));
  ep->sent = S;
  ep->received = R;
  ep->local_rows = Rr;
  return MOE_OK;
}

moe_status moe_ep_create_loopback(int32_t world, int32_t E, int32_t bm, int32_t bn, int32_t fused, moe_ep** eps_out) {
  moe::clear_error();
  if (!eps_out || world < 1 || E < 1 || E % world) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_create_loopback: bad arguments");
  auto lb = std::make_shared<Loopback>();
  lb->G = world;
  lb->src.assign(world, nullptr);
  lb->send.assign(world, {});
  lb->ready.assign(world, nullptr);
  lb->done.assign(world, nullptr);
  lb->rows_base.assign(world, nullptr);
  lb->meta_base.assign(world, nullptr);
  for (int r = 0; r < world; ++r) {
    if (cudaEventCreateWithFlags(&lb->ready[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&lb->done[r], cudaEventDisableTiming) != cudaSuccess)
      MOE_FAIL(MOE_ERR_CUDA, "moe_ep_create_loopback: events");
  }
  for (int r = 0; r < world; ++r) {
    moe_ep* ep = new moe_ep;
    ep->rank = r;
    ep->world = world;
    ep->E = E;
    ep->bm = bm;
    ep->bn = bn;
    ep->lb = lb;
    ep->fused = fused != 0 && bm != 64;
    if (make_pool(&ep->pool) != cudaSuccess || cudaMallocHost((void**)&ep->host, host_staging_bytes(world)) != cudaSuccess ||
        cudaEventCreate(&ep->gemm_ev[0]) != cudaSuccess || cudaEventCreate(&ep->gemm_ev[1]) != cudaSuccess)
      MOE_FAIL(MOE_ERR_CUDA, "moe_ep_create_loopback: staging");
    eps_out[r] = ep;
  }
  return MOE_OK;
}

moe_status moe_ep_last_rows(const moe_ep* ep, int64_t* sent, int64_t* received, int64_t* local_rows) {
  moe::clear_error();
  if (!ep) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_last_rows: null handle");
  if (ep->peer) return moe::ep_peer_last_rows(ep, sent, received, local_rows);
  if (sent) *sent = ep->sent;
  if (received) *received = ep->received;
  if (local_rows) *local_rows = ep->local_rows;
  return MOE_OK;
}

moe_status moe_ep_last_gemm_ms(const moe_ep* ep, float* ms) {
  moe::clear_error();
  if (!ep || !ms) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_last_gemm_ms: null argument");
  *ms = 0.f;
  if (!ep->gemm_timed) return MOE_OK_EMPTY;
  CUDA_TRY(cudaEventSynchronize(ep->gemm_ev[1]));
  CUDA_TRY(cudaEventElapsedTime(ms, ep->gemm_ev[0], ep->gemm_ev[1]));
  return MOE_OK;
}

void moe_ep_destroy(moe_ep* ep) {
  if (!ep) return;
  if (ep->peer) moe::ep_peer_release(ep);
  for (cudaEvent_t e : ep->gemm_ev)
    if (e) cudaEventDestroy(e);
  if (ep->rows_buf) cudaFree(ep->rows_buf);
  if (ep->meta_buf) cudaFree(ep->meta_buf);
  if (ep->plan) moe_plan_destroy(ep->plan);
  if (ep->comm) nccl().CommDestroy(static_cast<ncclComm_t>(ep->comm));
  if (ep->host) cudaFreeHost(ep->host);
  if (ep->pool) {
    cudaDeviceSynchronize();                       // frees enqueued on the step streams have run
    cudaMemPoolDestroy(ep->pool);
  }
  delete ep;
}

}  // extern "C"
