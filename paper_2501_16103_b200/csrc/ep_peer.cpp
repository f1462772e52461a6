// The expert-parallel step over symmetric peer memory (include/moe_sm100_ep.h, moe_ep_peer_*;
// SURVEY §8(e), §8(f) row 3).
//
// Experts are partitioned as in the NCCL path (R8).  Every rank owns one
// device region holding its receive buffers (token rows, destination-local ids, source token
// indices), its output rows in (token, slot) order and its epoch flags.  The region is exported
// with a CUDA IPC handle; every rank maps every other rank's region once (moe_ep_peer_connect), so
// one step needs no collective library and no host synchronisation:
//   dispatch plan -> ep_peer_dispatch: each token row stored ONCE into each owning rank's receive
//   buffer at a fixed per-source segment (rank * T_max) -> signal / wait (dispatch epoch) ->
//   moe_route_plan over the received ids (empty rows are masked, -1) -> reset the ids to -1 ->
//   ep_peer_combine_ptr: the address of every local CSR row in its token owner's output ->
//   moe_gemm_rowptr: the GEMM epilogue stores each result row there (NVLink stores between GPUs,
//   overlapping the GEMM tile by tile) -> signal / wait (combine epoch) -> optional copy into the
//   caller's buffer.
// Reuse of the receive buffers across steps is safe without a separate acknowledgement: a rank
// dispatches step n + 1 only after its own combine wait of step n, which follows every peer's step-n
// GEMM, which follows that peer's last read of its receive buffers (route, id reset, row pointers).
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "ep_internal.h"
#include "moe_sm100_fp8.h"

namespace moe {

struct PeerBlob {
  uint32_t magic, version;
  int32_t rank, world, k, device, pid, pad;
  int64_t T_max, x_cap, y_cap, bytes, hostid;
  uint64_t ptr;
  cudaIpcMemHandle_t handle;
};
static_assert(sizeof(PeerBlob) <= MOE_EP_PEER_BLOB_BYTES, "peer blob too large");
constexpr uint32_t kBlobMagic = 0x4d455042u;  // "MEPB"

struct PeerState {
  int64_t T_max = 0, x_cap = 0, y_cap = 0;
  int k = 0, device = 0;
  size_t off_tok = 0, off_meta = 0, off_x = 0, off_out = 0, bytes = 0;
  char* region = nullptr;                   // this rank's symmetric region (cudaMalloc, IPC-exported)
  std::vector<char*> bases;                 // every rank's region as mapped in this process
  std::vector<bool> opened;                 // mapped with cudaIpcOpenMemHandle (closed on release)
  PeerPtrs* peers_dev = nullptr;            // [G]
  uint32_t* epoch_dev = nullptr;            // this rank's step epoch (device: graph-capturable)
  int32_t* status_dev = nullptr;            // 0, or 2 after a wait timed out
  void* scratch = nullptr;                  // persistent step scratch (one allocation)
  int32_t *counts2 = nullptr, *send_off = nullptr, *send_tok = nullptr, *send_meta = nullptr;
  int32_t *counts_l = nullptr, *row_off_l = nullptr, *tok_l = nullptr, *slot_l = nullptr;
  unsigned long long* row_ptr = nullptr;
  PeerBlob blob = {};
  bool connected = false;
  long long timeout_ns = 60000000000LL;     // a wait gives up after 60 s (status 2), never hangs
  cudaStream_t last = nullptr;
  bool stepped = false;                     // a step has been enqueued (last may be the legacy stream 0)
};

namespace {
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
}  // namespace

moe_status ep_peer_forward(moe_ep* ep, const int32_t* topk, int64_t T, int32_t k, const void* X, int64_t H,
                           int32_t x_dtype, const void* W, int64_t N, const float* w_scale, void* out,
                           int32_t out_dtype, cudaStream_t s) {
  moe::NvtxRange nvtx("moe_ep_forward (peer)");
  PeerState& P = *ep->peer;
  if (!P.connected) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_forward: peer handle not connected (moe_ep_peer_connect)");
  const int G = ep->world, El = ep->E / G;
  const int64_t x_row = H * (x_dtype == MOE_DTYPE_E4M3 ? 1 : 2);
  const int64_t y_row = N * (out_dtype == MOE_DTYPE_F32 ? 4 : 2);
  if (x_row % 16 || y_row % 16) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_forward: rows must be multiples of 16 bytes");
  if (T > P.T_max || k != P.k || x_row > P.x_cap || y_row > P.y_cap)
    MOE_FAIL(MOE_ERR_CAPACITY, "moe_ep_forward: T %lld k %d rows %lld / %lld B exceed the peer buffers (T_max %lld, "
             "k %d, %lld / %lld B)", (long long)T, k, (long long)x_row, (long long)y_row, (long long)P.T_max, P.k,
             (long long)P.x_cap, (long long)P.y_cap);
  const int64_t R = G * P.T_max;            // receive rows (fixed segments, unused rows masked)
  char* mine = P.region;
  int32_t* meta_mine = reinterpret_cast<int32_t*>(mine + P.off_meta);
  const int32_t* tok_mine = reinterpret_cast<const int32_t*>(mine + P.off_tok);
  const uint32_t* flags_mine = reinterpret_cast<const uint32_t*>(mine);
  cudaError_t e;
#define PEER_CUDA(expr)                                                                    \
  do {                                                                                     \
    e = (expr);                                                                            \
    if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e)); \
  } while (0)
#define PEER_TRY(expr)      \
  do {                      \
    moe_status s_ = (expr); \
    if (s_ < 0) return s_;  \
  } while (0)
  // 0. host-side setup first (a plan for new H / N: host work and a small copy), before anything of this
  //    step that waits on the device for the peers is enqueued
  if (!ep->plan || ep->plan_H != H || ep->plan_N != N) {
    if (ep->plan) moe_plan_destroy(ep->plan);
    ep->plan = nullptr;
    // expected local rows: G sources x T_max tokens x k slots spread over G ranks
    PEER_TRY(moe_plan_create_expected(P.T_max * k, El, H, N, ep->bm, ep->bn, 0, s, &ep->plan));
    ep->plan_H = H;
    ep->plan_N = N;
  }
  // 1. dispatch: per-destination deduplicated rows, stored into the owners' receive buffers
  {
    moe::NvtxRange nvtx("ep_dispatch");
    PEER_TRY(moe_ep_dispatch_plan(topk, T, k, ep->E, G, P.counts2, P.send_off, P.send_tok, P.send_meta, s));
    PEER_CUDA(ep_peer_dispatch(X, x_row, P.send_off, P.send_tok, P.send_meta, G, k, ep->rank, P.T_max, P.peers_dev, s));
    if (G > 1) {                                     // one rank: stream order is the whole protocol
      PEER_CUDA(ep_peer_signal(P.peers_dev, G, ep->rank, kDispatchWord, P.epoch_dev, true, s));
      PEER_CUDA(ep_peer_wait(flags_mine, G, kDispatchWord, P.epoch_dev, P.status_dev, P.timeout_ns, s));
    }
  }
  // 2. local experts: buckets over the received ids (empty rows are -1), device plan
  PEER_TRY(moe_route_plan(meta_mine, R, k, El, P.counts_l, P.row_off_l, P.tok_l, P.slot_l, nullptr, ep->plan, s));
  PEER_CUDA(cudaMemsetAsync(meta_mine, 0xff, sizeof(int32_t) * (size_t)(R * k), s));   // next step's empty rows
  // 3. the owner-side address of every local result row, then the GEMM storing there
  PEER_CUDA(ep_peer_combine_ptr(P.row_off_l, El, P.tok_l, P.slot_l, tok_mine, P.T_max, k, P.peers_dev, y_row, R * k,
                                P.row_ptr, s));
  PEER_CUDA(cudaEventRecord(ep->gemm_ev[0], s));
  PEER_TRY(moe_gemm_rowptr(ep->plan, mine + P.off_x, R, P.tok_l, W, x_dtype, w_scale, P.row_ptr, out_dtype, s));
  PEER_CUDA(cudaEventRecord(ep->gemm_ev[1], s));
  ep->gemm_timed = true;
  // 4. every peer's GEMM has stored this rank's rows
  moe::NvtxRange nvtx_combine("ep_combine");
  if (G > 1) {
    PEER_CUDA(ep_peer_signal(P.peers_dev, G, ep->rank, kCombineWord, P.epoch_dev, false, s));
    PEER_CUDA(ep_peer_wait(flags_mine, G, kCombineWord, P.epoch_dev, P.status_dev, P.timeout_ns, s));
  }
  void* out_mine = mine + P.off_out;
  if (out && out != out_mine) PEER_CUDA(ep_peer_copy_out(out_mine, topk, T, k, y_row, out, s));
  P.last = s;
  P.stepped = true;
  ep->sent = ep->received = ep->local_rows = -1;   // on the device: moe_ep_last_rows reads them
  return MOE_OK;
#undef PEER_CUDA
#undef PEER_TRY
}

moe_status ep_peer_last_rows(const moe_ep* ep, int64_t* sent, int64_t* received, int64_t* local_rows) {
  const PeerState& P = *ep->peer;
  int32_t snd = 0, loc = 0, cnt[kPeerMaxWorld] = {};
  if (P.stepped) {
    const int G = ep->world, El = ep->E / G;
    if (cudaStreamSynchronize(P.last) != cudaSuccess ||
        cudaMemcpy(&snd, P.send_off + G, 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&loc, P.row_off_l + El, 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(cnt, reinterpret_cast<const int32_t*>(P.region) + kCountWord, 4 * (size_t)G,
                   cudaMemcpyDeviceToHost) != cudaSuccess)
      MOE_FAIL(MOE_ERR_CUDA, "moe_ep_last_rows: %s", cudaGetErrorString(cudaGetLastError()));
  }
  int64_t rcv = 0;
  for (int i = 0; i < ep->world; ++i) rcv += cnt[i];
  if (sent) *sent = snd;
  if (received) *received = rcv;
  if (local_rows) *local_rows = loc;
  return MOE_OK;
}

void ep_peer_release(moe_ep* ep) {
  PeerState& P = *ep->peer;
  cudaDeviceSynchronize();
  for (size_t i = 0; i < P.bases.size(); ++i)
    if (P.opened[i] && P.bases[i]) cudaIpcCloseMemHandle(P.bases[i]);
  if (P.region) cudaFree(P.region);
  if (P.scratch) cudaFree(P.scratch);
  if (P.peers_dev) cudaFree(P.peers_dev);
  ep->peer.reset();
}

}  // namespace moe

extern "C" {

moe_status moe_ep_peer_create(int32_t rank, int32_t world, int32_t E, int32_t bm, int32_t bn, int64_t max_tokens,
                              int32_t k, int64_t max_x_row_bytes, int64_t max_y_row_bytes, moe_ep** out,
                              void* blob_out) {
  using namespace moe;
  clear_error();
  if (!out || !blob_out) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_peer_create: null argument");
  if (world < 1 || world > kPeerMaxWorld || rank < 0 || rank >= world || E < 1 || E % world)
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_peer_create: rank %d, world %d (<= %d), E %d (E %% world must be 0)", rank, world,
             kPeerMaxWorld, E);
  if (max_tokens < 1 || k < 1 || k > 32 || max_x_row_bytes < 16 || max_x_row_bytes % 16 || max_y_row_bytes < 16 ||
      max_y_row_bytes % 16 || world * max_tokens * k >= INT32_MAX)
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_peer_create: max_tokens %lld, k %d, row bytes %lld / %lld", (long long)max_tokens,
             k, (long long)max_x_row_bytes, (long long)max_y_row_bytes);
  // the step's GEMM stores through row pointers (moe_gemm_rowptr): no bm = 64 decode-tile form; failing here
  // keeps every rank out of a step whose GEMM would fail after the dispatch (the peers would time out)
  if (bm == 64) MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_ep_peer_create: bm = 64 tiles have no row-pointer epilogue");
  auto P = std::make_shared<PeerState>();
  P->T_max = max_tokens;
  P->k = k;
  P->x_cap = max_x_row_bytes;
  P->y_cap = max_y_row_bytes;
  const int64_t R = world * max_tokens;
  P->off_tok = kFlagBytes;
  P->off_meta = align_up(P->off_tok + 4 * (size_t)R, 256);
  P->off_x = align_up(P->off_meta + 4 * (size_t)(R * k), 256);
  P->off_out = align_up(P->off_x + (size_t)(R * max_x_row_bytes), 256);
  P->bytes = align_up(P->off_out + (size_t)(max_tokens * k * max_y_row_bytes), 4096);
  auto fail = [&](const char* what, cudaError_t e) -> moe_status {
    if (P->region) cudaFree(P->region);
    if (P->scratch) cudaFree(P->scratch);
    if (P->peers_dev) cudaFree(P->peers_dev);
    MOE_FAIL(MOE_ERR_CUDA, "moe_ep_peer_create: %s: %s", what, cudaGetErrorString(e));
  };
  cudaError_t e = cudaGetDevice(&P->device);
  if (e != cudaSuccess) return fail("cudaGetDevice", e);
  // every kernel of the step loaded now: lazy loading at a later first launch could wait for this rank's
  // queued device-side waits (see common.h)
  if ((e = preload_gemm_kernels()) != cudaSuccess || (e = preload_route_kernels()) != cudaSuccess ||
      (e = preload_ep_kernels()) != cudaSuccess)
    return fail("kernel preload", e);
  if ((e = cudaMalloc((void**)&P->region, P->bytes)) != cudaSuccess) return fail("region", e);
  // scratch: epoch, status, dispatch plan, route outputs, row pointers
  const size_t n_send = (size_t)world * max_tokens;
  const size_t n_rows = (size_t)(R * k);
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t o_epoch = carve(8), o_status = carve(8), o_c2 = carve(8 * (size_t)world),
               o_soff = carve(4 * (size_t)(world + 1)), o_stok = carve(4 * n_send), o_smeta = carve(4 * n_send * k),
               o_cl = carve(4 * (size_t)(E / world)), o_rol = carve(4 * (size_t)(E / world + 1)),
               o_tl = carve(4 * n_rows), o_sl = carve(4 * n_rows), o_rp = carve(8 * n_rows);
  if ((e = cudaMalloc(&P->scratch, off)) != cudaSuccess) return fail("scratch", e);
  char* b = static_cast<char*>(P->scratch);
  P->epoch_dev = reinterpret_cast<uint32_t*>(b + o_epoch);
  P->status_dev = reinterpret_cast<int32_t*>(b + o_status);
  P->counts2 = reinterpret_cast<int32_t*>(b + o_c2);
  P->send_off = reinterpret_cast<int32_t*>(b + o_soff);
  P->send_tok = reinterpret_cast<int32_t*>(b + o_stok);
  P->send_meta = reinterpret_cast<int32_t*>(b + o_smeta);
  P->counts_l = reinterpret_cast<int32_t*>(b + o_cl);
  P->row_off_l = reinterpret_cast<int32_t*>(b + o_rol);
  P->tok_l = reinterpret_cast<int32_t*>(b + o_tl);
  P->slot_l = reinterpret_cast<int32_t*>(b + o_sl);
  P->row_ptr = reinterpret_cast<unsigned long long*>(b + o_rp);
  if ((e = cudaMalloc((void**)&P->peers_dev, sizeof(PeerPtrs) * world)) != cudaSuccess) return fail("peer table", e);
  // flags = 0 (epochs start at 1), ids = -1 (every receive row empty), epoch 0, status 0; complete
  // before the blob leaves this call, so no peer can store into an uninitialised region.
  if ((e = cudaMemset(P->region, 0, kFlagBytes)) != cudaSuccess ||
      (e = cudaMemset(P->region + P->off_meta, 0xff, 4 * n_rows)) != cudaSuccess ||
      (e = cudaMemset(P->scratch, 0, off)) != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess)
    return fail("initialisation", e);
  PeerBlob& bl = P->blob;
  std::memset(&bl, 0, sizeof(bl));
  bl.magic = kBlobMagic;
  bl.version = 1;
  bl.rank = rank;
  bl.world = world;
  bl.k = k;
  bl.device = P->device;
  bl.pid = (int32_t)getpid();
  bl.T_max = max_tokens;
  bl.x_cap = max_x_row_bytes;
  bl.y_cap = max_y_row_bytes;
  bl.bytes = (int64_t)P->bytes;
  bl.hostid = (int64_t)gethostid();
  bl.ptr = reinterpret_cast<uint64_t>(P->region);
  if ((e = cudaIpcGetMemHandle(&bl.handle, P->region)) != cudaSuccess) return fail("cudaIpcGetMemHandle", e);
  std::memset(blob_out, 0, MOE_EP_PEER_BLOB_BYTES);
  std::memcpy(blob_out, &bl, sizeof(bl));
  moe_ep* ep = new moe_ep;
  ep->rank = rank;
  ep->world = world;
  ep->E = E;
  ep->bm = bm;
  ep->bn = bn;
  ep->fused = true;
  ep->peer = P;
  if (cudaEventCreate(&ep->gemm_ev[0]) != cudaSuccess || cudaEventCreate(&ep->gemm_ev[1]) != cudaSuccess) {
    moe_ep_destroy(ep);
    MOE_FAIL(MOE_ERR_CUDA, "moe_ep_peer_create: events");
  }
  *out = ep;
  return MOE_OK;
}

moe_status moe_ep_peer_connect(moe_ep* ep, const void* blobs) {
  using namespace moe;
  clear_error();
  if (!ep || !ep->peer || !blobs) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_peer_connect: null argument or not a peer handle");
  PeerState& P = *ep->peer;
  if (P.connected) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_peer_connect: already connected");
  const int G = ep->world;
  std::vector<PeerBlob> all(G);
  for (int r = 0; r < G; ++r) {
    std::memcpy(&all[r], static_cast<const char*>(blobs) + (size_t)r * MOE_EP_PEER_BLOB_BYTES, sizeof(PeerBlob));
    const PeerBlob& q = all[r];
    if (q.magic != kBlobMagic || q.version != 1 || q.rank != r || q.world != G || q.k != P.k || q.T_max != P.T_max ||
        q.x_cap != P.x_cap || q.y_cap != P.y_cap || q.bytes != (int64_t)P.bytes)
      MOE_FAIL(MOE_ERR_INVALID, "moe_ep_peer_connect: blob %d does not match this group (rank order, world, k, "
               "max_tokens and row capacities must agree)", r);
  }
  if (std::memcmp(&all[ep->rank], &P.blob, sizeof(PeerBlob)))
    MOE_FAIL(MOE_ERR_INVALID, "moe_ep_peer_connect: blob %d is not this handle's", ep->rank);
  P.bases.assign(G, nullptr);
  P.opened.assign(G, false);
  std::vector<PeerPtrs> ptrs(G);
  for (int r = 0; r < G; ++r) {
    const PeerBlob& q = all[r];
    char* base = nullptr;
    if (r == ep->rank) {
      base = P.region;
    } else if (q.pid == P.blob.pid && q.hostid == P.blob.hostid) {
      // another handle of this process (virtual ranks on one device): the pointer is valid here
      if (q.device != P.device)
        MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_ep_peer_connect: in-process ranks must share one device");
      base = reinterpret_cast<char*>(q.ptr);
    } else {
      cudaIpcMemHandle_t h = q.handle;
      cudaError_t e = cudaIpcOpenMemHandle((void**)&base, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        for (int i = 0; i < r; ++i)
          if (P.opened[i]) cudaIpcCloseMemHandle(P.bases[i]);
        MOE_FAIL(MOE_ERR_CUDA, "moe_ep_peer_connect: cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
      }
      P.opened[r] = true;
    }
    P.bases[r] = base;
    ptrs[r].flags = reinterpret_cast<unsigned long long>(base);
    ptrs[r].tok = reinterpret_cast<unsigned long long>(base + P.off_tok);
    ptrs[r].meta = reinterpret_cast<unsigned long long>(base + P.off_meta);
    ptrs[r].x = reinterpret_cast<unsigned long long>(base + P.off_x);
    ptrs[r].out = reinterpret_cast<unsigned long long>(base + P.off_out);
  }
  cudaError_t e = cudaMemcpy(P.peers_dev, ptrs.data(), sizeof(PeerPtrs) * G, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_ep_peer_connect: peer table: %s", cudaGetErrorString(e));
  P.connected = true;
  return MOE_OK;
}

moe_status moe_ep_peer_output(const moe_ep* ep, void** out_dev, int64_t* bytes) {
  moe::clear_error();
  if (!ep || !ep->peer || !out_dev) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_peer_output: null argument or not a peer handle");
  *out_dev = ep->peer->region + ep->peer->off_out;
  if (bytes) *bytes = (int64_t)(ep->peer->bytes - ep->peer->off_out);
  return MOE_OK;
}

moe_status moe_ep_peer_set_timeout(moe_ep* ep, int64_t timeout_ns) {
  moe::clear_error();
  if (!ep || !ep->peer || timeout_ns < 1) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_peer_set_timeout: bad argument");
  ep->peer->timeout_ns = timeout_ns;
  return MOE_OK;
}

moe_status moe_ep_peer_status(moe_ep* ep, int32_t* status) {
  moe::clear_error();
  if (!ep || !ep->peer || !status) MOE_FAIL(MOE_ERR_INVALID, "moe_ep_peer_status: null argument or not a peer handle");
  moe::PeerState& P = *ep->peer;
  if (P.stepped && cudaStreamSynchronize(P.last) != cudaSuccess)
    MOE_FAIL(MOE_ERR_CUDA, "moe_ep_peer_status: %s", cudaGetErrorString(cudaGetLastError()));
  cudaError_t e = cudaMemcpy(status, P.status_dev, 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_ep_peer_status: %s", cudaGetErrorString(e));
  return MOE_OK;
}

}  // extern "C"
