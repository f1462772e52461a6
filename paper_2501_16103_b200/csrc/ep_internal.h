// Internal state of the expert-parallel handle (include/moe_sm100_ep.h, moe_ep_*), shared by the
// NCCL / loopback orchestration (ep_nccl.cpp) and the peer-memory transport (ep_peer.cpp).
// Not part of the ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "common.h"

namespace moe {

struct Loopback;    // ep_nccl.cpp: test transport, G virtual ranks in one process
struct PeerState;   // ep_peer.cpp: symmetric buffers mapped across processes (CUDA IPC)

// Device addresses of one rank's symmetric buffers, as mapped in THIS process (host + device).
struct PeerPtrs {
  unsigned long long x;      // [G * T_max] received token rows (row stride = the step's x row bytes)
  unsigned long long meta;   // [G * T_max, k] int32 destination-local expert ids (-1: masked / empty)
  unsigned long long tok;    // [G * T_max] int32 the source-local token index of each received row
  unsigned long long out;    // [T_max * k] result rows in (token, slot) order (stride = the step's y row bytes)
  unsigned long long flags;  // uint32 words: [kDispatchWord + s], [kCombineWord + s] epochs, [kCountWord + s] rows
};
constexpr int kPeerMaxWorld = 64;
constexpr int kDispatchWord = 0;
constexpr int kCombineWord = 128;
constexpr int kCountWord = 256;
constexpr size_t kFlagBytes = 4096;

// Peer-transport kernels (ep.cu); every launcher returns cudaGetLastError() after the launch.
cudaError_t ep_peer_dispatch(const void* X, int64_t x_row, const int32_t* send_off, const int32_t* send_tok,
                             const int32_t* send_meta, int G, int k, int rank, int64_t T_max, const PeerPtrs* peers_dev,
                             cudaStream_t s);
cudaError_t ep_peer_signal(const PeerPtrs* peers_dev, int G, int rank, int word0, uint32_t* epoch_dev, bool bump,
                           cudaStream_t s);
cudaError_t ep_peer_wait(const uint32_t* my_flags, int G, int word0, const uint32_t* epoch_dev, int32_t* status_dev,
                         long long timeout_ns, cudaStream_t s);
cudaError_t ep_peer_combine_ptr(const int32_t* row_off_l, int El, const int32_t* tok_l, const int32_t* slot_l,
                                const int32_t* recv_tok, int64_t T_max, int k, const PeerPtrs* peers_dev,
                                int64_t y_row, int64_t n_cap, unsigned long long* row_ptr, cudaStream_t s);
cudaError_t ep_peer_copy_out(const void* src, const int32_t* topk, int64_t T, int k, int64_t y_row, void* out,
                             cudaStream_t s);

}  // namespace moe

struct moe_ep {
  void* comm = nullptr;                // ncclComm_t (NCCL transport)
  int32_t rank = 0, world = 1, E = 0, bm = 0, bn = 0;
  moe_plan* plan = nullptr;            // local experts, device-planned each step
  int64_t plan_H = -1, plan_N = -1, plan_rows = -1;
  int32_t* host = nullptr;             // pinned: counts [G][2] + recv [G][2] + offsets 3 (G+1)
  int64_t sent = 0, received = 0, local_rows = 0;
  cudaEvent_t gemm_ev[2] = {nullptr, nullptr};   // around the last step's GEMM launch
  bool gemm_timed = false;
  std::shared_ptr<moe::Loopback> lb;              // test transport instead of NCCL (moe_ep_create_loopback)
  std::shared_ptr<moe::PeerState> peer;           // peer-memory transport (moe_ep_peer_create)
  // Fused combine: the GEMM epilogue stores result rows into the owners' receive buffers (this
  // rank's own with one rank; the peers' with the loopback transport).  Persistent, grow-only.
  bool fused = false;
  cudaMemPool_t pool = nullptr;                   // step scratch (private to this handle)
  char* rows_buf = nullptr;
  int32_t* meta_buf = nullptr;
  int64_t cap_bytes = 0, cap_rows = 0;
};

namespace moe {
moe_status ep_peer_forward(moe_ep* ep, const int32_t* topk, int64_t T, int32_t k, const void* X, int64_t H,
                           int32_t x_dtype, const void* W, int64_t N, const float* w_scale, void* out,
                           int32_t out_dtype, cudaStream_t s);
moe_status ep_peer_last_rows(const moe_ep* ep, int64_t* sent, int64_t* received, int64_t* local_rows);
void ep_peer_release(moe_ep* ep);
}  // namespace moe
