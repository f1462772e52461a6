// Internal helpers shared by the library's translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "moe_sm100.h"
#include "moe_sm100_ep.h"
#include "moe_sm100_ffn.h"

namespace moe {

void set_error(const char* fmt, ...);
void clear_error();

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Split-K of one-CTA memory-bound tiles (moe_gemm.cu): every tile's K blocks in S equal
// parts, at most kSKUnitsPerCta parts per CTA; partial accumulators of tasks of at most kSKRows rows, one
// slot per part, 256 fp32 columns per row; per-tile arrival counters for at most kSKMaxTiles tiles.  The
// plan owns the workspace (plan.cpp).
constexpr int kSKRows = 16;
constexpr int kSKCols = 256;
constexpr int kSKUnitsPerCta = 6;
constexpr int kSKMaxTiles = 1024;

// Host-side view of a plan blob (offsets into the int32 word array).
struct BlobView {
  int32_t M, total, M_pad, E, N, H, bm, bn, n_tasks;
  uint32_t flags;
  int64_t off_prefix, off_sigma, off_params, off_row_off, words;
};
bool blob_view(const int32_t* blob, int64_t len, BlobView* v);

struct moe_plan_impl;

// Load every kernel of a translation unit on the current device now (CUDA lazy loading would otherwise
// load a kernel at its first launch, which can wait for work already queued on the device — a deadlock
// when that work waits, on the device, for a peer this thread has not enqueued yet; ep_peer.cpp).
cudaError_t preload_gemm_kernels();
cudaError_t preload_route_kernels();
cudaError_t preload_ep_kernels();
cudaError_t preload_plan_kernel();

// NVTX range over a host entry point (route / plan / gemm / ep step / combine; SURVEY §5 tracing): nsys or
// ncu --nvtx attribute the launches it encloses to it.  Header-only NVTX 3: without a tool attached a
// push / pop is a call through a null-injection stub.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace moe

#define MOE_FAIL(status, ...)        \
  do {                               \
    ::moe::set_error(__VA_ARGS__);   \
    return (status);                 \
  } while (0)
