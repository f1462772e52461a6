// Device-side planner: device-resident expert token counts -> the compressed mapping,
// written in place into the plan's device blob by ONE single-block kernel launch.
//
// P:142 "this can be either pre-computed on the host and then copied to the device, or
// directly generated on the device"; "the prefix sum can be computed with parallel
// implementation".  Same arithmetic as moe_plan_build (Alg. 1 over the non-empty tasks of
// Alg. 4's extra stage; padding P:203), as block-wide scans: one thread per
// expert.  The blob layout is the header file's, with M_pad fixed at pad32(E) so the
// layout does not depend on the counts (the GEMM can be launched without knowing them).
#include <cuda_runtime.h>

#include <climits>

#include "common.h"
#include "plan_body.cuh"

namespace moe {
bool plan_device_mode(const moe_plan* p);
void plan_set_device_mode(moe_plan* p, bool on);
void plan_shape(const moe_plan* p, int32_t* E, int32_t* H, int32_t* N, int32_t* bm, int32_t* bn, uint32_t* flags);
int32_t* plan_blob_dev_mut(moe_plan* p);
}  // namespace moe

namespace {

using moe::dplan::kPlanThreads;

__global__ void __launch_bounds__(kPlanThreads)
    plan_device_kernel(const int32_t* __restrict__ counts, int E, int H, int N, int bm, int bn, uint32_t flags,
                       int32_t* __restrict__ blob) {
  const int t = threadIdx.x;
  moe::dplan::plan_body(t < E ? (long long)max(counts[t], 0) : 0, E, H, N, bm, bn, flags, blob);
}

}  // namespace

extern "C" moe_status moe_plan_device(moe_plan* plan, const int32_t* counts_dev, void* stream) {
  moe::NvtxRange nvtx("moe_plan_device");
  moe::clear_error();
  if (!plan || !counts_dev) MOE_FAIL(MOE_ERR_INVALID, "moe_plan_device: null argument");
  int32_t E, H, N, bm, bn;
  uint32_t flags;
  moe::plan_shape(plan, &E, &H, &N, &bm, &bn, &flags);
  if (E > kPlanThreads) MOE_FAIL(MOE_ERR_UNSUPPORTED, "moe_plan_device: E=%d > %d", E, kPlanThreads);
  plan_device_kernel<<<1, kPlanThreads, 0, (cudaStream_t)stream>>>(counts_dev, E, H, N, bm, bn, flags,
                                                                   moe::plan_blob_dev_mut(plan));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) MOE_FAIL(MOE_ERR_CUDA, "moe_plan_device launch: %s", cudaGetErrorString(e));
  moe::plan_set_device_mode(plan, true);
  return MOE_OK;
}

cudaError_t moe::preload_plan_kernel() {
  cudaFuncAttributes fa;
  return cudaFuncGetAttributes(&fa, (const void*)plan_device_kernel);
}
