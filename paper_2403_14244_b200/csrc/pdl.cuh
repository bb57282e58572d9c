// pdl.cuh — programmatic dependent launch for the frame's kernel chain.
//
// A kernel launched with launch_pdl may become resident while its predecessor in the stream
// (or CUDA graph) is still draining its last CTAs, so the launch latency and CTA rasterisation
// of every kernel boundary overlap the predecessor's tail.  Every kernel launched this way
// calls pdl_wait() first, before it touches global memory: it returns once the predecessor
// grid has completed and its writes are visible, exactly like plain stream order.  The
// kernels also call pdl_trigger() right away, which lets their own successor launch as soon
// as every CTA of this grid has started.
#pragma once
#include <cuda_runtime.h>

#include <utility>

namespace isg {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// both, at the top of a kernel
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

// Off while per-stage event timing is on (isg_profile_enable): with an event recorded between
// every two kernels the early launch only parks CTAs and skews the per-kernel times.
inline bool g_pdl_enabled = true;

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl_enabled ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace isg
