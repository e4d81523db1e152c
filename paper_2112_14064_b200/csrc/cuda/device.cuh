// SPDX-License-Identifier: Apache-2.0
// Shared device helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../engine.hpp"

namespace rqb {

constexpr int kNB = 32;            // panel width of the blocked front LU
constexpr int kSmallNf = 160;      // fronts up to this size are factored whole in SMEM
constexpr int kPanelRowsMax = 768; // candidate rows one CTA keeps in SMEM per panel
constexpr double kPivThreshold = 0.1;   // SPEC.md:363, SURVEY App. B D2
constexpr double kSingularTiny = 1e-300;

#define RQB_CUDA(x) ::rqb::cuda_check((x), #x)

// Dynamic shared memory limit of a kernel, raised (never lowered) to `bytes`.
// The limit is per-function process state: another engine with a smaller plan
// must not lower it under a launch configured earlier, so every launch site
// calls this right before launching.
template <class Kernel>
inline void smem_at_least(Kernel kern, size_t bytes) {
  cudaFuncAttributes a{};
  RQB_CUDA(cudaFuncGetAttributes(&a, kern));
  if (static_cast<size_t>(a.maxDynamicSharedSizeBytes) < bytes)
    RQB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov > v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace rqb
