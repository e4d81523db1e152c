// SPDX-License-Identifier: Apache-2.0
// Host -> device upload of large caller arrays (the K, C, M values and the
// pattern of a host pencil, rq_operator_create; the values of rq_factor_create).
// From pageable memory cudaMemcpy stages through one driver thread (about
// 11 GB/s measured on the bench host: 102 ms for cfg4_riga's 1.13 GB pencil);
// here the caller's array is copied into a ring of pinned staging buffers by
// the host threads (OpenMP, 1 MiB slices) while the copy engine drains the
// previous buffers. Pinned / registered sources go straight to the copy
// engine.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../engine.hpp"
#include "common.hpp"

namespace rqb {

namespace {

constexpr size_t kStageBytes = size_t(16) << 20;
constexpr int kStages = 4;

struct StagingRing {
  std::mutex mu;
  void* buf[kStages] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t done[kStages] = {nullptr, nullptr, nullptr, nullptr};
  bool ok = false;
  bool init() {
    if (ok) return true;
    for (int i = 0; i < kStages; ++i) {
      if (cudaMallocHost(&buf[i], kStageBytes) != cudaSuccess) return false;
      if (cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess) return false;
    }
    ok = true;
    return true;
  }
};

StagingRing& ring() {
  static StagingRing r;  // lives as long as the process (pinned memory is returned at exit)
  return r;
}

}  // namespace

void upload_host_sync(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  static const bool off = std::getenv("RQB_STAGED_UPLOAD") && std::atoi(std::getenv("RQB_STAGED_UPLOAD")) == 0;
  cudaPointerAttributes at{};
  const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();  // an unregistered pointer may leave an error state on older drivers
  StagingRing& R = ring();
  std::unique_lock<std::mutex> lock(R.mu, std::defer_lock);
  if (off || pinned || bytes < 2 * kStageBytes || (lock.lock(), !R.init())) {
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "upload");
    cuda_check(cudaStreamSynchronize(s), "upload sync");
    return;
  }
  const char* sp = static_cast<const char*>(src);
  char* dp = static_cast<char*>(dst);
  const int nt = std::max(1, host_threads());
  int k = 0;
  for (size_t o = 0; o < bytes; o += kStageBytes, ++k) {
    const int b = k % kStages;
    const size_t len = std::min(kStageBytes, bytes - o);
    if (k >= kStages) cuda_check(cudaEventSynchronize(R.done[b]), "staging wait");
    char* st = static_cast<char*>(R.buf[b]);
    const int64_t nsl = static_cast<int64_t>((len + (size_t(1) << 20) - 1) >> 20);
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t i = 0; i < nsl; ++i) {
      const size_t a = static_cast<size_t>(i) << 20;
      std::memcpy(st + a, sp + o + a, std::min(size_t(1) << 20, len - a));
    }
    cuda_check(cudaMemcpyAsync(dp + o, st, len, cudaMemcpyHostToDevice, s), "staged upload");
    cuda_check(cudaEventRecord(R.done[b], s), "staging event");
  }
  cuda_check(cudaStreamSynchronize(s), "upload sync");
}

}  // namespace rqb
