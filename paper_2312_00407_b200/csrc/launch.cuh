// Launch helpers shared by the flat kernels (flat.cu, flat_list.cu): persistent
// grid-stride grids sized to the resident CTAs per SM, alignment checks.
#pragma once

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace mco {
namespace flatk {

constexpr int kThreads = 256;

// min(SMs x resident CTAs of `kernel`, CTAs needed for work_items threads).
template <typename K>
int grid_for(K kernel, uint64_t work_items, int device) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;  // kernel -> resident CTAs per SM
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find((const void*)kernel);
    if (it == cache.end()) {
      MCO_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0));
      per_sm = std::max(per_sm, 1);
      cache[(const void*)kernel] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  const uint64_t full = (uint64_t)device_info(device).sms * (uint64_t)per_sm;
  const uint64_t need = (work_items + kThreads - 1) / kThreads;
  return (int)std::max<uint64_t>(1, std::min(full, need));
}

inline bool aligned(const void* ptr, size_t bytes) {
  return ptr == nullptr || ((uintptr_t)ptr % bytes) == 0;
}

}  // namespace flatk
}  // namespace mco
