// Host-side helpers shared by the C-ABI translation units (abi.cpp, shard.cpp):
// exception -> mco_status conversion with the thread-local last-error message, and an
// RAII current-device switch.
#pragma once

#include <cuda_runtime.h>

#include <new>
#include <string>

#include "common.cuh"

namespace mco {

void set_last_error(const std::string& m);  // abi.cpp: what mco_last_error() returns

// Runs f; Error -> its status, anything else -> MCO_CUDA; the message is recorded.
template <class F>
mco_status guard(F&& f) {
  try {
    f();
    return MCO_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return MCO_CUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return MCO_CUDA;
  }
}

// device < 0 means the calling thread's current CUDA device (mco.h "device" arguments).
inline int resolve_device(int dev) {
  if (dev >= 0) return dev;
  int cur = 0;
  MCO_CUDA_CHECK(cudaGetDevice(&cur));
  return cur;
}

// RAII current-device switch.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    MCO_CUDA_CHECK(cudaGetDevice(&prev));
    if (prev != dev) MCO_CUDA_CHECK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

}  // namespace mco
