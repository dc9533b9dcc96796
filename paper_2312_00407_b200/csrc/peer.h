// Peer-memory (NVLink) ZeRO step: launch interface.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mco {

constexpr int kMaxPeers = 8;  // one 8x B200 NVSwitch domain

struct PeerPtrs {
  const void* g[kMaxPeers];  // every rank's flat gradient buffer (mapped)
  void* p[kMaxPeers];        // every rank's flat parameter replica (mapped)
  int n;
};

void launch_peer_step(int kind, const PeerPtrs& pp, int grad_dtype, int replica_dtype,
                      float* master, void* const* state, uint64_t off, uint64_t n,
                      const StepConsts<float>& k, cudaStream_t st);

// LOMO fused with RS / AG: optional global-norm pass (peer_sumsq) then the update
// written into every rank's replica.  master (f32, may be null -> rank 0's
// replica is read as the current parameter).  ws: sumsq_ws_bytes() workspace.
void launch_peer_sumsq(const PeerPtrs& pp, int grad_dtype, uint64_t off, uint64_t n, double* out,
                       void* ws, cudaStream_t st);
void launch_peer_lomo(const PeerPtrs& pp, int grad_dtype, int replica_dtype, float* master,
                      uint64_t off, uint64_t n, double lr, double scale, const double* sumsq,
                      double clip, cudaStream_t st);

}  // namespace mco
