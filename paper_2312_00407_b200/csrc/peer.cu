// ZeRO step fused with its collectives over NVLink peer memory -- one kernel
// instead of reduce-scatter -> update -> all-gather (parallel.cpp:656-666).
//
// Every rank maps every other rank's flat gradient buffer and flat parameter
// replica (CUDA IPC, mco_peer_*).  For its ZeroPlan-owned range [off, off+n) a
// rank's kernel:
//   g      = sum over ranks r = 0..N-1 of grads_r[off+i]   (peer loads, rank order:
//                                                          deterministic)
//   update   master / state of the owned slice (local HBM), optim.cpp arithmetic
//   params_r[off+i] = p  for every rank r                  (peer stores, f32 or bf16)
// so the reduce-scatter reads, the update and the all-gather writes of a tile
// overlap inside one pass, and no intermediate reduced-gradient buffer exists.
// NVLink bytes per rank: (N-1)/N * P * (grad bytes + replica bytes), the same
// wire volume as NCCL RS + AG.  The caller orders ranks around the launch
// (all grads final before it, nobody reads params until all ranks finished):
// PeerShardedOptimizer uses a one-element NCCL all-reduce on the stream.
#include <algorithm>

#include "kernels.h"
#include "peer.h"
#include "update.cuh"

namespace mco {
namespace {

using namespace upd;
constexpr int kThreads = 256;

__device__ __forceinline__ void ldg8(const float* g, float (&r)[8]) { ld_stream_ro(g, r); }
__device__ __forceinline__ void ldg8(const uint16_t* g, float (&r)[8]) {
  ld_stream_ro_bf16x8(g, r);
}
__device__ __forceinline__ void ldp8(const float* p, float (&r)[8]) { ld_stream(p, r); }
__device__ __forceinline__ void ldp8(const uint16_t* p, float (&r)[8]) { ld_stream_bf16x8(p, r); }
__device__ __forceinline__ float ldg1(const float* g) { return *g; }
__device__ __forceinline__ float ldg1(const uint16_t* g) { return bf2f(*g); }
__device__ __forceinline__ void st8(float* p, const float (&r)[8]) { st_stream(p, r); }
__device__ __forceinline__ void st8(uint16_t* p, const float (&r)[8]) { st_stream_bf16x8(p, r); }
__device__ __forceinline__ void st1(float* p, float v) { *p = v; }
__device__ __forceinline__ void st1(uint16_t* p, float v) { *p = (uint16_t)f2bf_bits(v); }

// Sum over ranks of one 8-element gradient vector: every peer load is issued before the
// first add (unrolled to kMaxPeers, predicated on the rank count), so the N-1 NVLink
// round trips overlap instead of serialising; the adds then run in rank order (the
// deterministic order of CommHub's reduce, comm.cpp:157-181), bit-identical to the loop.
template <typename GT>
__device__ __forceinline__ void rank_sum8(const PeerPtrs& pp, uint64_t ge, float (&g)[8]) {
  float t[kMaxPeers][8];
#pragma unroll
  for (int r = 0; r < kMaxPeers; ++r)
    if (r < pp.n) ldg8((const GT*)pp.g[r] + ge, t[r]);
#pragma unroll
  for (int j = 0; j < 8; ++j) g[j] = t[0][j];
#pragma unroll
  for (int r = 1; r < kMaxPeers; ++r)
    if (r < pp.n) {
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = g[j] + t[r][j];
    }
}
template <typename GT>
__device__ __forceinline__ float rank_sum1(const PeerPtrs& pp, uint64_t ge) {
  float t[kMaxPeers];
#pragma unroll
  for (int r = 0; r < kMaxPeers; ++r)
    if (r < pp.n) t[r] = ldg1((const GT*)pp.g[r] + ge);
  float g = t[0];
#pragma unroll
  for (int r = 1; r < kMaxPeers; ++r)
    if (r < pp.n) g = g + t[r];
  return g;
}

template <int KIND, typename GT, typename RT>
__global__ void __launch_bounds__(kThreads)
    peer_step_kernel(PeerPtrs pp, float* master, float* s0, float* s1, float* s2, float* s3,
                     uint64_t off, uint64_t nvec, uint64_t n, const StepConsts<float> k) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const int np = pp.n;
  for (uint64_t vi = tid; vi < nvec; vi += stride) {
    const uint64_t e = vi * 8, ge = off + e;
    float g[8], pv[8], a[8], b[8], c[8], d[8];
    rank_sum8<GT>(pp, ge, g);  // reduce-scatter part: peer loads, rank-order sum
    ld_stream(master + e, pv);
    ld_stream(s0 + e, a);
    if constexpr (KIND != K_LION) ld_stream(s1 + e, b);
    if constexpr (KIND == K_ADAN) {
      ld_stream(s2 + e, c);
      if (!k.first) ld_stream(s3 + e, d);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if constexpr (KIND == K_LION) b[j] = 0.f;
      if constexpr (KIND != K_ADAN) c[j] = d[j] = 0.f;
      if constexpr (KIND == K_ADAN) {
        if (k.first) d[j] = 0.f;
      }
      update<KIND, float>(pv[j], g[j], a[j], b[j], c[j], d[j], k);
    }
    st_stream(master + e, pv);
    st_stream(s0 + e, a);
    if constexpr (KIND == K_ADAMW || KIND == K_ADAN) st_stream(s1 + e, b);
    if constexpr (KIND == K_SOPHIA) {
      if (k.refresh) st_stream(s1 + e, b);
    }
    if constexpr (KIND == K_ADAN) {
      st_stream(s2 + e, c);
      st_stream(s3 + e, d);
    }
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)  // all-gather part
      if (r < np) st8((RT*)pp.p[r] + ge, pv);
  }
  for (uint64_t e = nvec * 8 + tid; e < n; e += stride) {
    const uint64_t ge = off + e;
    const float gg = rank_sum1<GT>(pp, ge);
    float pp_ = master[e], aa = s0[e], bb = 0.f, cc = 0.f, dd = 0.f;
    if constexpr (KIND != K_LION) bb = s1[e];
    if constexpr (KIND == K_ADAN) {
      cc = s2[e];
      if (!k.first) dd = s3[e];
    }
    update<KIND, float>(pp_, gg, aa, bb, cc, dd, k);
    master[e] = pp_;
    s0[e] = aa;
    if constexpr (KIND == K_ADAMW || KIND == K_ADAN) s1[e] = bb;
    if constexpr (KIND == K_SOPHIA) {
      if (k.refresh) s1[e] = bb;
    }
    if constexpr (KIND == K_ADAN) {
      s2[e] = cc;
      s3[e] = dd;
    }
    for (int r = 0; r < np; ++r) st1((RT*)pp.p[r] + ge, pp_);
  }
}

// ---- LOMO over peer memory (C5: bf16 LOMO across 8 GPUs with the global clip) ---
// pass A: sum over the owned range of (sum over ranks of g_r)^2 -> per-block fp64
// partials -> last CTA sums them in block order (deterministic);
// pass B: p_r[i] = p - f * sum_r g_r[i] for every rank's replica, f from the
// all-reduced sum of squares (optim.cpp:302-303) or lr*scale.
template <typename GT>
__global__ void __launch_bounds__(kThreads)
    peer_sumsq_kernel(PeerPtrs pp, uint64_t off, uint64_t n, double* out, double* partials,
                      unsigned* counter) {
  __shared__ double scratch[32];
  __shared__ bool is_last;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (uint64_t e = tid; e < n; e += stride) {
    const float g = rank_sum1<GT>(pp, off + e);
    acc += (double)g * (double)g;
  }
  const double b = block_sum(acc, scratch);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = b;
    __threadfence();
    is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
    double s = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) s += ((volatile double*)partials)[i];
    s = block_sum(s, scratch);
    if (threadIdx.x == 0) {
      *out = s;
      *counter = 0u;
    }
  }
}

template <typename GT, typename RT>
__global__ void __launch_bounds__(kThreads)
    peer_lomo_kernel(PeerPtrs pp, float* master, uint64_t off, uint64_t nvec, uint64_t n, double lr,
                     double scale, const double* sumsq, double clip) {
  if (sumsq) {
    const double norm = sqrt(*sumsq);
    scale = (norm > clip && norm > 0) ? clip / norm : 1.0;
  }
  const float f = (float)(lr * scale);
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t vi = tid; vi < nvec; vi += stride) {  // 8-element vectors
    const uint64_t e = vi * 8, ge = off + e;
    float g[8], p[8];
    rank_sum8<GT>(pp, ge, g);
    if (master)
      ld_stream(master + e, p);
    else
      ldp8((const RT*)pp.p[0] + ge, p);
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = p[j] - f * g[j];
    if (master) st_stream(master + e, p);
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)
      if (r < pp.n) st8((RT*)pp.p[r] + ge, p);
  }
  for (uint64_t e = nvec * 8 + tid; e < n; e += stride) {
    const float g = rank_sum1<GT>(pp, off + e);
    const float p = (master ? master[e] : ldg1((const RT*)pp.p[0] + off + e)) - f * g;
    if (master) master[e] = p;
    for (int r = 0; r < pp.n; ++r) st1((RT*)pp.p[r] + off + e, p);
  }
}

inline bool al(const void* p, size_t b) { return ((uintptr_t)p % b) == 0; }

template <int KIND, typename GT, typename RT>
void run(const PeerPtrs& pp, float* master, void* const* s, uint64_t off, uint64_t n,
         const StepConsts<float>& k, cudaStream_t st) {
  bool vec = (off % 8 == 0) && al(master, 32);
  for (int i = 0; i < 4; ++i) vec = vec && (s[i] == nullptr || al(s[i], 32));
  for (int r = 0; r < pp.n; ++r)
    vec = vec && al(pp.g[r], 8 * sizeof(GT)) && al(pp.p[r], 8 * sizeof(RT));
  const uint64_t nvec = vec ? n / 8 : 0;
  auto kern = peer_step_kernel<KIND, GT, RT>;
  int per_sm = 0;
  MCO_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0));
  const uint64_t full = (uint64_t)device_info(current_device()).sms * std::max(per_sm, 1);
  const uint64_t need = ((nvec ? nvec : n) + kThreads - 1) / kThreads;
  const int grid = (int)std::max<uint64_t>(1, std::min(full, need));
  kern<<<grid, kThreads, 0, st>>>(pp, master, (float*)s[0], (float*)s[1], (float*)s[2],
                                  (float*)s[3], off, nvec, n, k);
  launch_check("peer_step_kernel");
}

template <int KIND>
void dispatch(const PeerPtrs& pp, int gdt, int rdt, float* master, void* const* s, uint64_t off,
              uint64_t n, const StepConsts<float>& k, cudaStream_t st) {
  if (gdt == MCO_F32 && rdt == MCO_F32)
    run<KIND, float, float>(pp, master, s, off, n, k, st);
  else if (gdt == MCO_F32 && rdt == MCO_BF16)
    run<KIND, float, uint16_t>(pp, master, s, off, n, k, st);
  else if (gdt == MCO_BF16 && rdt == MCO_F32)
    run<KIND, uint16_t, float>(pp, master, s, off, n, k, st);
  else if (gdt == MCO_BF16 && rdt == MCO_BF16)
    run<KIND, uint16_t, uint16_t>(pp, master, s, off, n, k, st);
  else
    throw Error(MCO_CONTRACT, "peer step: grads / replicas must be f32 or bf16");
}

}  // namespace

void launch_peer_lomo(const PeerPtrs& pp, int grad_dtype, int replica_dtype, float* master,
                      uint64_t off, uint64_t n, double lr, double scale, const double* sumsq,
                      double clip, cudaStream_t st) {
  if (n == 0) return;
  if (pp.n < 1 || pp.n > kMaxPeers)
    throw Error(MCO_CONTRACT, "peer lomo: 1.." + std::to_string(kMaxPeers) + " ranks");
  const size_t gsz = grad_dtype == MCO_BF16 ? 2 : 4, rsz = replica_dtype == MCO_BF16 ? 2 : 4;
  bool vec = off % 8 == 0 && (master == nullptr || al(master, 32));
  for (int r = 0; r < pp.n; ++r) vec = vec && al(pp.g[r], 8 * gsz) && al(pp.p[r], 8 * rsz);
  const uint64_t nvec = vec ? n / 8 : 0;
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>(
      ((nvec ? nvec : n) + kThreads - 1) / kThreads,
      (uint64_t)device_info(current_device()).sms * 8));
  auto go = [&](auto kern) {
    kern<<<(unsigned)blocks, kThreads, 0, st>>>(pp, master, off, nvec, n, lr, scale, sumsq, clip);
    launch_check("peer_lomo_kernel");
  };
  if (grad_dtype == MCO_F32 && replica_dtype == MCO_F32)
    go(peer_lomo_kernel<float, float>);
  else if (grad_dtype == MCO_BF16 && replica_dtype == MCO_BF16)
    go(peer_lomo_kernel<uint16_t, uint16_t>);
  else if (grad_dtype == MCO_F32 && replica_dtype == MCO_BF16)
    go(peer_lomo_kernel<float, uint16_t>);
  else if (grad_dtype == MCO_BF16 && replica_dtype == MCO_F32)
    go(peer_lomo_kernel<uint16_t, float>);
  else
    throw Error(MCO_CONTRACT, "peer lomo: grads / replicas must be f32 or bf16");
}

void launch_peer_sumsq(const PeerPtrs& pp, int grad_dtype, uint64_t off, uint64_t n, double* out,
                       void* ws, cudaStream_t st) {
  double* partials = (double*)ws;
  unsigned* counter = (unsigned*)((char*)ws + 1024 * sizeof(double));
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>(
      (n + kThreads - 1) / kThreads, std::min<uint64_t>(1024, device_info(current_device()).sms * 4)));
  if (grad_dtype == MCO_F32)
    peer_sumsq_kernel<float><<<(unsigned)blocks, kThreads, 0, st>>>(pp, off, n, out, partials,
                                                                     counter);
  else if (grad_dtype == MCO_BF16)
    peer_sumsq_kernel<uint16_t><<<(unsigned)blocks, kThreads, 0, st>>>(pp, off, n, out, partials,
                                                                        counter);
  else
    throw Error(MCO_CONTRACT, "peer sumsq: grads must be f32 or bf16");
  launch_check("peer_sumsq_kernel");
}

void launch_peer_step(int kind, const PeerPtrs& pp, int grad_dtype, int replica_dtype,
                      float* master, void* const* state, uint64_t off, uint64_t n,
                      const StepConsts<float>& k, cudaStream_t st) {
  if (n == 0) return;
  if (pp.n < 1 || pp.n > kMaxPeers)
    throw Error(MCO_CONTRACT, "peer step: 1.." + std::to_string(kMaxPeers) + " ranks");
  switch (kind) {
    case MCO_ADAMW: dispatch<K_ADAMW>(pp, grad_dtype, replica_dtype, master, state, off, n, k, st); break;
    case MCO_LION: dispatch<K_LION>(pp, grad_dtype, replica_dtype, master, state, off, n, k, st); break;
    case MCO_ADAN: dispatch<K_ADAN>(pp, grad_dtype, replica_dtype, master, state, off, n, k, st); break;
    case MCO_SOPHIA: dispatch<K_SOPHIA>(pp, grad_dtype, replica_dtype, master, state, off, n, k, st); break;
    default: throw Error(MCO_CONTRACT, "peer step: fused kind");
  }
}

}  // namespace mco
