// Internals shared by the C-ABI translation units (abi.cpp: common entry points and
// helpers; abi_flat.cpp: FlatOptimizer, LOMO, peer-memory ZeRO; abi_adalomo.cpp:
// AdaLomoState).  Not part of the public interface (include/mco.h).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "abi_util.h"
#include "adalomo.h"
#include "kernels.h"
#include "mco.h"
#include "peer.h"
#include "update.cuh"

namespace mco {

const char* kind_cstr(int kind);       // optim.cpp:17-28
std::string kind_str(int kind);        // throws CONFIG on an unknown kind
bool fused(int kind);                  // optim.cpp:30
mco_config defaults(int kind);         // optim.cpp:32-61
void validate(const mco_config& c);    // optim.cpp:63-70
size_t dtype_size(int dt);
void* sumsq_ws(cudaStream_t st);       // per (device, stream) sum-of-squares workspace

// sqrt_plus_eps (update.cuh): the largest x with RN(sqrt(RN(x / c)) + eps) == eps
// guaranteed, (ulp(eps)/4)^2 * c rounded down; fp32 only (0 = no shortcut).
template <typename T>
T sqrt_eps_threshold(T eps, T c) {
  if constexpr (sizeof(T) == 4) {
    if (!(eps > 0) || !std::isnormal(eps) || !(c > 0)) return 0;
    const double q = ((double)std::nextafter(eps, INFINITY) - (double)eps) / 4.0;
    const double thr = q * q * (double)c;
    float f = (float)thr;
    if ((double)f > thr) f = std::nextafter(f, 0.0f);
    return f;
  } else {
    return 0;
  }
}

// The multiply form sqrt(x * rc) + eps (fp32 Adan): x < thr guarantees RN(x * rc) <=
// (ulp(eps)/4)^2, so RN(sqrt(.) + eps) == eps -- thr = (ulp(eps)/4)^2 / rc rounded down
// with a 2^-20 margin.
template <typename T>
T sqrt_eps_threshold_mul(T eps, T rc) {
  if constexpr (sizeof(T) == 4) {
    if (!(eps > 0) || !std::isnormal(eps) || !(rc > 0)) return 0;
    const double q = ((double)std::nextafter(eps, INFINITY) - (double)eps) / 4.0;
    const double thr = q * q / (double)rc * (1.0 - std::ldexp(1.0, -20));
    float f = (float)thr;
    if ((double)f > thr) f = std::nextafter(f, 0.0f);
    return f;
  } else {
    return 0;
  }
}

template <typename T>
StepConsts<T> make_consts(const mco_config& c, int64_t t, double lr) {
  StepConsts<T> k{};
  k.b1 = (T)c.beta1;
  k.b2 = (T)c.beta2;
  k.b3 = (T)c.beta3;
  k.omb1 = (T)(1 - c.beta1);
  k.omb2 = (T)(1 - c.beta2);
  k.omb3 = (T)(1 - c.beta3);
  k.c1 = (T)(1.0 - std::pow(c.beta1, static_cast<double>(t)));
  k.c2 = (T)(1.0 - std::pow(c.beta2, static_cast<double>(t)));
  k.c3 = (T)(1.0 - std::pow(c.beta3, static_cast<double>(t)));
  k.lr = (T)lr;
  k.eps = (T)c.eps;
  k.wd = (T)c.weight_decay;
  k.lrwd = (T)(lr * c.weight_decay);
  k.den = (T)(1.0 + lr * c.weight_decay);
  k.rho = (T)c.sophia_rho;
  // fp32 Adan multiplies by the reciprocals (update.cuh): 1 IEEE division per element
  // instead of 5 -- the per-element scalars are rounded once from their double values
  const double c1d = 1.0 - std::pow(c.beta1, static_cast<double>(t));
  const double c2d = 1.0 - std::pow(c.beta2, static_cast<double>(t));
  const double c3d = 1.0 - std::pow(c.beta3, static_cast<double>(t));
  k.rc1 = (T)(1.0 / c1d);
  k.rc2 = (T)(1.0 / c2d);
  k.rc3 = (T)(1.0 / c3d);
  k.rden = (T)(1.0 / (1.0 + lr * c.weight_decay));
  if (c.kind == MCO_ADAN && sizeof(T) == 4)
    k.sthr = sqrt_eps_threshold_mul<T>(k.eps, k.rc3);
  else
    k.sthr = sqrt_eps_threshold<T>(k.eps, c.kind == MCO_ADAN ? k.c3 : k.c2);
  k.first = t == 1 ? 1 : 0;
  // only Sophia reads the refresh flag (optim.cpp:161); interval < 1 is refused for it at
  // create, every other kind ignores the field as the reference does
  k.refresh = (c.kind == MCO_SOPHIA && c.update_interval >= 1 &&
               ((t - 1) % c.update_interval) == 0) ? 1 : 0;
  return k;
}


// Host-span staging: [H2D a, H2D b] -> kernel -> D2H a, chunk by chunk on
// kHostStages streams, so both PCIe directions and the kernels overlap.  One staging set
// per device (host-span calls are synchronous; the mutex serialises them).
#ifndef MCO_HOST_STAGES
#define MCO_HOST_STAGES 3
#endif
constexpr int kHostStages = MCO_HOST_STAGES;  // chunk k+S reuses chunk k's buffers
struct HostStage {
  std::mutex mu;
  cudaStream_t st[kHostStages] = {};
  void* buf[kHostStages][2] = {};
  uint64_t chunk_bytes = 0;
  // mco_lomo_apply_host's device-resident gradient, kept between calls: freeing 27 GB
  // (7B fp32) costs ~150 ms of cudaFree per call, 13 % of the call (MCO_HOST_TRACE)
  std::mutex gres_mu;  // held for a whole call that uses gres
  void* gres = nullptr;
  uint64_t gres_bytes = 0;
};
// mco_host_release: every device's HostStage::gres
void host_release_all();

HostStage& host_stage(int dev);

// MCO_HOST_TRACE=1: wall time of each stage of a host-span call on stderr (what = null
// starts the clock).
void host_trace(const char* what);

// fn(dev_a, dev_b, offset, count, stream) runs the kernel(s) for one chunk.
template <class F>
void host_pipeline(int dev, void* a, size_t as, const void* b, size_t bs, uint64_t n,
                   bool write_back, F&& fn) {
  HostStage& hs = host_stage(dev);
  std::lock_guard<std::mutex> lock(hs.mu);
  const uint64_t C = hs.chunk_bytes / 8;
  int k = 0;
  for (uint64_t off = 0; off < n; off += C, k = (k + 1) % kHostStages) {
    const uint64_t m = std::min(C, n - off);
    cudaStream_t st = hs.st[k];
    MCO_CUDA_CHECK(cudaMemcpyAsync(hs.buf[k][0], (const char*)a + off * as, m * as,
                                   cudaMemcpyHostToDevice, st));
    if (b)
      MCO_CUDA_CHECK(cudaMemcpyAsync(hs.buf[k][1], (const char*)b + off * bs, m * bs,
                                     cudaMemcpyHostToDevice, st));
    fn(hs.buf[k][0], hs.buf[k][1], off, m, st);
    if (write_back)
      MCO_CUDA_CHECK(cudaMemcpyAsync((char*)a + off * as, hs.buf[k][0], m * as,
                                     cudaMemcpyDeviceToHost, st));
  }
  for (int i = 0; i < kHostStages; ++i) MCO_CUDA_CHECK(cudaStreamSynchronize(hs.st[i]));
}

}  // namespace mco

struct mco_flat;
namespace mco {
// abi_flat.cpp: one piece of a step at the handle's current t (sharders, shard.cpp).
void flat_step_range(mco_flat* h, void* p, int pdt, const void* g, int gdt, uint16_t* pout,
                     uint64_t n, uint64_t state_off, double lr, cudaStream_t st);
}  // namespace mco

// ---- handles ---------------------------------------------------------------------
struct mco_flat {
  mco_config cfg{};
  uint64_t n = 0;
  int device = 0;
  int state_dtype = MCO_F32;
  int64_t t = 0;
  void* slot[4] = {nullptr, nullptr, nullptr, nullptr};  // kernel slots s0..s3
  void* base[4] = {nullptr, nullptr, nullptr, nullptr};  // allocations (8 elements slack)
  int phase = 0;         // slot = base + phase elements (matches the params' phase mod 8)
  bool exposed = false;  // buffers() handed out: the layout is frozen
  bool stepped = false;  // a step was launched (graph mode leaves t on the device)
  std::vector<std::pair<const char*, void*>> named;       // buffers() order
  // graph mode (mco_flat_graph_enable): device step counter + scalar rows
  mco::FlatGraphDev* gdev = nullptr;
  mco::GraphRow<float>* grow_f = nullptr;
  mco::GraphRow<double>* grow_d = nullptr;
  int64_t grows = 0;
  const double* glr = nullptr;  // device lr (null: the lr argument of each call)
  // element size of state slot i: MCO_F32M64 (Sophia precise-m) keeps m (slot 0) in fp64
  size_t slot_es(int i) const {
    if (state_dtype == MCO_F32M64) return i == 0 ? 8 : 4;
    return state_dtype == MCO_F64 ? 8 : 4;
  }
  int slot_dtype(int i) const {
    if (state_dtype == MCO_F32M64) return i == 0 ? MCO_F64 : MCO_F32;
    return state_dtype;
  }
  void free_graph() {
    for (void* p : {(void*)gdev, (void*)grow_f, (void*)grow_d})
      if (p) cudaFree(p);
    gdev = nullptr, grow_f = nullptr, grow_d = nullptr, grows = 0, glr = nullptr;
  }
  ~mco_flat() {
    free_graph();
    for (void* p : base)
      if (p) cudaFree(p);
  }
};

struct mco_adalomo {
  mco::AdaLomoPlan plan;
  // host-span path (lazily created): device copies of the flat set, 3 streams,
  // per-tensor events for the H2D -> apply -> D2H pipeline
  float* hp = nullptr;
  void* hg = nullptr;
  cudaStream_t hst[3] = {nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> ev_in, ev_out;
  // last hook-form call (tensor, stream): the next one on the same stream for another
  // tensor may start its K1 under the previous K6 (adalomo.h AdaLomoCall::early)
  int last_hook = -1;
  void* last_stream = nullptr;
  ~mco_adalomo() {
    if (hp) cudaFree(hp);
    if (hg) cudaFree(hg);
    for (auto s : hst)
      if (s) cudaStreamDestroy(s);
    for (auto e : ev_in) cudaEventDestroy(e);
    for (auto e : ev_out) cudaEventDestroy(e);
    void* ptrs[] = {plan.d_tiles, plan.d_chunks, plan.d_chunk_sc, plan.d_tensors, plan.d_item_off, plan.d_col_off,
                    plan.d_payload, plan.d_state,
                    plan.d_colpart, plan.d_rowpart, plan.d_tile_sc, plan.d_tens_sc,
                    plan.d_fa,    plan.d_fb,      plan.d_glob, plan.d_fra, plan.d_frb,
                    plan.d_mins};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
};
