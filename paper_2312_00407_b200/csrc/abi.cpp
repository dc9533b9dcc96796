// C-ABI (include/mco.h) over the sm_100a kernels: the drop-in boundary for
// minicollie::optim (optim.hpp).  Host logic here restates the reference's
// non-kernel behaviour -- kind names, defaults, validation, error messages,
// state accounting, step counter, buffer naming -- citing optim.cpp lines.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "adalomo.h"
#include "kernels.h"
#include "mco.h"
#include "abi_util.h"
#include "peer.h"

namespace mco {

namespace {
std::atomic<uint64_t> g_launches{0};
thread_local std::string g_err;
}  // namespace

void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void set_last_error(const std::string& m) { g_err = m; }

const DeviceInfo& device_info(int device) {
  static std::mutex mu;
  static std::unordered_map<int, DeviceInfo> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(device);
  if (it != cache.end()) return it->second;
  DeviceInfo d;
  MCO_CUDA_CHECK(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device));
  MCO_CUDA_CHECK(cudaDeviceGetAttribute(&d.l2_bytes, cudaDevAttrL2CacheSize, device));
  return cache.emplace(device, d).first->second;
}

int current_device() {
  int d = 0;
  MCO_CUDA_CHECK(cudaGetDevice(&d));
  return d;
}

namespace {

// optim.cpp:17-28
const char* kind_cstr(int kind) {
  switch (kind) {
    case MCO_ADAMW: return "adamw";
    case MCO_LION: return "lion";
    case MCO_ADAN: return "adan";
    case MCO_SOPHIA: return "sophia";
    case MCO_LOMO: return "lomo";
    case MCO_ADALOMO: return "adalomo";
  }
  return nullptr;
}

std::string kind_str(int kind) {
  const char* s = kind_cstr(kind);
  if (!s) throw Error(MCO_CONFIG, "unknown optimizer kind");
  return s;
}

bool fused(int kind) { return kind == MCO_LOMO || kind == MCO_ADALOMO; }  // optim.cpp:30

// optim.cpp:32-61
mco_config defaults(int kind) {
  if (!kind_cstr(kind)) throw Error(MCO_CONFIG, "unknown optimizer kind");
  mco_config c{};
  c.kind = kind;
  c.lr = 1e-3;
  c.weight_decay = 0.0;
  c.beta1 = 0.9;
  c.beta2 = 0.999;
  c.beta3 = 0.99;
  c.eps = 1e-8;
  c.has_clip_threshold = 0;
  c.clip_threshold = 0.0;
  c.adalomo_clip = 1.0;
  c.sophia_rho = 0.04;
  c.update_interval = 10;
  switch (kind) {
    case MCO_ADAMW: c.beta1 = 0.9; c.beta2 = 0.999; break;
    case MCO_LION: c.beta1 = 0.9; c.beta2 = 0.99; break;
    case MCO_ADAN: c.beta1 = 0.98; c.beta2 = 0.92; c.beta3 = 0.99; break;
    case MCO_SOPHIA: c.beta1 = 0.965; c.beta2 = 0.99; break;
    case MCO_LOMO: break;
    case MCO_ADALOMO: c.beta2 = 0.99; c.eps = 1e-30; break;
  }
  return c;
}

// optim.cpp:63-70
void validate(const mco_config& c) {
  if (c.lr <= 0) throw Error(MCO_CONFIG, "optimizer: lr must be > 0");
  if (c.eps <= 0) throw Error(MCO_CONFIG, "optimizer: eps must be > 0");
  for (double b : {c.beta1, c.beta2, c.beta3})
    if (b < 0 || b >= 1) throw Error(MCO_CONFIG, "optimizer: betas must lie in [0, 1)");
  if (c.weight_decay < 0) throw Error(MCO_CONFIG, "optimizer: weight_decay must be >= 0");
  if (c.update_interval < 1) throw Error(MCO_CONFIG, "optimizer: update_interval must be >= 1");
}

// Per-step scalars (optim.cpp:116-117, 138-141, 159): double on the host, one
// rounding to the kernel's type.  Identical rule in oracle/mco_oracle.c.
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
  k.sthr = sqrt_eps_threshold<T>(k.eps, c.kind == MCO_ADAN ? k.c3 : k.c2);
  k.first = t == 1 ? 1 : 0;
  k.refresh = ((t - 1) % c.update_interval) == 0 ? 1 : 0;
  return k;
}

size_t dtype_size(int dt) {
  switch (dt) {
    case MCO_F32: return 4;
    case MCO_BF16: return 2;
    case MCO_F64: return 8;
  }
  throw Error(MCO_CONTRACT, "unknown dtype " + std::to_string(dt));
}

// Sum-of-squares workspace per (device, stream): launches on one stream are
// ordered, so the partials / ticket counter are never shared concurrently.
void* sumsq_ws(cudaStream_t st) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, void*> pool;
  const int dev = current_device();
  const uint64_t key = ((uint64_t)(uintptr_t)st) * 131 + (uint64_t)dev;
  std::lock_guard<std::mutex> lock(mu);
  auto it = pool.find(key);
  if (it != pool.end()) return it->second;
  void* p = nullptr;
  MCO_CUDA_CHECK(cudaMalloc(&p, sumsq_ws_bytes()));
  MCO_CUDA_CHECK(cudaMemset(p, 0, sumsq_ws_bytes()));
  pool[key] = p;
  return p;
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
};

HostStage& host_stage(int dev) {
  static std::mutex mu;
  static std::unordered_map<int, HostStage*> stages;
  std::lock_guard<std::mutex> lock(mu);
  auto& s = stages[dev];
  if (!s) {
    s = new HostStage;
    s->chunk_bytes = 8ull << 24;  // 16 Mi elements of <= 8 bytes
    for (int i = 0; i < kHostStages; ++i) {
      MCO_CUDA_CHECK(cudaStreamCreateWithFlags(&s->st[i], cudaStreamNonBlocking));
      MCO_CUDA_CHECK(cudaMalloc(&s->buf[i][0], s->chunk_bytes));
      MCO_CUDA_CHECK(cudaMalloc(&s->buf[i][1], s->chunk_bytes));
    }
  }
  return *s;
}

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

}  // namespace
}  // namespace mco

using namespace mco;

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
  std::vector<std::pair<const char*, void*>> named;       // buffers() order
  ~mco_flat() {
    for (void* p : base)
      if (p) cudaFree(p);
  }
};

struct mco_adalomo {
  AdaLomoPlan plan;
  // host-span path (lazily created): device copies of the flat set, 3 streams,
  // per-tensor events for the H2D -> apply -> D2H pipeline
  float* hp = nullptr;
  void* hg = nullptr;
  cudaStream_t hst[3] = {nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> ev_in, ev_out;
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
                    plan.d_fa,    plan.d_fb,      plan.d_glob};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
};

extern "C" {

const char* mco_last_error(void) { return g_err.c_str(); }
const char* mco_version(void) { return "mco 0.1 (sm_100a)"; }
uint64_t mco_launch_count(void) { return g_launches.load(); }

mco_status mco_parse_kind(const char* name, int* out) {
  return guard([&] {
    const std::string s = name ? name : "";
    for (int k = 0; k <= MCO_ADALOMO; ++k)
      if (s == kind_cstr(k)) {
        *out = k;
        return;
      }
    throw Error(MCO_CONFIG, "unknown optimizer kind '" + s + "'");  // optim.cpp:15
  });
}

const char* mco_kind_name(int kind) { return kind_cstr(kind); }
int mco_is_fused(int kind) { return fused(kind) ? 1 : 0; }

mco_status mco_defaults_for(int kind, mco_config* out) {
  return guard([&] { *out = defaults(kind); });
}

mco_status mco_validate(const mco_config* cfg) { return guard([&] { validate(*cfg); }); }

// optim.cpp:339-362
mco_status mco_state_bytes(int kind, uint64_t count, int param_bytes, int grad_bytes,
                           int master_copy, int nshapes, const int* ndims, const int64_t* dims,
                           uint64_t* out) {
  (void)grad_bytes;
  return guard([&] {
    const bool needs_master = master_copy && param_bytes < 4;  // optim.hpp:118
    const uint64_t master = needs_master ? 4 * count : 0;
    switch (kind) {
      case MCO_ADAMW: *out = 8 * count + master; return;
      case MCO_LION: *out = 4 * count + master; return;
      case MCO_ADAN: *out = 12 * count + master; return;
      case MCO_SOPHIA: *out = 8 * count + master; return;
      case MCO_LOMO: *out = 0; return;
      case MCO_ADALOMO: {
        if (nshapes == 0 && count > 0)
          throw Error(MCO_CONFIG,
                      "state_bytes: adalomo needs parameter shapes for factored accounting");
        uint64_t bytes = 0;
        const int64_t* d = dims;
        for (int k = 0; k < nshapes; ++k) {
          if (ndims[k] == 2) {
            bytes += static_cast<uint64_t>(d[0] + d[1]) * 4;
          } else {
            int64_t n = 1;
            for (int j = 0; j < ndims[k]; ++j) n *= d[j];
            bytes += static_cast<uint64_t>(n) * 4;
          }
          d += ndims[k];
        }
        *out = bytes;
        return;
      }
    }
    throw Error(MCO_CONFIG, "state_bytes: unknown optimizer kind");
  });
}

// ---- FlatOptimizer ---------------------------------------------------------------
// optim.cpp:74-98
mco_status mco_flat_create(const mco_config* cfg, uint64_t owned_len, int device,
                           int state_dtype, mco_flat** out) {
  return guard([&] {
    *out = nullptr;
    if (fused(cfg->kind))
      throw Error(MCO_CONTRACT, "FlatOptimizer: " + kind_str(cfg->kind) +
                                    " is a fused optimizer and keeps no flat state");
    kind_str(cfg->kind);
    if (state_dtype != MCO_F32 && state_dtype != MCO_F64)
      throw Error(MCO_CONTRACT, "FlatOptimizer: state dtype must be f32 or f64");
    DeviceGuard dg(device);
    auto h = std::make_unique<mco_flat>();
    h->cfg = *cfg;
    h->n = owned_len;
    h->device = device;
    h->state_dtype = state_dtype;
    // slots s0..s3 and the reference's buffers() names / order (optim.cpp:173-181)
    const char* names[4] = {nullptr, nullptr, nullptr, nullptr};
    int nslots = 0;
    switch (cfg->kind) {
      case MCO_ADAMW: names[0] = "m"; names[1] = "v"; nslots = 2; break;
      case MCO_LION: names[0] = "m"; nslots = 1; break;
      case MCO_ADAN: names[0] = "m"; names[1] = "v"; names[2] = "n"; names[3] = "g_prev";
        nslots = 4; break;
      case MCO_SOPHIA: names[0] = "m"; names[1] = "h"; nslots = 2; break;
    }
    // 8 elements of slack: the state is shifted to the parameters' alignment phase at
    // the first step (align_state_to), so shard views at odd offsets stay vectorised
    const size_t bytes = (std::max<uint64_t>(owned_len, 1) + 8) * dtype_size(state_dtype);
    for (int i = 0; i < nslots; ++i) {
      MCO_CUDA_CHECK(cudaMalloc(&h->base[i], bytes));
      MCO_CUDA_CHECK(cudaMemset(h->base[i], 0, bytes));
      h->slot[i] = h->base[i];
      h->named.emplace_back(names[i], h->slot[i]);
    }
    *out = h.release();
  });
}

mco_status mco_flat_destroy(mco_flat* h) {
  return guard([&] {
    if (!h) return;
    DeviceGuard dg(h->device);
    delete h;
  });
}

namespace {
void check_lengths(const mco_flat* h, uint64_t np, uint64_t ng) {
  if (np != ng)  // optim.cpp:101-103
    throw Error(MCO_CONTRACT, "optimizer step: params/grads length mismatch: " +
                                  std::to_string(np) + " vs " + std::to_string(ng));
  if (np > h->n)
    throw Error(MCO_CONTRACT, "optimizer step: " + std::to_string(np) +
                                  " elements exceed the owned state of " + std::to_string(h->n));
}

// Before the first step (state still all zero, never handed out) the state buffers are
// shifted within their slack so that state[i] has the same address phase (mod 8
// elements) as params[i]: the launch can then peel a short head and run the rest
// aligned (flat.cu, launch_flat_step).
void align_state_to(mco_flat* h, const void* params) {
  if (h->exposed || h->t != 0 || !params) return;
  const size_t es = dtype_size(h->state_dtype);
  const uintptr_t u = (uintptr_t)params;
  if (u % es) return;
  const int want = (int)((u / es) % 8);
  if (want == h->phase) return;
  h->phase = want;
  for (int i = 0; i < 4; ++i)
    if (h->base[i]) h->slot[i] = (char*)h->base[i] + (size_t)want * es;
  for (size_t i = 0; i < h->named.size(); ++i) h->named[i].second = h->slot[i];
}

void flat_launch(mco_flat* h, void* p, int pdt, const void* g, int gdt, uint16_t* pout,
                 uint64_t n, uint64_t state_off, double lr, cudaStream_t st) {
  FlatArgs a{};
  a.kind = h->cfg.kind;
  a.state_dtype = h->state_dtype;
  a.p = p;
  a.p_dtype = pdt;
  a.g = g;
  a.g_dtype = gdt;
  const size_t es = dtype_size(h->state_dtype);
  for (int i = 0; i < 4; ++i) a.s[i] = h->slot[i] ? (char*)h->slot[i] + state_off * es : nullptr;
  a.p_out_bf16 = pout;
  a.n = n;
  const auto kf = make_consts<float>(h->cfg, h->t, lr);
  const auto kd = make_consts<double>(h->cfg, h->t, lr);
  launch_flat_step(a, kf, kd, st);
}

void check_dtypes(const mco_flat* h, int pdt, int gdt) {
  if (h->state_dtype == MCO_F64) {
    if (pdt != MCO_F64 || gdt != MCO_F64)
      throw Error(MCO_CONTRACT, "optimizer step: f64 state takes f64 params and grads");
  } else if (pdt != MCO_F32 || (gdt != MCO_F32 && gdt != MCO_BF16)) {
    throw Error(MCO_CONTRACT, "optimizer step: f32 state takes f32 params and f32/bf16 grads");
  }
}
}  // namespace

// optim.cpp:100-112
mco_status mco_flat_step(mco_flat* h, void* params, int pdt, uint64_t np, const void* grads,
                         int gdt, uint64_t ng, double lr, void* stream) {
  return guard([&] {
    check_lengths(h, np, ng);
    check_dtypes(h, pdt, gdt);
    DeviceGuard dg(h->device);
    align_state_to(h, params);
    ++h->t;  // optim.cpp:104
    flat_launch(h, params, pdt, grads, gdt, nullptr, np, 0, lr, (cudaStream_t)stream);
  });
}

mco_status mco_flat_step_mixed(mco_flat* h, float* master, const void* grads, int gdt,
                               uint16_t* pout, uint64_t n, double lr, void* stream) {
  return guard([&] {
    check_lengths(h, n, n);
    check_dtypes(h, MCO_F32, gdt);
    if (h->state_dtype != MCO_F32) throw Error(MCO_CONTRACT, "mixed step needs f32 state");
    if (!pout) throw Error(MCO_CONTRACT, "mixed step: param_out is null");
    DeviceGuard dg(h->device);
    align_state_to(h, master);
    ++h->t;
    flat_launch(h, master, MCO_F32, grads, gdt, pout, n, 0, lr, (cudaStream_t)stream);
  });
}

// Host-span overload: pipelined H2D(p,g) -> step -> D2H(p) over chunks on two
// streams, so PCIe traffic in both directions overlaps the kernels.
mco_status mco_flat_step_host(mco_flat* h, void* params, int pdt, uint64_t np, const void* grads,
                              int gdt, uint64_t ng, double lr) {
  return guard([&] {
    check_lengths(h, np, ng);
    check_dtypes(h, pdt, gdt);
    DeviceGuard dg(h->device);
    ++h->t;
    host_pipeline(h->device, params, dtype_size(pdt), grads, dtype_size(gdt), np, true,
                  [&](void* dp, void* dg_, uint64_t off, uint64_t m, cudaStream_t st) {
                    flat_launch(h, dp, pdt, dg_, gdt, nullptr, m, off, lr, st);
                  });
  });
}

mco_status mco_flat_get_steps(const mco_flat* h, int64_t* t) {
  return guard([&] { *t = h->t; });
}
mco_status mco_flat_set_steps(mco_flat* h, int64_t t) {
  return guard([&] { h->t = t; });
}
mco_status mco_flat_state_bytes(const mco_flat* h, uint64_t* out) {
  return guard([&] { *out = h->named.size() * h->n * dtype_size(h->state_dtype); });
}
mco_status mco_flat_config(const mco_flat* h, mco_config* out) {
  return guard([&] { *out = h->cfg; });
}
mco_status mco_flat_num_buffers(const mco_flat* h, int* out) {
  return guard([&] { *out = (int)h->named.size(); });
}
mco_status mco_flat_buffer(mco_flat* h, int i, const char** name, void** ptr, uint64_t* len,
                           int* dtype) {
  return guard([&] {
    if (i < 0 || i >= (int)h->named.size())
      throw Error(MCO_CONTRACT, "buffers(): index out of range");
    h->exposed = true;  // callers may keep the pointer: no more relayout
    *name = h->named[i].first;
    *ptr = h->named[i].second;
    *len = h->n;
    *dtype = h->state_dtype;
  });
}

// ---- ZeRO step fused with RS / AG over peer memory (peer.cu) ------------------------
mco_status mco_flat_step_peers(mco_flat* h, const void* const* grad_bufs, int grad_dtype,
                               void* const* param_bufs, int param_dtype, int npeers,
                               float* master, uint64_t offset, uint64_t n, double lr,
                               void* stream) {
  return guard([&] {
    check_lengths(h, n, n);
    if (h->state_dtype != MCO_F32)
      throw Error(MCO_CONTRACT, "peer step: f32 optimizer state required");
    if (!master) throw Error(MCO_CONTRACT, "peer step: master is null");
    if (npeers < 1 || npeers > kMaxPeers)
      throw Error(MCO_CONTRACT, "peer step: npeers must be 1.." + std::to_string(kMaxPeers));
    PeerPtrs pp{};
    pp.n = npeers;
    for (int r = 0; r < npeers; ++r) {
      if (!grad_bufs[r] || !param_bufs[r])
        throw Error(MCO_CONTRACT, "peer step: null peer buffer");
      pp.g[r] = grad_bufs[r];
      pp.p[r] = param_bufs[r];
    }
    DeviceGuard dg(h->device);
    ++h->t;
    const auto kf = make_consts<float>(h->cfg, h->t, lr);
    launch_peer_step(h->cfg.kind, pp, grad_dtype, param_dtype, master, h->slot, offset, n, kf,
                     (cudaStream_t)stream);
  });
}

namespace {
PeerPtrs make_peers(const void* const* grad_bufs, void* const* param_bufs, int npeers) {
  if (npeers < 1 || npeers > kMaxPeers)
    throw Error(MCO_CONTRACT, "peer step: npeers must be 1.." + std::to_string(kMaxPeers));
  PeerPtrs pp{};
  pp.n = npeers;
  for (int r = 0; r < npeers; ++r) {
    if (!grad_bufs[r] || (param_bufs && !param_bufs[r]))
      throw Error(MCO_CONTRACT, "peer step: null peer buffer");
    pp.g[r] = grad_bufs[r];
    pp.p[r] = param_bufs ? param_bufs[r] : nullptr;
  }
  return pp;
}
}  // namespace

// (sum over ranks of g_r)^2 summed over this rank's owned range, into *dev_out.
mco_status mco_sumsq_peers(const void* const* grad_bufs, int grad_dtype, int npeers,
                           uint64_t offset, uint64_t n, double* dev_out, void* stream) {
  return guard([&] {
    const PeerPtrs pp = make_peers(grad_bufs, nullptr, npeers);
    cudaStream_t st = (cudaStream_t)stream;
    launch_peer_sumsq(pp, grad_dtype, offset, n, dev_out, sumsq_ws(st), st);
  });
}

// LOMO fused with its collectives: p = p - f * sum_r g_r over the owned range,
// written into every rank's replica; f = lr*scale, or from the all-reduced
// dev_sumsq and clip (optim.cpp:302-303) when dev_sumsq is not null.
mco_status mco_lomo_apply_peers(const void* const* grad_bufs, int grad_dtype,
                                void* const* param_bufs, int param_dtype, int npeers,
                                float* master, uint64_t offset, uint64_t n, double lr,
                                double scale, const double* dev_sumsq, double clip,
                                void* stream) {
  return guard([&] {
    const PeerPtrs pp = make_peers(grad_bufs, param_bufs, npeers);
    launch_peer_lomo(pp, grad_dtype, param_dtype, master, offset, n, lr, scale, dev_sumsq, clip,
                     (cudaStream_t)stream);
  });
}

// Symmetric buffers for the peer step: allocation + CUDA IPC export / import.
mco_status mco_peer_alloc(uint64_t bytes, int device, void** out) {
  return guard([&] {
    DeviceGuard dg(device);
    MCO_CUDA_CHECK(cudaMalloc(out, std::max<uint64_t>(bytes, 1)));
  });
}
mco_status mco_peer_free(void* p) {
  return guard([&] { MCO_CUDA_CHECK(cudaFree(p)); });
}
mco_status mco_peer_export(void* p, void* handle_out) {
  return guard([&] {
    cudaIpcMemHandle_t h;
    MCO_CUDA_CHECK(cudaIpcGetMemHandle(&h, p));
    static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
    std::memcpy(handle_out, &h, sizeof(h));
  });
}
mco_status mco_peer_import(const void* handle, int device, void** out) {
  return guard([&] {
    DeviceGuard dg(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    MCO_CUDA_CHECK(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  });
}
mco_status mco_peer_close(void* p) {
  return guard([&] { MCO_CUDA_CHECK(cudaIpcCloseMemHandle(p)); });
}

// ---- LOMO -------------------------------------------------------------------------
mco_status mco_lomo_apply(void* p, int pdt, const void* g, int gdt, uint64_t n, double lr,
                          double scale, void* stream) {
  return guard([&] { launch_lomo(p, pdt, g, gdt, n, lr, scale, nullptr, 0.0, (cudaStream_t)stream); });
}

mco_status mco_lomo_apply_clipped(void* p, int pdt, const void* g, int gdt, uint64_t n, double lr,
                                  const double* dev_sumsq, double clip, void* stream) {
  return guard([&] {
    if (!dev_sumsq) throw Error(MCO_CONTRACT, "lomo clip: device sum of squares is null");
    launch_lomo(p, pdt, g, gdt, n, lr, 1.0, dev_sumsq, clip, (cudaStream_t)stream);
  });
}

// lomo_apply on host spans (the reference's Tensor data is host memory).
// clip >= 0: two passes over the gradient -- sum of squares, then the update.
mco_status mco_lomo_apply_host(void* p, int pdt, const void* g, int gdt, uint64_t n, double lr,
                               double scale, double clip) {
  return guard([&] {
    const int dev = current_device();
    const double* dnorm = nullptr;
    double* acc = nullptr;
    if (clip >= 0) {
      MCO_CUDA_CHECK(cudaMalloc(&acc, sizeof(double)));
      MCO_CUDA_CHECK(cudaMemset(acc, 0, sizeof(double)));
      HostStage& hs = host_stage(dev);
      host_pipeline(dev, const_cast<void*>(g), dtype_size(gdt), nullptr, 0, n, false,
                    [&](void* dg_, void*, uint64_t, uint64_t m, cudaStream_t st) {
                      // one accumulator, chunks strictly ordered through stream 0
                      if (st != hs.st[0]) {
                        cudaEvent_t ev;
                        MCO_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                        MCO_CUDA_CHECK(cudaEventRecord(ev, hs.st[0]));
                        MCO_CUDA_CHECK(cudaStreamWaitEvent(st, ev, 0));
                        MCO_CUDA_CHECK(cudaEventDestroy(ev));
                      }
                      launch_sumsq(dg_, gdt, m, acc, 1, sumsq_ws(st), st);
                      if (st != hs.st[0]) {
                        cudaEvent_t ev;
                        MCO_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                        MCO_CUDA_CHECK(cudaEventRecord(ev, st));
                        MCO_CUDA_CHECK(cudaStreamWaitEvent(hs.st[0], ev, 0));
                        MCO_CUDA_CHECK(cudaEventDestroy(ev));
                      }
                    });
      dnorm = acc;
    }
    host_pipeline(dev, p, dtype_size(pdt), g, dtype_size(gdt), n, true,
                  [&](void* dp, void* dg_, uint64_t, uint64_t m, cudaStream_t st) {
                    launch_lomo(dp, pdt, dg_, gdt, m, lr, scale, dnorm, clip, st);
                  });
    if (acc) cudaFree(acc);
  });
}

mco_status mco_sumsq(const void* x, int dtype, uint64_t n, double* out, int accumulate,
                     void* stream) {
  return guard([&] {
    dtype_size(dtype);
    cudaStream_t st = (cudaStream_t)stream;
    launch_sumsq(x, dtype, n, out, accumulate, sumsq_ws(st), st);
  });
}

// ---- AdaLomo ----------------------------------------------------------------------
// optim.cpp:192-207
mco_status mco_adalomo_create(const mco_config* cfg, int ntensors, const int* ndims,
                              const int64_t* dims, int device, mco_adalomo** out) {
  return guard([&] {
    *out = nullptr;
    DeviceGuard dg(device);
    auto h = std::make_unique<mco_adalomo>();
    auto& pl = h->plan;
    pl.cfg = *cfg;
    pl.device = device;
    std::vector<std::vector<int64_t>> shapes;
    const int64_t* d = dims;
    for (int k = 0; k < ntensors; ++k) {
      shapes.emplace_back(d, d + ndims[k]);
      d += ndims[k];
    }
    build_adalomo_plan(pl, shapes, device_info(device).sms);
    auto alloc = [](auto** p, size_t count, size_t esz) {
      MCO_CUDA_CHECK(cudaMalloc((void**)p, std::max<size_t>(count, 1) * esz));
      MCO_CUDA_CHECK(cudaMemset(*p, 0, std::max<size_t>(count, 1) * esz));
    };
    alloc(&pl.d_tiles, pl.h_tiles.size(), sizeof(Tile));
    alloc(&pl.d_chunks, pl.h_chunks.size(), sizeof(Chunk));
    alloc(&pl.d_chunk_sc, pl.h_chunks.size(), sizeof(double));
    alloc(&pl.d_tensors, pl.h_tensors.size(), sizeof(TensorInfo));
    alloc(&pl.d_item_off, pl.h_item_off.size(), sizeof(int64_t));
    alloc(&pl.d_col_off, pl.h_col_off.size(), sizeof(int64_t));
    alloc(&pl.d_payload, pl.stats_len + pl.usq_len, sizeof(double));
    alloc(&pl.d_state, pl.state_len, sizeof(double));
    alloc(&pl.d_colpart, pl.colpart_len, sizeof(float));
    alloc(&pl.d_rowpart, pl.rowpart_len, sizeof(double));
    alloc(&pl.d_tile_sc, pl.h_tiles.size() * 4, sizeof(double));
    alloc(&pl.d_tens_sc, pl.h_tensors.size() * 8, sizeof(double));
    alloc(&pl.d_fa, pl.fa_len, sizeof(float));
    alloc(&pl.d_fb, pl.fb_len, sizeof(float));
    alloc(&pl.d_glob, 4, sizeof(double));
    MCO_CUDA_CHECK(cudaMemcpy(pl.d_tiles, pl.h_tiles.data(), pl.h_tiles.size() * sizeof(Tile),
                              cudaMemcpyHostToDevice));
    MCO_CUDA_CHECK(cudaMemcpy(pl.d_chunks, pl.h_chunks.data(),
                              pl.h_chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
    MCO_CUDA_CHECK(cudaMemcpy(pl.d_tensors, pl.h_tensors.data(),
                              pl.h_tensors.size() * sizeof(TensorInfo), cudaMemcpyHostToDevice));
    MCO_CUDA_CHECK(cudaMemcpy(pl.d_col_off, pl.h_col_off.data(),
                              pl.h_col_off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    MCO_CUDA_CHECK(cudaMemcpy(pl.d_item_off, pl.h_item_off.data(),
                              pl.h_item_off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    *out = h.release();
  });
}

mco_status mco_adalomo_destroy(mco_adalomo* h) {
  return guard([&] {
    if (!h) return;
    DeviceGuard dg(h->plan.device);
    delete h;
  });
}

namespace {
void check_ada_dtypes(int pdt, int gdt) {
  const bool ok = (pdt == MCO_F32 && (gdt == MCO_F32 || gdt == MCO_BF16)) ||
                  (pdt == MCO_BF16 && gdt == MCO_BF16);
  if (!ok)
    throw Error(MCO_CONTRACT,
                "adalomo: params / grads must be f32 / f32, f32 / bf16 or bf16 / bf16");
}
}  // namespace

// optim.cpp:215-275 (hook form: one tensor)
mco_status mco_adalomo_apply(mco_adalomo* h, int idx, void* param, int pdt, const void* grad,
                             int gdt, double lr, const double* dev_grad_sumsq, void* stream) {
  return guard([&] {
    if (idx < 0 || idx >= (int)h->plan.h_tensors.size())  // optim.cpp:212
      throw Error(MCO_CONTRACT, "adalomo: unknown parameter '" + std::to_string(idx) + "'");
    check_ada_dtypes(pdt, gdt);
    DeviceGuard dg(h->plan.device);
    AdaLomoCall c{};
    c.t0 = idx;
    c.t1 = idx + 1;
    c.p = param;
    c.p_dtype = pdt;
    c.g = grad;
    c.g_dtype = gdt;
    c.single = 1;
    c.lr = lr;
    c.use_clip = (dev_grad_sumsq != nullptr && h->plan.cfg.has_clip_threshold) ? 1 : 0;
    c.ext_sumsq = dev_grad_sumsq;
    launch_adalomo(h->plan, c, (cudaStream_t)stream);
    h->plan.h_tensors[idx].t += 1;
  });
}

// List form of the hook: tensors t0..t1-1 at separate device pointers, one launch chain
// per kMaxTab tensors (AdaLomo's statistics are per tensor, so the split is exact).
mco_status mco_adalomo_apply_list(mco_adalomo* h, int t0, int t1, void* const* params,
                                  int pdt, const void* const* grads, int gdt, double lr,
                                  const double* dev_grad_sumsq, void* stream) {
  return guard([&] {
    const int nt = (int)h->plan.h_tensors.size();
    if (t0 < 0 || t1 > nt || t0 > t1)
      throw Error(MCO_CONTRACT, "adalomo: tensor range [" + std::to_string(t0) + ", " +
                                    std::to_string(t1) + ") outside 0.." + std::to_string(nt));
    check_ada_dtypes(pdt, gdt);
    for (int k = t0; k < t1; ++k)
      if (!params[k - t0] || !grads[k - t0])
        throw Error(MCO_CONTRACT, "adalomo: null tensor pointer for index " + std::to_string(k));
    DeviceGuard dg(h->plan.device);
    for (int a = t0; a < t1; a += kMaxTab) {
      const int b = std::min(t1, a + kMaxTab);
      AdaLomoCall c{};
      c.t0 = a;
      c.t1 = b;
      c.p_dtype = pdt;
      c.g_dtype = gdt;
      c.lr = lr;
      c.use_clip = (dev_grad_sumsq != nullptr && h->plan.cfg.has_clip_threshold) ? 1 : 0;
      c.ext_sumsq = dev_grad_sumsq;
      c.ntab = b - a;
      for (int k = a; k < b; ++k) {
        c.ptab[k - a] = params[k - t0];
        c.gtab[k - a] = grads[k - t0];
      }
      launch_adalomo(h->plan, c, (cudaStream_t)stream);
    }
    for (int k = t0; k < t1; ++k) h->plan.h_tensors[k].t += 1;
  });
}

mco_status mco_adalomo_apply_all(mco_adalomo* h, void* flat_p, int pdt, const void* flat_g,
                                 int gdt, double lr, void* stream) {
  return guard([&] {
    check_ada_dtypes(pdt, gdt);
    DeviceGuard dg(h->plan.device);
    AdaLomoCall c{};
    c.t0 = 0;
    c.t1 = (int)h->plan.h_tensors.size();
    c.p = flat_p;
    c.p_dtype = pdt;
    c.g = flat_g;
    c.g_dtype = gdt;
    c.single = 0;
    c.lr = lr;
    c.use_clip = h->plan.cfg.has_clip_threshold ? 1 : 0;
    c.ext_sumsq = nullptr;
    launch_adalomo(h->plan, c, (cudaStream_t)stream);
    for (auto& T : h->plan.h_tensors) T.t += 1;
  });
}

// Host spans (the reference's Tensor data lives in host memory): per tensor,
// H2D(p_k, g_k) -> hook-form apply(k) -> D2H(p_k) on three streams, so tensor
// k+1's upload overlaps tensor k's update and tensor k-1's download.  With a
// global clip every gradient must be seen first: upload all, apply_all, download.
mco_status mco_adalomo_apply_all_host(mco_adalomo* h, void* p, int pdt, const void* g, int gdt,
                                      double lr) {
  return guard([&] {
    check_ada_dtypes(pdt, gdt);
    auto& pl = h->plan;
    DeviceGuard dg(pl.device);
    const int nt = (int)pl.h_tensors.size();
    const uint64_t total = nt ? (uint64_t)(pl.h_tensors.back().elem_off +
                                           pl.h_tensors.back().numel) : 0;
    const size_t gs = dtype_size(gdt), ps = dtype_size(pdt);
    if (!h->hp) {
      MCO_CUDA_CHECK(cudaMalloc(&h->hp, std::max<uint64_t>(total, 1) * 4));
      MCO_CUDA_CHECK(cudaMalloc(&h->hg, std::max<uint64_t>(total, 1) * 4));
      for (auto& st : h->hst) MCO_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      h->ev_in.resize(nt);
      h->ev_out.resize(nt);
      for (int k = 0; k < nt; ++k) {
        MCO_CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_in[k], cudaEventDisableTiming));
        MCO_CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_out[k], cudaEventDisableTiming));
      }
    }
    cudaStream_t up = h->hst[0], comp = h->hst[1], down = h->hst[2];
    AdaLomoCall c{};
    c.p_dtype = pdt;
    c.g_dtype = gdt;
    c.lr = lr;
    if (pl.cfg.has_clip_threshold) {
      MCO_CUDA_CHECK(cudaMemcpyAsync(h->hp, p, total * ps, cudaMemcpyHostToDevice, up));
      MCO_CUDA_CHECK(cudaMemcpyAsync(h->hg, g, total * gs, cudaMemcpyHostToDevice, up));
      MCO_CUDA_CHECK(cudaStreamSynchronize(up));
      c.t0 = 0;
      c.t1 = nt;
      c.p = h->hp;
      c.g = h->hg;
      c.single = 0;
      c.use_clip = 1;
      launch_adalomo(pl, c, comp);
      MCO_CUDA_CHECK(cudaStreamSynchronize(comp));
      MCO_CUDA_CHECK(cudaMemcpyAsync(p, h->hp, total * ps, cudaMemcpyDeviceToHost, down));
    } else {
      for (int k = 0; k < nt; ++k) {
        const TensorInfo& T = pl.h_tensors[k];
        const uint64_t off = (uint64_t)T.elem_off, n = (uint64_t)T.numel;
        char* dp = (char*)h->hp + off * ps;
        char* dgp = (char*)h->hg + off * gs;
        MCO_CUDA_CHECK(cudaMemcpyAsync(dp, (const char*)p + off * ps, n * ps,
                                       cudaMemcpyHostToDevice, up));
        MCO_CUDA_CHECK(cudaMemcpyAsync(dgp, (const char*)g + off * gs, n * gs,
                                       cudaMemcpyHostToDevice, up));
        MCO_CUDA_CHECK(cudaEventRecord(h->ev_in[k], up));
        MCO_CUDA_CHECK(cudaStreamWaitEvent(comp, h->ev_in[k], 0));
        c.t0 = k;
        c.t1 = k + 1;
        c.p = dp;
        c.g = dgp;
        c.single = 1;
        c.use_clip = 0;
        launch_adalomo(pl, c, comp);
        MCO_CUDA_CHECK(cudaEventRecord(h->ev_out[k], comp));
        MCO_CUDA_CHECK(cudaStreamWaitEvent(down, h->ev_out[k], 0));
        MCO_CUDA_CHECK(cudaMemcpyAsync((char*)p + off * ps, dp, n * ps, cudaMemcpyDeviceToHost,
                                       down));
      }
    }
    for (auto st : h->hst) MCO_CUDA_CHECK(cudaStreamSynchronize(st));
    for (auto& T : pl.h_tensors) T.t += 1;
  });
}

// ---- AdaLomo row-split sharding ---------------------------------------------------
// Tensor `idx` holds a row slice of a global (global_rows x C) matrix (or a
// replica of a 1-D tensor): statistics normalise by the global shape and the
// payload contribution is scaled by `weight` (1 for a row slice, 1 on exactly
// one rank for a replica, 0 elsewhere).
mco_status mco_adalomo_set_shard(mco_adalomo* h, int idx, int64_t global_rows, double weight) {
  return guard([&] {
    auto& pl = h->plan;
    if (idx < 0 || idx >= (int)pl.h_tensors.size())
      throw Error(MCO_CONTRACT, "adalomo: tensor index out of range");
    TensorInfo& T = pl.h_tensors[idx];
    if (global_rows < T.rows)
      throw Error(MCO_CONTRACT, "adalomo: global rows smaller than the local slice");
    DeviceGuard dg(pl.device);
    // keep the device-side step counter (advanced by k2_scalars)
    MCO_CUDA_CHECK(cudaMemcpy(&T.t, &pl.d_tensors[idx].t, sizeof(int64_t),
                              cudaMemcpyDeviceToHost));
    T.rows_global = global_rows;
    T.numel_global = T.factored ? global_rows * T.cols : T.numel;
    T.weight = weight;
    MCO_CUDA_CHECK(cudaMemcpy(&pl.d_tensors[idx], &T, sizeof(TensorInfo),
                              cudaMemcpyHostToDevice));
  });
}

// One phase of apply_all (1: stats, 2: moments + sum u^2, 3: update).  A
// row-split caller all-reduces payload 0 after phase 1 and payload 1 after phase 2.
mco_status mco_adalomo_phase(mco_adalomo* h, int phase, void* flat_p, int pdt,
                             const void* flat_g, int gdt, double lr, void* stream) {
  return guard([&] {
    check_ada_dtypes(pdt, gdt);
    if (phase < 1 || phase > 3) throw Error(MCO_CONTRACT, "adalomo: phase must be 1, 2 or 3");
    DeviceGuard dg(h->plan.device);
    AdaLomoCall c{};
    c.t0 = 0;
    c.t1 = (int)h->plan.h_tensors.size();
    c.p = flat_p;
    c.p_dtype = pdt;
    c.g = flat_g;
    c.g_dtype = gdt;
    c.single = 0;
    c.lr = lr;
    c.use_clip = h->plan.cfg.has_clip_threshold ? 1 : 0;
    launch_adalomo_phase(h->plan, c, phase, (cudaStream_t)stream);
    if (phase == 3)
      for (auto& T : h->plan.h_tensors) T.t += 1;
  });
}

// which 0: stats payload (3 per tensor + column sums), 1: sum u^2 payload.
mco_status mco_adalomo_payload(mco_adalomo* h, int which, double** dev_ptr, uint64_t* len) {
  return guard([&] {
    if (which == 0) {
      *dev_ptr = h->plan.d_payload;
      *len = (uint64_t)h->plan.stats_len;
    } else if (which == 1) {
      *dev_ptr = h->plan.d_payload + h->plan.stats_len;
      *len = (uint64_t)h->plan.usq_len;
    } else {
      throw Error(MCO_CONTRACT, "adalomo: payload must be 0 or 1");
    }
  });
}

// optim.cpp:277-282 (fp64 state, as the reference)
mco_status mco_adalomo_state_bytes(const mco_adalomo* h, uint64_t* out) {
  return guard([&] { *out = (uint64_t)h->plan.state_len * sizeof(double); });
}

mco_status mco_adalomo_get_steps(const mco_adalomo* h, int idx, int64_t* t) {
  return guard([&] {
    if (idx < 0 || idx >= (int)h->plan.h_tensors.size())
      throw Error(MCO_CONTRACT, "adalomo: tensor index out of range");
    // the device counter is the truth (K2 advances it): steps replayed from a captured
    // CUDA graph count too, which a host mirror would miss
    DeviceGuard dg(h->plan.device);
    MCO_CUDA_CHECK(cudaDeviceSynchronize());
    const TensorInfo* dT = reinterpret_cast<const TensorInfo*>(h->plan.d_tensors) + idx;
    MCO_CUDA_CHECK(cudaMemcpy(t, &dT->t, sizeof(int64_t), cudaMemcpyDeviceToHost));
  });
}

mco_status mco_adalomo_buffer(mco_adalomo* h, int idx, int which, void** ptr, uint64_t* len) {
  return guard([&] {
    if (idx < 0 || idx >= (int)h->plan.h_tensors.size())
      throw Error(MCO_CONTRACT, "adalomo: tensor index out of range");
    const TensorInfo& T = h->plan.h_tensors[idx];
    int64_t off = -1, n = 0;
    if (which == 0 && T.factored) off = T.vrow_off, n = T.rows;
    if (which == 1 && T.factored) off = T.vcol_off, n = T.cols;
    if (which == 2 && !T.factored) off = T.vfull_off, n = T.numel;
    *ptr = off >= 0 ? (void*)(h->plan.d_state + off) : nullptr;
    *len = (uint64_t)n;
  });
}

// ---- ZeroPlan (parallel.cpp:20-34) -------------------------------------------------
mco_status mco_zero_plan(uint64_t total, int dp, int stage, uint64_t* part_sizes,
                         uint64_t* offsets) {
  return guard([&] {
    if (dp < 1) throw Error(MCO_CONFIG, "zero plan: dp_size must be >= 1");
    if (stage < 0 || stage > 3) throw Error(MCO_CONFIG, "zero plan: stage must be in 0..3");
    const uint64_t q = total / (uint64_t)dp, r = total % (uint64_t)dp;
    offsets[0] = 0;
    for (int i = 0; i < dp; ++i) {
      part_sizes[i] = q + ((uint64_t)i < r ? 1 : 0);  // ceil split, trailing smaller
      offsets[i + 1] = offsets[i] + part_sizes[i];
    }
  });
}

// ---- synthetic inputs --------------------------------------------------------------
mco_status mco_synth_fill(void* dst, int dtype, uint64_t n, uint64_t seed, uint32_t role,
                          uint32_t tensor, uint32_t step, int64_t cols, int scale_log2,
                          int zero_log2, int rowcol, void* stream) {
  return guard([&] {
    dtype_size(dtype);
    launch_synth(dst, dtype, n, synth_key(seed, role, tensor, step), cols, scale_log2, zero_log2,
                 rowcol, (cudaStream_t)stream);
  });
}

mco_status mco_sync(void* stream) {
  return guard([&] { MCO_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream)); });
}

mco_status mco_set_flat_variant(const char* name) {
  return guard([&] { set_flat_variant(name ? name : ""); });
}

const char* mco_flat_variant(void) { return flat_variant_name(); }

mco_status mco_device_count(int* out) {
  return guard([&] {
    *out = 0;
    const cudaError_t e = cudaGetDeviceCount(out);
    if (e != cudaSuccess) {
      *out = 0;
      cudaGetLastError();
    }
  });
}

}  // extern "C"
