// C-ABI (include/mco.h) over the sm_100a kernels: the drop-in boundary for
// minicollie::optim (optim.hpp).  Host logic here restates the reference's
// non-kernel behaviour -- kind names, defaults, validation, error messages,
// state accounting, step counter, buffer naming -- citing optim.cpp lines.
// This unit: errors, kinds / config, state bytes, ZeroPlan, synthetic inputs and the
// shared helpers (abi_internal.h); abi_flat.cpp and abi_adalomo.cpp hold the handles.
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

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "abi_internal.h"

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

void host_trace(const char* what) {
  static const bool on = [] {
    const char* e = getenv("MCO_HOST_TRACE");
    return e && atoi(e) != 0;
  }();
  if (!on) return;
  thread_local std::chrono::steady_clock::time_point t0;
  const auto now = std::chrono::steady_clock::now();
  if (what)
    fprintf(stderr, "[mco host] %s: %.1f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t0).count());
  t0 = now;
}

static std::mutex g_stage_mu;
static std::unordered_map<int, HostStage*> g_stages;

void host_release_all() {
  std::vector<std::pair<int, HostStage*>> all;
  {
    std::lock_guard<std::mutex> lock(g_stage_mu);  // not held below: a running call takes
    all.assign(g_stages.begin(), g_stages.end());  // gres_mu, then g_stage_mu
  }
  for (auto& kv : all) {
    HostStage& hs = *kv.second;
    std::lock_guard<std::mutex> g(hs.gres_mu);  // waits for a running call
    if (hs.gres) {
      DeviceGuard dg(kv.first);
      MCO_CUDA_CHECK(cudaFree(hs.gres));
      hs.gres = nullptr;
      hs.gres_bytes = 0;
    }
  }
}

HostStage& host_stage(int dev) {
  std::lock_guard<std::mutex> lock(g_stage_mu);
  auto& s = g_stages[dev];
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

}  // namespace mco

using namespace mco;

extern "C" {


const char* mco_last_error(void) { return g_err.c_str(); }
const char* mco_version(void) { return "mco 0.1 (sm_100a)"; }
uint64_t mco_launch_count(void) { return g_launches.load(); }
mco_status mco_host_release(void) { return guard([&] { host_release_all(); }); }

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
