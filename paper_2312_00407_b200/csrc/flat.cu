// Fused elementwise optimizer steps for sm_100a: AdamW / Lion / Adan / Sophia
// (optim.cpp:114-167), LOMO (optim.cpp:185-190), the LOMO global grad-norm
// reduction (optim.cpp:294-303) and the synthetic-input generator.
//
// One pass per step: every param / grad / state element is read once and
// written at most once (HBM roofline: SURVEY.md 8(d) bytes per param).
// Dispatch (launch_flat_step / launch_lomo): fp32 calls go to the warp-specialised
// cp.async.bulk pipeline of flat_tma.cu (the default "tma" variant); everything
// else -- bf16 gradients, f64 state, unaligned ZeRO shard edges, the "ldg" variant --
// runs the kernels here: persistent grid-stride CTAs (SMs x resident CTAs), 256-bit
// LDG/STG (ld.global.v8.f32 -> LDG.E.256), L1 no-allocate + L2 evict-first for the
// streams, U vectors in flight per thread.  Compiled with --fmad=false: the
// arithmetic is the reference's operation order, no fused multiply-add, IEEE
// division and square root -- bit-identical to oracle/mco_oracle.c, whichever
// variant moves the data.
#include <algorithm>
#include <atomic>
#include <initializer_list>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>

#include "flat_tma.h"
#include "kernels.h"
#include "launch.cuh"
#include "update.cuh"

namespace mco {
namespace {

using namespace upd;
using flatk::aligned;
using flatk::grid_for;
using flatk::kThreads;

// MINB > 1 caps registers so MINB CTAs fit per SM (Adan streams 11 buffers).
// WV: elements per vector access (8 f32 = 256-bit, 4 f32 = 128-bit, 4 f64 = 256-bit).
__device__ __forceinline__ void prefetch_l2(const void* ptr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}

// PFD > 0: each warp bulk-prefetches (cp.async.bulk.prefetch.L2) the 1 KB segments of
// every input stream it will load PFD grid-stride iterations later, so the LDGs of
// that iteration hit L2 (more bytes in flight than the register file holds).
// DEV: graph mode -- the step scalars are derived from the device step counter
// (common.cuh step_consts / graph_bump) instead of the by-value kv.
template <int KIND, typename T, typename GT, bool MIXED, int U, int MINB = 1,
          int WV = Vec<T>::W, int PFD = 0, bool DEV = false>
__global__ void __launch_bounds__(kThreads, MINB)
    flat_step_kernel(T* __restrict__ p, const GT* __restrict__ g, T* __restrict__ s0,
                     T* __restrict__ s1, T* __restrict__ s2, T* __restrict__ s3,
                     uint16_t* __restrict__ pout, uint64_t nvec, uint64_t n,
                     const StepConsts<T> kv, const GraphStep gs) {
  const StepConsts<T> k = step_consts<DEV>(kv, gs);
  constexpr int W = WV;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = tid; base < nvec; base += stride * U) {
    if constexpr (PFD > 0) {
      constexpr int NIN = KIND == K_ADAN ? 6 : (reads_s1(KIND) ? 4 : 3);
      const int lane = threadIdx.x & 31;
      const int j = lane % NIN, u = lane / NIN;
      const uint64_t w0 = base - lane + (uint64_t)PFD * stride * U + (uint64_t)u * stride;
      if (u < U && w0 + 32 <= nvec && !(KIND == K_ADAN && j == 5 && k.first)) {
        const uint64_t e = w0 * W;
        if (j == 1) {
          prefetch_l2(g + e, 32 * W * sizeof(GT));
        } else {
          const T* src = j == 0 ? p : j == 2 ? s0 : j == 3 ? s1 : j == 4 ? s2 : s3;
          prefetch_l2(src + e, 32 * W * sizeof(T));
        }
      }
    }
    T pv[U][W], gv[U][W], a[U][W], b[U][W], c[U][W], d[U][W];
    // issue every load of the U vectors before any arithmetic
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = base + (uint64_t)u * stride;
      if (vi < nvec) {
        const uint64_t e = vi * W;
        ld_stream(p + e, pv[u]);
        load_grad(g + e, gv[u]);
        ld_stream(s0 + e, a[u]);
        if constexpr (reads_s1(KIND)) ld_stream(s1 + e, b[u]);
        if constexpr (KIND == K_ADAN) {
          ld_stream(s2 + e, c[u]);
          if (!k.first) ld_stream(s3 + e, d[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = base + (uint64_t)u * stride;
      if (vi < nvec) {
        const uint64_t e = vi * W;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          if constexpr (KIND != K_ADAN) c[u][j] = d[u][j] = T(0);
          if constexpr (KIND == K_ADAN) {
            if (k.first) d[u][j] = T(0);
          }
          if constexpr (!reads_s1(KIND)) b[u][j] = T(0);
          update<KIND, T>(pv[u][j], gv[u][j], a[u][j], b[u][j], c[u][j], d[u][j], k);
        }
        st_stream(p + e, pv[u]);
        st_stream(s0 + e, a[u]);
        if constexpr (KIND == K_ADAMW || KIND == K_ADAN) st_stream(s1 + e, b[u]);
        if constexpr (KIND == K_SOPHIA) {
          if (k.refresh) st_stream(s1 + e, b[u]);
        }
        if constexpr (KIND == K_ADAN) {
          st_stream(s2 + e, c[u]);
          st_stream(s3 + e, d[u]);
        }
        if constexpr (MIXED) {
          if constexpr (W == 8) {
            st_stream_bf16x8(pout + e, pv[u]);
          } else {
#pragma unroll
            for (int j = 0; j < W; j += 2)
              *reinterpret_cast<uint32_t*>(pout + e + j) = f2bf2_bits(pv[u][j], pv[u][j + 1]);
          }
        }
      }
    }
  }
  // scalar remainder (unaligned buffers take this path for every element)
  for (uint64_t e = nvec * W + tid; e < n; e += stride) {
    T pp = p[e], gg = (T)load_grad1(g + e), aa = s0[e], bb = T(0), cc = T(0), dd = T(0);
    if constexpr (reads_s1(KIND)) bb = s1[e];
    if constexpr (KIND == K_ADAN) {
      cc = s2[e];
      if (!k.first) dd = s3[e];
    }
    update<KIND, T>(pp, gg, aa, bb, cc, dd, k);
    p[e] = pp;
    s0[e] = aa;
    if constexpr (KIND == K_ADAMW || KIND == K_ADAN) s1[e] = bb;
    if constexpr (KIND == K_SOPHIA) {
      if (k.refresh) s1[e] = bb;
    }
    if constexpr (KIND == K_ADAN) {
      s2[e] = cc;
      s3[e] = dd;
    }
    if constexpr (MIXED) pout[e] = (uint16_t)f2bf_bits((float)pp);
  }
  graph_bump<DEV>(gs);
}

// Software-pipelined variant: the next vector's loads are issued before the
// current vector's arithmetic (static ping-pong buffers, no local memory).
template <int KIND, typename T, typename GT>
struct PfBuf {
  static constexpr int W = Vec<T>::W;
  T p[W], g[W], a[W], b[W], c[W], d[W];
  __device__ __forceinline__ void load(const T* pp, const GT* gg, const T* s0, const T* s1,
                                       const T* s2, const T* s3, uint64_t e, bool first) {
    ld_stream(pp + e, p);
    load_grad(gg + e, g);
    ld_stream(s0 + e, a);
    if constexpr (reads_s1(KIND)) ld_stream(s1 + e, b);
    if constexpr (KIND == K_ADAN) {
      ld_stream(s2 + e, c);
      if (!first) ld_stream(s3 + e, d);
    }
  }
  __device__ __forceinline__ void run_store(T* pp, T* s0, T* s1, T* s2, T* s3, uint16_t* pout,
                                            uint64_t e, const StepConsts<T>& k, bool mixed) {
#pragma unroll
    for (int j = 0; j < W; ++j) {
      if constexpr (KIND != K_ADAN) c[j] = d[j] = T(0);
      if constexpr (KIND == K_ADAN) {
        if (k.first) d[j] = T(0);
      }
      if constexpr (!reads_s1(KIND)) b[j] = T(0);
      update<KIND, T>(p[j], g[j], a[j], b[j], c[j], d[j], k);
    }
    st_stream(pp + e, p);
    st_stream(s0 + e, a);
    if constexpr (KIND == K_ADAMW || KIND == K_ADAN) st_stream(s1 + e, b);
    if constexpr (KIND == K_SOPHIA) {
      if (k.refresh) st_stream(s1 + e, b);
    }
    if constexpr (KIND == K_ADAN) {
      st_stream(s2 + e, c);
      st_stream(s3 + e, d);
    }
    if constexpr (sizeof(T) == 4) {
      if (mixed) st_stream_bf16x8(pout + e, p);
    }
  }
};

template <int KIND, typename T, typename GT, bool MIXED>
__global__ void __launch_bounds__(kThreads)
    flat_step_kernel_pf(T* __restrict__ p, const GT* __restrict__ g, T* __restrict__ s0,
                        T* __restrict__ s1, T* __restrict__ s2, T* __restrict__ s3,
                        uint16_t* __restrict__ pout, uint64_t nvec, uint64_t n,
                        const StepConsts<T> k, const GraphStep) {
  constexpr int W = Vec<T>::W;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  PfBuf<KIND, T, GT> A, B;
  uint64_t vi = tid;
  if (vi < nvec) A.load(p, g, s0, s1, s2, s3, vi * W, k.first);
  while (vi < nvec) {
    const uint64_t v1 = vi + stride;
    if (v1 < nvec) B.load(p, g, s0, s1, s2, s3, v1 * W, k.first);
    A.run_store(p, s0, s1, s2, s3, pout, vi * W, k, MIXED);
    if (v1 >= nvec) break;
    const uint64_t v2 = v1 + stride;
    if (v2 < nvec) A.load(p, g, s0, s1, s2, s3, v2 * W, k.first);
    B.run_store(p, s0, s1, s2, s3, pout, v1 * W, k, MIXED);
    vi = v2;
  }
  for (uint64_t e = nvec * W + tid; e < n; e += stride) {
    T pp = p[e], gg = (T)load_grad1(g + e), aa = s0[e], bb = T(0), cc = T(0), dd = T(0);
    if constexpr (reads_s1(KIND)) bb = s1[e];
    if constexpr (KIND == K_ADAN) {
      cc = s2[e];
      if (!k.first) dd = s3[e];
    }
    update<KIND, T>(pp, gg, aa, bb, cc, dd, k);
    p[e] = pp;
    s0[e] = aa;
    if constexpr (KIND == K_ADAMW || KIND == K_ADAN) s1[e] = bb;
    if constexpr (KIND == K_SOPHIA) {
      if (k.refresh) s1[e] = bb;
    }
    if constexpr (KIND == K_ADAN) {
      s2[e] = cc;
      s3[e] = dd;
    }
    if constexpr (MIXED) pout[e] = (uint16_t)f2bf_bits((float)pp);
  }
}

// ---- LOMO ---------------------------------------------------------------------


template <typename PT, typename GT>
__global__ void __launch_bounds__(kThreads)
    lomo_kernel(PT* __restrict__ p, const GT* __restrict__ g, uint64_t nvec, uint64_t n,
                double lr, double scale, const double* __restrict__ sumsq, double clip) {
  using T = typename std::conditional<std::is_same<PT, double>::value, double, float>::type;
  constexpr int W = lomo_width<PT, GT>();
  pdl_wait();
  const T f = lomo_factor<T>(lr, scale, sumsq, clip);
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  constexpr int U = 2;
  for (uint64_t base = tid; base < nvec; base += stride * U) {
    T pv[U][W], gv[U][W];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = base + (uint64_t)u * stride;
      if (vi < nvec) {
        if constexpr (W == 16) {  // bf16 params and grads: one 256-bit access each
          ld_stream_bf16x16(p + vi * W, pv[u]);
          ld_stream_ro_bf16x16(g + vi * W, gv[u]);
        } else {
          if constexpr (std::is_same<PT, uint16_t>::value)
            ld_stream_bf16x8(p + vi * W, pv[u]);
          else
            ld_stream(p + vi * W, pv[u]);
          load_grad(g + vi * W, gv[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = base + (uint64_t)u * stride;
      if (vi < nvec) {
#pragma unroll
        for (int j = 0; j < W; ++j) pv[u][j] = pv[u][j] - f * gv[u][j];
        if constexpr (W == 16)
          st_stream_bf16x16(p + vi * W, pv[u]);
        else if constexpr (std::is_same<PT, uint16_t>::value)
          st_stream_bf16x8(p + vi * W, pv[u]);
        else
          st_stream(p + vi * W, pv[u]);
      }
    }
  }
  for (uint64_t e = nvec * W + tid; e < n; e += stride) {
    if constexpr (std::is_same<PT, uint16_t>::value) {
      p[e] = (uint16_t)f2bf_bits(bf2f(p[e]) - f * load_grad1(g + e));
    } else {
      p[e] = p[e] - f * (T)load_grad1(g + e);
    }
  }
}

// ---- deterministic sum of squares --------------------------------------------
// Per-thread fp64 accumulation in a fixed element order, fixed-order block
// reduction, per-block partials, and the last CTA to finish sums the partials
// in block order.  Bit-reproducible for a given (n, grid).
constexpr int kSumsqMaxBlocks = 1024;

template <typename XT>
constexpr int sumsq_width() {
  return std::is_same<XT, double>::value ? 4 : (std::is_same<XT, uint16_t>::value ? 16 : 8);
}

template <typename XT>
__global__ void __launch_bounds__(kThreads)
    sumsq_kernel(const XT* __restrict__ x, uint64_t nvec, uint64_t n, double* __restrict__ out,
                 int accumulate, double* __restrict__ partials, unsigned* __restrict__ counter) {
  __shared__ double scratch[32];
  __shared__ bool is_last;
  constexpr int W = sumsq_width<XT>();
  pdl_wait();
  using LT = typename std::conditional<std::is_same<XT, double>::value, double, float>::type;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (uint64_t vi = tid; vi < nvec; vi += stride) {
    LT v[W];
    if constexpr (W == 16)
      ld_stream_ro_bf16x16(x + vi * W, v);
    else
      load_grad(x + vi * W, v);
#pragma unroll
    for (int j = 0; j < W; ++j) acc += (double)v[j] * (double)v[j];
  }
  for (uint64_t e = nvec * W + tid; e < n; e += stride) {
    const double v = (double)load_grad1(x + e);
    acc += v * v;
  }
  const double bsum = block_sum(acc, scratch);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bsum;
    __threadfence();
    const unsigned ticket = atomicAdd(counter, 1u);
    is_last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
    double s = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
      s += ((volatile double*)partials)[b];
    s = block_sum(s, scratch);
    if (threadIdx.x == 0) {
      *out = accumulate ? *out + s : s;
      *counter = 0u;  // re-arm for the next launch on this stream
    }
  }
}

// ---- synthetic generator (oracle/mco_oracle.c restates it) ---------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

__global__ void synth_kernel(void* dst, int dtype, uint64_t n, uint64_t key, int64_t cols,
                             int scale_log2, int zero_log2, int rowcol) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t x = fmix64(key + (i + 1) * kGolden);
    double v = dtype == MCO_BF16 ? (double)((int32_t)(x >> 56) - 128) * 0x1.0p-7
                                 : (double)((int32_t)(x >> 40) - (1 << 23)) * 0x1.0p-23;
    if (zero_log2 > 0 && (x & ((1ULL << zero_log2) - 1)) == 0) v = 0.0;
    int e = scale_log2;
    if (rowcol && cols > 0) {
      const uint64_t r = i / (uint64_t)cols, c = i % (uint64_t)cols;
      e += (int)(fmix64(key ^ (0xA5A5A5A5A5A5A5A5ULL + r * kGolden)) >> 62) - 1;
      e += (int)(fmix64(key ^ (0x5A5A5A5A5A5A5A5AULL + c * kGolden)) >> 62) - 1;
    }
    v = ldexp(v, e);
    if (dtype == MCO_F32)
      static_cast<float*>(dst)[i] = (float)v;
    else if (dtype == MCO_F64)
      static_cast<double*>(dst)[i] = v;
    else
      static_cast<uint16_t*>(dst)[i] = (uint16_t)(__float_as_uint((float)v) >> 16);
  }
}

// ---- data-movement variant of the fp32 stored-state kernels -------------------------
// mco_set_flat_variant(name) or MCO_FLAT_VARIANT (read at first use).  Default "tma":
// the cp.async.bulk / mbarrier pipeline (flat_tma.cu) when the call is eligible (fp32
// params / grads / state, 16 B aligned, >= one tile), else the LDG kernel.  The rest
// are the measured alternatives kept for A/B runs; every variant
// produces the same bits.
enum Variant {
  V_TMA, V_LDG, V_W4M4, V_W8M4, V_W4M1, V_PF, V_U1M3, V_U2M3, V_L2PF1, V_L2PF2, V_L2PF4,
  V_TMA_S3, V_TMA_S5, V_TMA24, V_TMA8, V_TMA_E2, V_TMA_HINT, V_TMA24_E2, V_TMA_DS, V_TMA_S2, V_COUNT
};
const char* const kVariantNames[V_COUNT] = {
    "tma",   "ldg",   "w4m4",  "w8m4",   "w4m1",   "pf",    "u1m3", "u2m3",
    "l2pf1", "l2pf2", "l2pf4", "tma_s3", "tma_s5", "tma24", "tma8",
    "tma_e2", "tma_hint", "tma24_e2", "tma_ds", "tma_s2"};
std::atomic<int> g_variant{-1};

int parse_flat_variant(const char* name) {
  const std::string s(name ? name : "");
  if (s.empty()) return V_TMA;
  for (int i = 0; i < V_COUNT; ++i)
    if (s == kVariantNames[i]) return i;
  return -1;
}

int flat_variant() {
  int v = g_variant.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("MCO_FLAT_VARIANT");
    v = e ? std::max(parse_flat_variant(e), 0) : 0;
    g_variant.store(v, std::memory_order_relaxed);
  }
  return v;
}


template <int KIND, typename T, typename GT, bool MIXED>
void run_flat(const FlatArgs& a, const StepConsts<T>& k, cudaStream_t st) {
  constexpr int U = (KIND == K_ADAN) ? 1 : 2;
  // 3 resident CTAs (768 threads) per SM: registers capped at 80 (ncu r01: Adan at
  // 84 registers fell to 2 CTAs/SM and 0.88 of the HBM copy bandwidth)
  constexpr int MINB = (sizeof(T) == 4 && (KIND == K_ADAN || KIND == K_LION)) ? 3 : 1;
  int W = Vec<T>::W;
  int u_eff = U;
  auto kern = flat_step_kernel<KIND, T, GT, MIXED, U, MINB>;
  const bool dev_step = a.gs.d != nullptr;
  if (dev_step) kern = flat_step_kernel<KIND, T, GT, MIXED, U, MINB, Vec<T>::W, 0, true>;
  if constexpr (sizeof(T) == 4) {
    const int variant = dev_step ? (flat_variant() == V_LDG ? V_LDG : V_TMA) : flat_variant();
    int tma_cfg = -1;  // flat_tma.h configurations
    switch (variant) {
      // Adan: 3 stages (7B, same box: 45.52 vs 46.62 ms at 4; the other kinds lose 15-30 %
      // with 3 -- AdamW 34.2 vs 29.2 ms -- and keep 4)
      case V_TMA: tma_cfg = KIND == K_ADAN ? 1 : 0; break;
      case V_TMA_S3: tma_cfg = 1; break;
      case V_TMA_S5: tma_cfg = 2; break;
      case V_TMA24: tma_cfg = 3; break;
      case V_TMA8: tma_cfg = 4; break;
      case V_TMA_E2: tma_cfg = 5; break;
      case V_TMA_HINT: tma_cfg = 6; break;
      case V_TMA24_E2: tma_cfg = 7; break;
      case V_TMA_DS: tma_cfg = 8; break;
      case V_TMA_S2: tma_cfg = 9; break;
      case V_W4M4: kern = flat_step_kernel<KIND, T, GT, MIXED, U, 4, 4>; W = 4; break;
      case V_W8M4: kern = flat_step_kernel<KIND, T, GT, MIXED, U, 4, 8>; break;
      case V_W4M1: kern = flat_step_kernel<KIND, T, GT, MIXED, U, 1, 4>; W = 4; break;
      case V_PF: kern = flat_step_kernel_pf<KIND, T, GT, MIXED>; break;
      case V_U1M3: kern = flat_step_kernel<KIND, T, GT, MIXED, 1, 3>; u_eff = 1; break;
      case V_U2M3: kern = flat_step_kernel<KIND, T, GT, MIXED, 2, 3>; u_eff = 2; break;
      case V_L2PF1: kern = flat_step_kernel<KIND, T, GT, MIXED, U, MINB, 8, 1>; break;
      case V_L2PF2: kern = flat_step_kernel<KIND, T, GT, MIXED, U, MINB, 8, 2>; break;
      case V_L2PF4: kern = flat_step_kernel<KIND, T, GT, MIXED, U, MINB, 8, 4>; break;
      default: break;  // V_LDG
    }
    static const int cfg_force = [] {  // MCO_TMA_CFG=<id>: force a configuration (A/B)
      const char* e = getenv("MCO_TMA_CFG");
      return e ? atoi(e) : -1;
    }();
    if (tma_cfg >= 0 && cfg_force >= 0 && !dev_step) tma_cfg = cfg_force;
    if (tma_cfg >= 0 && flat_tma_eligible(a, tma_cfg)) {
      launch_flat_tma(a, k, st, tma_cfg);
      return;
    }
  }
  bool vec = aligned(a.p, sizeof(T) * W) && aligned(a.g, sizeof(GT) * W);
  for (int i = 0; i < 4; ++i) vec = vec && aligned(a.s[i], sizeof(T) * W);
  if (MIXED) vec = vec && aligned(a.p_out_bf16, 2 * W);
  const uint64_t nvec = vec ? a.n / W : 0;
  const uint64_t items = nvec ? (nvec + u_eff - 1) / u_eff : a.n;
  const int dev = current_device();
  const int grid = grid_for(kern, std::max<uint64_t>(items, 1), dev);
  kern<<<grid, kThreads, 0, st>>>((T*)a.p, (const GT*)a.g, (T*)a.s[0], (T*)a.s[1], (T*)a.s[2],
                                  (T*)a.s[3], a.p_out_bf16, nvec, a.n, k, a.gs);
  launch_check("flat_step_kernel");
}

template <int KIND>
void dispatch_dtypes(const FlatArgs& a, const StepConsts<float>& kf, const StepConsts<double>& kd,
                     cudaStream_t st) {
  const bool mixed = a.p_out_bf16 != nullptr;
  if (a.state_dtype == MCO_F64) {
    if (a.p_dtype != MCO_F64 || a.g_dtype != MCO_F64 || mixed)
      throw Error(MCO_CONTRACT, "flat step: f64 state takes f64 params and grads");
    run_flat<KIND, double, double, false>(a, kd, st);
    return;
  }
  if (a.p_dtype != MCO_F32)
    throw Error(MCO_CONTRACT, "flat step: f32 state takes f32 (master) params");
  if (a.g_dtype == MCO_F32) {
    if (mixed)
      run_flat<KIND, float, float, true>(a, kf, st);
    else
      run_flat<KIND, float, float, false>(a, kf, st);
  } else if (a.g_dtype == MCO_BF16) {
    if (mixed)
      run_flat<KIND, float, uint16_t, true>(a, kf, st);
    else
      run_flat<KIND, float, uint16_t, false>(a, kf, st);
  } else {
    throw Error(MCO_CONTRACT, "flat step: f32 state takes f32 or bf16 grads");
  }
}

template <typename PT, typename GT>
void run_lomo(void* p, const void* g, uint64_t n, double lr, double scale, const double* sumsq,
              double clip, cudaStream_t st) {
  constexpr int W = lomo_width<PT, GT>();
  auto kern = lomo_kernel<PT, GT>;
  const bool vec = aligned(p, sizeof(PT) * W) && aligned(g, sizeof(GT) * W);
  const uint64_t nvec = vec ? n / W : 0;
  const uint64_t items = nvec ? (nvec + 1) / 2 : n;
  const int grid = grid_for(kern, std::max<uint64_t>(items, 1), current_device());
  launch_pdl(kern, grid, kThreads, st, (PT*)p, (const GT*)g, nvec, n, lr, scale, sumsq, clip);
  launch_check("lomo_kernel");
}

template <typename XT>
void run_sumsq(const void* x, uint64_t n, double* out, int accumulate, double* partials,
               unsigned* counter, int dev, cudaStream_t st) {
  constexpr int W = sumsq_width<XT>();
  auto kern = sumsq_kernel<XT>;
  const bool vec = aligned(x, sizeof(XT) * W);
  const uint64_t nvec = vec ? n / W : 0;
  int grid = grid_for(kern, std::max<uint64_t>(nvec ? nvec : n, 1), dev);
  grid = std::min(grid, kSumsqMaxBlocks);
  launch_pdl(kern, grid, kThreads, st, (const XT*)x, nvec, n, out, accumulate, partials, counter);
  launch_check("sumsq_kernel");
}

size_t dtype_bytes(int dt) { return dt == MCO_F64 ? 8 : dt == MCO_BF16 ? 2 : 4; }

// Element phase shared by every stream of a launch: (address / element size) mod 8,
// or -1 when the streams disagree (or one is not element-aligned).  With a common
// nonzero phase -- a ZeRO shard at an odd element offset, with its state laid out to
// match (abi.cpp) -- the first 8 - phase elements go to a small launch of their own and
// the rest starts 32 B-aligned on the vector / TMA paths (else every element of the
// shard took the scalar path: 2-2.6x slower).
int common_phase(std::initializer_list<std::pair<const void*, size_t>> ptrs) {
  int ph = -1;
  for (const auto& [ptr, es] : ptrs) {
    if (!ptr) continue;
    const uintptr_t u = (uintptr_t)ptr;
    if (u % es) return -1;
    const int q = (int)((u / es) % 8);
    if (ph >= 0 && q != ph) return -1;
    ph = q;
  }
  return ph < 0 ? 0 : ph;
}

template <typename T>
T* advance(T* ptr, uint64_t elems, size_t es) {
  return ptr ? (T*)((char*)ptr + elems * es) : nullptr;
}

void launch_flat_one(const FlatArgs& a, const StepConsts<float>& kf,
                     const StepConsts<double>& kd, cudaStream_t st) {
  switch (a.kind) {
    case MCO_ADAMW: dispatch_dtypes<K_ADAMW>(a, kf, kd, st); break;
    case MCO_LION: dispatch_dtypes<K_LION>(a, kf, kd, st); break;
    case MCO_ADAN: dispatch_dtypes<K_ADAN>(a, kf, kd, st); break;
    case MCO_SOPHIA: dispatch_dtypes<K_SOPHIA>(a, kf, kd, st); break;
    default: throw Error(MCO_CONTRACT, "FlatOptimizer: fused kind");
  }
}

void launch_lomo_one(void* p, int p_dtype, const void* g, int g_dtype, uint64_t n, double lr,
                     double scale, const double* dev_sumsq, double clip, cudaStream_t st);

}  // namespace

void launch_flat_step(const FlatArgs& a, const StepConsts<float>& kf,
                      const StepConsts<double>& kd, cudaStream_t st) {
  if (a.n == 0) {
    if (a.gs.d) launch_flat_graph_bump(a.gs.d, st);
    return;
  }
  const size_t ps = dtype_bytes(a.p_dtype), gs = dtype_bytes(a.g_dtype),
               ss = dtype_bytes(a.state_dtype);
  int ph = common_phase({{a.p, ps}, {a.g, gs}, {a.s[0], ss}, {a.s[1], ss},
                         {a.s[2], ss}, {a.s[3], ss}, {a.p_out_bf16, 2}});
  if (ph < 0 && ((uintptr_t)a.g % gs) == 0) {
    // only the (read-only) gradient disagrees -- a gradient buffer at another offset than
    // the parameters, e.g. a reduce-scattered shard against an odd ZeroPlan slice: align
    // the other streams as below, the TMA pipeline reads the gradient shifted
    ph = common_phase({{a.p, ps}, {a.s[0], ss}, {a.s[1], ss}, {a.s[2], ss}, {a.s[3], ss},
                       {a.p_out_bf16, 2}});
    if (ph < 0 && !a.p_out_bf16 && a.state_dtype == MCO_F32 && a.p_dtype == MCO_F32 &&
        flat_variant() == V_TMA) {
      // parameters and state disagree too (a caller-laid-out state): a one-tensor list
      // step -- the list pipeline reads and writes every stream at its own phase
      FlatListArgs la{};
      la.kind = a.kind;
      la.state_dtype = a.state_dtype;
      la.p_dtype = a.p_dtype;
      la.g_dtype = a.g_dtype;
      la.count = 1;
      void* pp[1] = {a.p};
      const void* gp[1] = {a.g};
      const uint64_t len[1] = {a.n};
      la.p = pp;
      la.g = gp;
      la.len = len;
      for (int i = 0; i < 4; ++i) la.s[i] = a.s[i];
      la.gs = a.gs;
      launch_flat_step_list(la, kf, kd, st);
      return;
    }
  }
  if (ph <= 0 || a.n <= (uint64_t)(8 - ph)) {
    launch_flat_one(a, kf, kd, st);
    return;
  }
  const uint64_t head = 8 - ph;
  FlatArgs h = a, b = a;
  h.gs.bump = 0;  // graph mode: the body launch advances the step
  h.n = head;
  b.n = a.n - head;
  b.p = advance(a.p, head, ps);
  b.g = advance(a.g, head, gs);
  for (int i = 0; i < 4; ++i) b.s[i] = advance(a.s[i], head, ss);
  b.p_out_bf16 = advance(a.p_out_bf16, head, 2);
  launch_flat_one(h, kf, kd, st);
  launch_flat_one(b, kf, kd, st);
}

namespace {
__global__ void flat_graph_bump(FlatGraphDev* d) { d->t += 1; }
}  // namespace

void launch_flat_graph_bump(FlatGraphDev* d, cudaStream_t st) {
  flat_graph_bump<<<1, 1, 0, st>>>(d);
  launch_check("flat_graph_bump");
}

void launch_lomo(void* p, int p_dtype, const void* g, int g_dtype, uint64_t n, double lr,
                 double scale, const double* dev_sumsq, double clip, cudaStream_t st) {
  if (n == 0) return;
  const size_t ps = dtype_bytes(p_dtype), gs = dtype_bytes(g_dtype);
  int ph = common_phase({{p, ps}, {g, gs}});
  if (ph < 0 && ((uintptr_t)g % gs) == 0) ph = common_phase({{p, ps}});  // gradient read shifted
  if (ph <= 0 || n <= (uint64_t)(8 - ph)) {
    launch_lomo_one(p, p_dtype, g, g_dtype, n, lr, scale, dev_sumsq, clip, st);
    return;
  }
  const uint64_t head = 8 - ph;
  launch_lomo_one(p, p_dtype, g, g_dtype, head, lr, scale, dev_sumsq, clip, st);
  launch_lomo_one(advance(p, head, ps), p_dtype, advance(g, head, gs), g_dtype, n - head, lr,
                  scale, dev_sumsq, clip, st);
}

namespace {

void launch_lomo_one(void* p, int p_dtype, const void* g, int g_dtype, uint64_t n, double lr,
                     double scale, const double* dev_sumsq, double clip, cudaStream_t st) {
  const int variant = flat_variant();
  // LOMO's 16 KB (fp32) stages want 8 in flight (measured: 4 -> 0.95, 8 -> 1.02 of the
  // copy bandwidth); "tma_s3" / "tma_s5" select 4 / 12 for A/B runs
  if ((variant == V_TMA || variant == V_TMA_S3 || variant == V_TMA_S5) &&
      lomo_tma_eligible(p, p_dtype, g, g_dtype, n)) {
    launch_lomo_tma(p, p_dtype, g, n, lr, scale, dev_sumsq, clip, st,
                    variant == V_TMA_S3 ? 4 : variant == V_TMA_S5 ? 12 : 8);
    return;
  }
  if (p_dtype == MCO_F32 && g_dtype == MCO_F32)
    run_lomo<float, float>(p, g, n, lr, scale, dev_sumsq, clip, st);
  else if (p_dtype == MCO_F32 && g_dtype == MCO_BF16)
    run_lomo<float, uint16_t>(p, g, n, lr, scale, dev_sumsq, clip, st);
  else if (p_dtype == MCO_BF16 && g_dtype == MCO_BF16)
    run_lomo<uint16_t, uint16_t>(p, g, n, lr, scale, dev_sumsq, clip, st);
  else if (p_dtype == MCO_F64 && g_dtype == MCO_F64)
    run_lomo<double, double>(p, g, n, lr, scale, dev_sumsq, clip, st);
  else
    throw Error(MCO_CONTRACT, "lomo_apply: unsupported param/grad dtype pair");
}

}  // namespace

size_t sumsq_ws_bytes() { return kSumsqMaxBlocks * sizeof(double) + 256; }

void launch_sumsq(const void* x, int dtype, uint64_t n, double* out, int accumulate, void* ws,
                  cudaStream_t st) {
  double* partials = (double*)ws;
  unsigned* counter = (unsigned*)((char*)ws + kSumsqMaxBlocks * sizeof(double));
  const int dev = current_device();
  if (dtype == MCO_F32)
    run_sumsq<float>(x, n, out, accumulate, partials, counter, dev, st);
  else if (dtype == MCO_BF16)
    run_sumsq<uint16_t>(x, n, out, accumulate, partials, counter, dev, st);
  else if (dtype == MCO_F64)
    run_sumsq<double>(x, n, out, accumulate, partials, counter, dev, st);
  else
    throw Error(MCO_CONTRACT, "sumsq: unsupported dtype");
}

uint64_t synth_key(uint64_t seed, uint32_t role, uint32_t tensor, uint32_t step) {
  const uint64_t a = fmix64(seed + (uint64_t)role * kGolden);
  return fmix64(a ^ (((uint64_t)tensor << 32) | (uint64_t)step));
}

void launch_synth(void* dst, int dtype, uint64_t n, uint64_t key, int64_t cols, int scale_log2,
                  int zero_log2, int rowcol, cudaStream_t st) {
  if (n == 0) return;
  const int dev = current_device();
  const uint64_t blocks = std::min<uint64_t>((n + kThreads - 1) / kThreads,
                                             (uint64_t)device_info(dev).sms * 8);
  synth_kernel<<<(unsigned)blocks, kThreads, 0, st>>>(dst, dtype, n, key, cols, scale_log2,
                                                      zero_log2, rowcol);
  launch_check("synth_kernel");
}

void set_flat_variant(const char* name) {
  const int v = parse_flat_variant(name);
  if (v < 0) throw Error(MCO_CONFIG, std::string("unknown flat-kernel variant '") + name + "'");
  g_variant.store(v, std::memory_order_relaxed);
}

const char* flat_variant_name() { return kVariantNames[flat_variant()]; }

}  // namespace mco
