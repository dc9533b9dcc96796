// Shared device helpers for the sm_100a optimizer kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "mco.h"

namespace mco {

// ---- host-side error plumbing ------------------------------------------------
// Exceptions carry an mco_status; the C-ABI layer (abi.cpp) converts them.
struct Error : std::runtime_error {
  mco_status status;
  Error(mco_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(MCO_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define MCO_CUDA_CHECK(x) ::mco::cuda_check((x), #x)

// Counts our own kernel launches (bench.py reports it as gpu_launches).
void note_launch(uint64_t n = 1);
inline void launch_check(const char* what) {
  note_launch();
  cuda_check(cudaGetLastError(), what);
}

// ---- Programmatic Dependent Launch ------------------------------------------------
// Kernels of dependent chains (AdaLomo's passes, LOMO's sum of squares -> update, the
// per-tensor hook forms) are launched with programmatic stream serialization and
// start with griddepcontrol.wait: the launch and CTA rasterisation overlap the tail of
// the previous kernel in the stream, while no CTA touches memory before that kernel
// has completed and flushed, so stream-order semantics are unchanged.
// Optional early trigger (griddepcontrol.launch_dependents once every CTA has passed its
// wait): the next PDL kernel's CTAs are rasterised while this grid runs and sit in their
// own wait.  Every PDL grid here fits in one wave, so it is safe, but the parked CTAs
// cost more than the launch latency they hide (same-box A/B), so it is off.
#ifndef MCO_PDL_TRIGGER
#define MCO_PDL_TRIGGER 0  // measured: hooks 32.15 -> 32.55 ms, multi-tensor +1 %
#endif
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if MCO_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// Explicit early trigger for one kernel (the hook-form K6, whose dependent is the next
// tensor's K1 -- see adalomo.cu).
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

#ifndef MCO_PDL
#define MCO_PDL 1
#endif

template <typename... KArgs, typename... Args>
void launch_pdl_smem(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                     cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = MCO_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...), "cudaLaunchKernelEx");
}
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t st,
                Args... args) {
  launch_pdl_smem(kern, grid, block, 0, st, args...);
}

struct DeviceInfo {
  int sms = 148;
  int l2_bytes = 0;
};
const DeviceInfo& device_info(int device);
int current_device();

// ---- per-step scalars ----------------------------------------------------------
// Derived in double on the host exactly once per step, rounded once to the
// kernel's arithmetic type T (float or double).  Same rule as
// oracle/mco_oracle.c's f32 functions.
template <typename T>
struct StepConsts {
  T b1, b2, b3, omb1, omb2, omb3;  // beta_k and (1 - beta_k)
  T c1, c2, c3;                    // 1 - beta_k^t
  T rc1, rc2, rc3;                 // 1 / (1 - beta_k^t), rounded once (fp32 Adan)
  T sthr;                          // sqrt_plus_eps threshold (AdamW: c2, Adan: c3; 0 = off)
  T lr, eps, wd, lrwd, den, rho;   // den = 1 + lr*wd (Adan), lrwd = lr*wd (Sophia)
  T rden;                          // 1 / (1 + lr*wd), rounded once (fp32 Adan)
  int first;                       // Adan: t == 1
  int refresh;                     // Sophia: (t-1) % k == 0
};

// ---- graph mode (mco_flat_graph_enable) --------------------------------------------
// The step counter lives on the device and DEV kernels derive the step scalars from it,
// so a step captured into a CUDA graph replays as the next step.  rows[t] holds the
// t-dependent scalars (1 - beta_k^t, the sqrt_plus_eps threshold) computed on the host
// exactly as make_consts does; past the last row they are constant (every 1 - beta_k^t
// has rounded to 1.0).  Thread 0 of each CTA is the CTA's only reader of t; the launch
// with bump = 1 (the step's last) advances t in its last CTA to finish (graph_bump).
struct FlatGraphDev {
  int64_t t;      // steps taken
  unsigned done;  // CTAs of the bumping launch that have finished
};
template <typename T>
struct GraphRow {
  T c1, c2, c3, sthr, rc1, rc2, rc3;
};
struct GraphStep {
  FlatGraphDev* d = nullptr;  // null: eager (the by-value scalars)
  const void* rows = nullptr;  // GraphRow<state type>[nrows]
  int64_t nrows = 0;
  const double* lr = nullptr;  // device lr (null: lr_host)
  double lr_host = 0, wd = 0;
  int64_t interval = 1;        // Sophia's update_interval
  int bump = 0;
};

template <bool DEV, typename T>
__device__ __forceinline__ StepConsts<T> step_consts(const StepConsts<T>& kv,
                                                     const GraphStep& gs) {
  if constexpr (!DEV) {
    return kv;
  } else {
    __shared__ int64_t t_sh;
    if (threadIdx.x == 0) t_sh = gs.d->t;
    __syncthreads();
    const int64_t t = t_sh + 1;
    const auto& r = static_cast<const GraphRow<T>*>(gs.rows)[t < gs.nrows ? t : gs.nrows - 1];
    const double lr = gs.lr ? *gs.lr : gs.lr_host;
    const double lw = lr * gs.wd;  // make_consts, same double arithmetic (--fmad=false)
    StepConsts<T> k = kv;
    k.c1 = r.c1, k.c2 = r.c2, k.c3 = r.c3, k.sthr = r.sthr;
    k.rc1 = r.rc1, k.rc2 = r.rc2, k.rc3 = r.rc3;
    k.lr = (T)lr;
    k.lrwd = (T)lw;
    k.den = (T)(1.0 + lw);
    k.rden = (T)(1.0 / (1.0 + lw));
    k.first = t == 1 ? 1 : 0;
    k.refresh = (gs.interval >= 1 && ((t - 1) % gs.interval) == 0) ? 1 : 0;
    return k;
  }
}

// List forms: largest i in [0, n) with b[i] <= v (prefix sums; skips empty ranges).
__device__ __forceinline__ int list_find(const uint64_t* b, int n, uint64_t v) {
  int lo = 0, hi = n - 1;  // largest i with b[i] <= v (skips empty ranges)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (b[mid] <= v) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// End of a DEV kernel, thread 0 (after its CTA's read of t): the last CTA of the
// bumping launch advances t; every CTA has read it by then.
template <bool DEV>
__device__ __forceinline__ void graph_bump(const GraphStep& gs) {
  if constexpr (DEV) {
    if (gs.bump && threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&gs.d->done, 1u) == gridDim.x - 1) {
        gs.d->done = 0;
        gs.d->t += 1;
        __threadfence();
      }
    }
  }
}

// ---- 256-bit global memory access (LDG.E.256 / STG.E.256 on sm_100a) ----------
// Streaming data larger than L2 is read once: no L1 allocation, evict-first in L2.
__device__ __forceinline__ void ld_stream(const float* p, float (&r)[8]) {
  asm volatile(
      "ld.global.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]),
        "=f"(r[7])
      : "l"(p));
}
// Read-only inputs (gradients) use the non-coherent path as well.
__device__ __forceinline__ void ld_stream_ro(const float* p, float (&r)[8]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]),
        "=f"(r[7])
      : "l"(p));
}
__device__ __forceinline__ void st_stream(float* p, const float (&r)[8]) {
  asm volatile(
      "st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r[0]),
      "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
      : "memory");
}
// 128-bit variants (L2 eviction hints need 256-bit accesses on sm_100a)
__device__ __forceinline__ void ld_stream(const float* p, float (&r)[4]) {
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3])
               : "l"(p));
}
__device__ __forceinline__ void ld_stream_ro(const float* p, float (&r)[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3])
               : "l"(p));
}
__device__ __forceinline__ void st_stream(float* p, const float (&r)[4]) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(r[0]),
               "f"(r[1]), "f"(r[2]), "f"(r[3])
               : "memory");
}
// Keep-in-L2 variants (AdaLomo re-reads gradients across passes).
__device__ __forceinline__ void ld_keep_ro(const float* p, float (&r)[8]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]),
        "=f"(r[7])
      : "l"(p));
}
__device__ __forceinline__ void ld_stream(const double* p, double (&r)[4]) {
  asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
               : "l"(p));
}
__device__ __forceinline__ void ld_stream_ro(const double* p, double (&r)[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
               : "l"(p));
}
__device__ __forceinline__ void st_stream(double* p, const double (&r)[4]) {
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r[0]),
               "d"(r[1]), "d"(r[2]), "d"(r[3])
               : "memory");
}
// 8 x bf16 = 128 bits
__device__ __forceinline__ void ld_stream_ro_bf16x8(const uint16_t* p, float (&r)[8]) {
  uint32_t a, b, c, d;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "l"(p));
  const uint32_t w[4] = {a, b, c, d};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    r[2 * k] = __uint_as_float(w[k] << 16);
    r[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
  }
}
__device__ __forceinline__ void ld_stream_bf16x8(const uint16_t* p, float (&r)[8]) {
  uint32_t a, b, c, d;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "l"(p));
  const uint32_t w[4] = {a, b, c, d};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    r[2 * k] = __uint_as_float(w[k] << 16);
    r[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
  }
}

// 16 x bf16 = 256 bits (LDG.E.256)
__device__ __forceinline__ void unpack_bf16x16(const uint32_t (&w)[8], float (&r)[16]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    r[2 * k] = __uint_as_float(w[k] << 16);
    r[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
  }
}
__device__ __forceinline__ void ld_stream_bf16x16(const uint16_t* p, float (&r)[16]) {
  uint32_t w[8];
  asm volatile(
      "ld.global.L1::no_allocate.L2::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7])
      : "l"(p));
  unpack_bf16x16(w, r);
}
__device__ __forceinline__ void ld_stream_ro_bf16x16(const uint16_t* p, float (&r)[16]) {
  uint32_t w[8];
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7])
      : "l"(p));
  unpack_bf16x16(w, r);
}

// fp32 -> bf16 round-to-nearest-even, NaN -> canonical 0x7fff: the hardware
// cvt.rn.bf16x2.f32 (F2FP.BF16.F32.PACK_AB); same rule as the oracle.
__device__ __forceinline__ uint32_t f2bf_bits(float f) {
  uint32_t r;
  asm("{ .reg .b16 lo; cvt.rn.bf16.f32 lo, %1; mov.b32 %0, {lo, lo}; }" : "=r"(r) : "f"(f));
  return r & 0xffffu;
}
// two floats -> packed bf16x2 (a in the low half), one instruction
__device__ __forceinline__ uint32_t f2bf2_bits(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ void st_stream_bf16x8(uint16_t* p, const float (&r)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) w[k] = f2bf2_bits(r[2 * k], r[2 * k + 1]);
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(w[0]),
               "r"(w[1]), "r"(w[2]), "r"(w[3])
               : "memory");
}
__device__ __forceinline__ void st_stream_bf16x16(uint16_t* p, const float (&r)[16]) {
  uint32_t w[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) w[k] = f2bf2_bits(r[2 * k], r[2 * k + 1]);
  asm volatile("st.global.L1::no_allocate.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
               "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]),
               "r"(w[7])
               : "memory");
}
__device__ __forceinline__ float bf2f(uint16_t h) { return __uint_as_float((uint32_t)h << 16); }

// ---- packed fp32 pairs (sm_100: FMUL2 / FFMA2, two IEEE fp32 operations per issue) ----
// Each lane of a pair is rounded exactly as the scalar instruction would round it.  Only
// mul and fma are used: ptxas contracts a packed mul feeding a packed add into FFMA2
// even under --fmad=false, so a packed add never follows a packed mul here.
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// ---- deterministic reductions --------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sums of N values (N = 1, 2, 4, 8) over the 32 lanes at once: the first log2 N
// butterfly steps halve the values each lane carries (it keeps one half, its partner the
// other), the remaining steps are a plain butterfly.  5 shuffles + (N-1) more instead of
// 5 N.  Lane L ends with the sum for value index warp_rows_index<N>(L).  Fixed order:
// deterministic.
template <int N>
__device__ __forceinline__ int warp_rows_index(int lane) {
  int r = 0;
#pragma unroll
  for (int step = 0; (1 << step) < N; ++step) r = (r << 1) | ((lane >> (4 - step)) & 1);
  return r;
}
template <int N>
__device__ __forceinline__ float warp_sum_rows(const float (&v)[N]) {
  const int lane = threadIdx.x & 31;
  float w[N];
#pragma unroll
  for (int i = 0; i < N; ++i) w[i] = v[i];
  int o = 16;
#pragma unroll
  for (int n = N; n > 1; n >>= 1, o >>= 1) {
    const bool up = lane & o;
    const int half = n >> 1;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = up ? w[i] : w[i + half];
      const float keep = up ? w[i + half] : w[i];
      w[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (; o > 0; o >>= 1) w[0] += __shfl_xor_sync(0xffffffffu, w[0], o);
  return w[0];
}

// Block sum in a fixed order (warp butterflies, then warp partials in warp
// order by warp 0).  Result valid in thread 0.  `scratch` >= 32 entries.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();  // scratch reuse guard
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  T r = 0;
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    r = lane < nw ? scratch[lane] : T(0);
    r = warp_sum(r);
  }
  return r;
}

}  // namespace mco
