// Sophia with an fp64 first moment (state dtype MCO_F32M64, opt-in "precise-m" mode).
//
// Why: Sophia's update is u = clamp(m / max(rho h, eps), -1, 1) (optim.cpp:160-166).
// m is an EMA of gradients that change sign, so it cancels: its fp32 rounding error is
// ~2^-24 |g| while m itself can be far smaller, and the division by rho h ~ 0.04 g^2
// amplifies that error by 1/(rho h) in the unclamped band.  With fp32 m, ~0.06 % of
// elements drift past the 1e-5 per-element bar of north_star after 20 steps (DESIGN
// section 4).  Keeping m in fp64 (and doing the per-element arithmetic in fp64, the
// reference's own type) leaves only the fp32 storage of p and h: measured <= 1.4e-6.
//
// Traffic: R p(4) g(4 | 2 bf16) m(8) h(4 on refresh... read always) + W p(4) m(8) [+ h(4)
// on refresh] = 32 B/param (36 on refresh) vs 24 / 28 for the fp32 kernel.
//
// Per element, operation order of optim.cpp:160-166 in fp64 on fp32-stored p, g, h:
//   m = b1 m + (1 - b1) g
//   refresh: h = (float)(b2 h + (1 - b2) g g)        (fp32 storage, rounded once)
//   denom = max(rho h, eps); u = clamp(m / denom, -1, 1)
//   p = (float)(p - (lr u + (lr wd) p))
// -- oracle/mco_oracle.c orc_sophia_m64 restates it (bit-exact test).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace mco {
namespace {

using flatk::grid_for;
using flatk::kThreads;

struct SophiaM64Consts {
  double b1, omb1, b2, omb2, rho, eps, lr, lrwd;
  int refresh;
};

__device__ __forceinline__ float sm64_one(float p, float g, double& m, float& h,
                                          const SophiaM64Consts& k) {
  const double gd = (double)g;
  m = k.b1 * m + k.omb1 * gd;
  if (k.refresh) h = (float)(k.b2 * (double)h + k.omb2 * gd * gd);
  const double rh = k.rho * (double)h;
  const double denom = rh < k.eps ? k.eps : rh;
  const double q = m / denom;
  const double u = q < -1.0 ? -1.0 : (1.0 < q ? 1.0 : q);
  const double pd = (double)p;
  return (float)(pd - (k.lr * u + k.lrwd * pd));
}

__device__ __forceinline__ float load_g(const float* g, uint64_t i) { return g[i]; }
__device__ __forceinline__ float load_g(const uint16_t* g, uint64_t i) {
  return __uint_as_float((uint32_t)g[i] << 16);
}

// Vector path: 4 elements per item (p, g, h: 16 B; m: 32 B), persistent grid-stride;
// elements [0, head) and [head + 4 nvec, n) take the scalar path.
template <typename GT>
__global__ void __launch_bounds__(256) sophia_m64_kernel(float* __restrict__ p,
                                                        const GT* __restrict__ g,
                                                        double* __restrict__ m,
                                                        float* __restrict__ h, uint64_t head,
                                                        uint64_t nvec, uint64_t n,
                                                        SophiaM64Consts k) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = tid; v < nvec; v += stride) {
    const uint64_t e = head + 4 * v;
    float pr[4], gr[4], hr[4];
    double mr[4];
    ld_stream(p + e, pr);
    if constexpr (sizeof(GT) == 4) {
      ld_stream_ro((const float*)g + e, gr);
    } else {
      const uint2 w = *reinterpret_cast<const uint2*>((const uint16_t*)g + e);
      gr[0] = __uint_as_float(w.x << 16);
      gr[1] = __uint_as_float(w.x & 0xffff0000u);
      gr[2] = __uint_as_float(w.y << 16);
      gr[3] = __uint_as_float(w.y & 0xffff0000u);
    }
    ld_stream(m + e, mr);
    ld_stream(h + e, hr);
#pragma unroll
    for (int j = 0; j < 4; ++j) pr[j] = sm64_one(pr[j], gr[j], mr[j], hr[j], k);
    st_stream(p + e, pr);
    st_stream(m + e, mr);
    if (k.refresh) st_stream(h + e, hr);
  }
  const uint64_t body_end = head + 4 * nvec;
  for (uint64_t i = tid; i < head + (n - body_end); i += stride) {
    const uint64_t e = i < head ? i : body_end + (i - head);
    double mm = m[e];
    float hh = h[e];
    p[e] = sm64_one(p[e], load_g(g, e), mm, hh, k);
    m[e] = mm;
    if (k.refresh) h[e] = hh;
  }
}

}  // namespace

void launch_sophia_m64(float* p, const void* g, int g_dtype, double* m, float* h, uint64_t n,
                       const StepConsts<double>& kd, cudaStream_t st) {
  if (n == 0) return;
  SophiaM64Consts k{kd.b1, kd.omb1, kd.b2, kd.omb2, kd.rho, kd.eps, kd.lr, kd.lrwd, kd.refresh};
  // head: elements until p is 16 B aligned; the vector path needs every stream aligned
  // at that element (same element phase), else everything is scalar
  const uint64_t ph = ((uintptr_t)p / 4) % 4;
  uint64_t head = ph ? 4 - ph : 0;
  if (head > n) head = n;
  const size_t gs = g_dtype == MCO_BF16 ? 2 : 4;
  const bool vec = ((uintptr_t)(p + head) % 16 == 0) && ((uintptr_t)(h + head) % 16 == 0) &&
                   ((uintptr_t)(m + head) % 32 == 0) &&
                   (((uintptr_t)g + head * gs) % (4 * gs) == 0);
  const uint64_t nvec = vec ? (n - head) / 4 : 0;
  if (!vec) head = n;  // all scalar
  const int dev = current_device();
  if (g_dtype == MCO_BF16) {
    auto kern = sophia_m64_kernel<uint16_t>;
    const int grid = grid_for(kern, std::max<uint64_t>(nvec ? nvec : n, 1), dev);
    kern<<<grid, kThreads, 0, st>>>(p, (const uint16_t*)g, m, h, head, nvec, n, k);
  } else {
    auto kern = sophia_m64_kernel<float>;
    const int grid = grid_for(kern, std::max<uint64_t>(nvec ? nvec : n, 1), dev);
    kern<<<grid, kThreads, 0, st>>>(p, (const float*)g, m, h, head, nvec, n, k);
  }
  launch_check("sophia_m64_kernel");
}

}  // namespace mco
