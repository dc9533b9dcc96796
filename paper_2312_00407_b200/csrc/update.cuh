// The per-element optimizer updates shared by the flat kernels (flat.cu) and the
// peer-memory ZeRO kernel (peer.cu).  Operation order = optim.cpp:114-167.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace mco {
namespace upd {

enum { K_ADAMW = 0, K_LION = 1, K_ADAN = 2, K_SOPHIA = 3 };

__device__ __forceinline__ float dsqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double dsqrt(double x) { return sqrt(x); }

// sqrt(x / c) + eps, bit-identical to the plain expression, without the IEEE slow paths
// of div.rn / sqrt.rn on tiny x (an EMA of squared gradients below ~1e-19 is
// subnormal: AdamW / Adan ran 2x slower).  thr (host, make_consts) = (ulp(eps)/4)^2 * c,
// so x < thr gives RN(sqrt(RN(x / c))) <= ulp(eps)/4 and the sum rounds back to eps;
// a normal stand-in keeps the unselected division and square root on the fast path.
__device__ __forceinline__ float sqrt_plus_eps(float x, float c, float eps, float thr) {
  const bool tiny = x < thr;
  const float r = dsqrt((tiny ? c : x) / c) + eps;
  return tiny ? eps : r;
}
__device__ __forceinline__ double sqrt_plus_eps(double x, double c, double eps, double) {
  return dsqrt(x / c) + eps;
}
// The multiply form (fp32 Adan): sqrt(x * rc) + eps, thr from sqrt_eps_threshold_mul.
__device__ __forceinline__ float sqrt_mul_plus_eps(float x, float rc, float eps, float thr) {
  const bool tiny = x < thr;
  const float r = dsqrt((tiny ? 1.0f : x) * rc) + eps;
  return tiny ? eps : r;
}

// The per-element update, operation for operation as optim.cpp.
template <int KIND, typename T>
__device__ __forceinline__ void update(T& p, const T g, T& a, T& b, T& c, T& d,
                                       const StepConsts<T>& k) {
  if constexpr (KIND == K_ADAMW) {  // optim.cpp:118-124; a = m, b = v
    a = k.b1 * a + k.omb1 * g;
    b = k.b2 * b + k.omb2 * g * g;
    const T mhat = a / k.c1;
    p = p - k.lr * (mhat / sqrt_plus_eps(b, k.c2, k.eps, k.sthr) + k.wd * p);
  } else if constexpr (KIND == K_LION) {  // optim.cpp:129-134; a = m
    const T u = k.b1 * a + k.omb1 * g;
    const T s = u > T(0) ? T(1) : (u < T(0) ? T(-1) : T(0));  // sign(0) = 0
    p = p - k.lr * (s + k.wd * p);
    a = k.b2 * a + k.omb2 * g;
  } else if constexpr (KIND == K_ADAN) {  // optim.cpp:142-154; a,b,c,d = m,v,n,g_prev
    const T gd = k.first ? T(0) : g - d;
    a = k.b1 * a + k.omb1 * g;
    b = k.b2 * b + k.omb2 * gd;
    const T nu = g + k.b2 * gd;
    c = k.b3 * c + k.omb3 * nu * nu;
    if constexpr (sizeof(T) == 4) {
      // fp32: the bias corrections and the decoupled decay as multiplications by
      // reciprocals rounded once on the host (1 IEEE division instead of 5 per element;
      // the division chains made this 11-stream kernel issue-bound at low SM clocks).
      // Within 1e-5 of the fp64 reference like the rest (tests/parity.py); the f64
      // mode keeps the reference's divisions and stays bit-exact to it.
      const T mhat = a * k.rc1;
      const T vhat = b * k.rc2;
      p = (p - k.lr * (mhat + k.b2 * vhat) / sqrt_mul_plus_eps(c, k.rc3, k.eps, k.sthr)) *
          k.rden;
    } else {
      const T mhat = a / k.c1;
      const T vhat = b / k.c2;
      p = (p - k.lr * (mhat + k.b2 * vhat) / sqrt_plus_eps(c, k.c3, k.eps, k.sthr)) / k.den;
    }
    d = g;
  } else {  // K_SOPHIA, optim.cpp:160-166; a = m, b = h
    a = k.b1 * a + k.omb1 * g;
    if (k.refresh) b = k.b2 * b + k.omb2 * g * g;  // squared-gradient proxy
    const T rh = k.rho * b;
    const T denom = rh < k.eps ? k.eps : rh;  // std::max(rho*h, eps)
    const T q = a / denom;
    const T u = q < T(-1) ? T(-1) : (T(1) < q ? T(1) : q);  // std::clamp
    p = p - (k.lr * u + k.lrwd * p);
  }
}

// LOMO step factor f = lr * scale (optim.cpp:188); with a device sum of squares the
// scale is the global-norm clip rule (optim.cpp:291-303).
template <typename T>
__device__ __forceinline__ T lomo_factor(double lr, double scale, const double* sumsq,
                                         double clip) {
  if (sumsq) {  // optim.cpp:302-303
    const double norm = sqrt(*sumsq);
    scale = (norm > clip && norm > 0) ? clip / norm : 1.0;
  }
  return (T)(lr * scale);  // optim.cpp:188  f = lr * scale
}

// ---- vector load helpers by element type -----------------------------------
template <typename T>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int W = 8;
};
template <>
struct Vec<double> {
  static constexpr int W = 4;
};

__device__ __forceinline__ void load_grad(const float* g, float (&r)[8]) { ld_stream_ro(g, r); }
__device__ __forceinline__ void load_grad(const uint16_t* g, float (&r)[8]) {
  ld_stream_ro_bf16x8(g, r);
}
__device__ __forceinline__ void load_grad(const double* g, double (&r)[4]) { ld_stream_ro(g, r); }
__device__ __forceinline__ void load_grad(const float* g, float (&r)[4]) { ld_stream_ro(g, r); }
__device__ __forceinline__ void load_grad(const uint16_t* g, float (&r)[4]) {
  const uint2 w = *reinterpret_cast<const uint2*>(g);
  r[0] = __uint_as_float(w.x << 16);
  r[1] = __uint_as_float(w.x & 0xffff0000u);
  r[2] = __uint_as_float(w.y << 16);
  r[3] = __uint_as_float(w.y & 0xffff0000u);
}
__device__ __forceinline__ float load_grad1(const float* g) { return *g; }
__device__ __forceinline__ float load_grad1(const uint16_t* g) { return bf2f(*g); }
__device__ __forceinline__ double load_grad1(const double* g) { return *g; }

// LOMO elements per 256-bit access: f64 4, bf16 params + bf16 grads 16, else 8.
template <typename PT, typename GT>
constexpr int lomo_width() {
  if constexpr (std::is_same<PT, double>::value) return 4;
  if constexpr (std::is_same<PT, uint16_t>::value && std::is_same<GT, uint16_t>::value) return 16;
  return 8;
}

constexpr bool reads_s1(int k) { return k == K_ADAMW || k == K_ADAN || k == K_SOPHIA; }

}  // namespace upd
}  // namespace mco
