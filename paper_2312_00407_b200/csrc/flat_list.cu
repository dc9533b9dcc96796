// FlatOptimizer list form (mco_flat_step_list): separate parameter / gradient tensors
// over the handle's flat state, one launch per kListMax tensors (kernels.h).  Same
// arithmetic as the flat kernels (update.cuh, --fmad=false): bit-identical to a flat
// step over the concatenation.
#include <algorithm>
#include <cstring>
#include <type_traits>

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

// ---- list form (mco_flat_step_list) --------------------------------------------------
// Separate parameter / gradient tensors over the handle's flat state: tensor i's state
// is elements [soff_i, soff_i + n_i) -- the layout of the flattened vector, so the state
// equals a flat step over the concatenation bit for bit.  The launch's vectors (of the
// tensors whose streams are all W-aligned) and scalar elements (tails, unaligned
// tensors) are two virtual index spaces; a thread finds its tensor by binary search over
// the prefix sums (shared memory).

template <int KIND, typename T, typename GT, int U, int MINB, bool DEV>
__global__ void __launch_bounds__(kThreads, MINB)
    flat_list_kernel(const __grid_constant__ FlatList L, T* __restrict__ s0,
                     T* __restrict__ s1, T* __restrict__ s2, T* __restrict__ s3,
                     const StepConsts<T> kv, const GraphStep gs) {
  const StepConsts<T> k = step_consts<DEV>(kv, gs);
  constexpr int W = Vec<T>::W;
  __shared__ uint64_t vb[kListMax + 1], eb[kListMax + 1];
  for (int i = threadIdx.x; i <= L.n; i += blockDim.x) vb[i] = L.vbeg[i], eb[i] = L.ebeg[i];
  __syncthreads();
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t nv = vb[L.n];
  int cur = 0;  // the thread's vectors only increase: step the owning tensor forward
  for (uint64_t base = tid; base < nv; base += stride * U) {
    T pv[U][W], gv[U][W], a[U][W], b[U][W], c[U][W], d[U][W];
    T* pp[U];
    uint64_t so[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = base + (uint64_t)u * stride;
      if (vi < nv) {
        while (cur + 1 < L.n && vb[cur + 1] <= vi) ++cur;
        const int i = cur;
        const uint64_t e = (vi - vb[i]) * W;
        pp[u] = static_cast<T*>(L.p[i]) + e;
        so[u] = L.soff[i] + e;
        ld_stream(pp[u], pv[u]);
        load_grad(static_cast<const GT*>(L.g[i]) + e, gv[u]);
        ld_stream(s0 + so[u], a[u]);
        if constexpr (reads_s1(KIND)) ld_stream(s1 + so[u], b[u]);
        if constexpr (KIND == K_ADAN) {
          ld_stream(s2 + so[u], c[u]);
          if (!k.first) ld_stream(s3 + so[u], d[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = base + (uint64_t)u * stride;
      if (vi < nv) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
          if constexpr (KIND != K_ADAN) c[u][j] = d[u][j] = T(0);
          if constexpr (KIND == K_ADAN) {
            if (k.first) d[u][j] = T(0);
          }
          if constexpr (!reads_s1(KIND)) b[u][j] = T(0);
          update<KIND, T>(pv[u][j], gv[u][j], a[u][j], b[u][j], c[u][j], d[u][j], k);
        }
        st_stream(pp[u], pv[u]);
        st_stream(s0 + so[u], a[u]);
        if constexpr (KIND == K_ADAMW || KIND == K_ADAN) st_stream(s1 + so[u], b[u]);
        if constexpr (KIND == K_SOPHIA) {
          if (k.refresh) st_stream(s1 + so[u], b[u]);
        }
        if constexpr (KIND == K_ADAN) {
          st_stream(s2 + so[u], c[u]);
          st_stream(s3 + so[u], d[u]);
        }
      }
    }
  }
  const uint64_t ne = eb[L.n];
  for (uint64_t x = tid; x < ne; x += stride) {
    const int i = list_find(eb, L.n, x);
    const uint64_t e = L.first_scalar[i] + (x - eb[i]), o = L.soff[i] + e;
    T* p = static_cast<T*>(L.p[i]);
    T pp = p[e], gg = (T)load_grad1(static_cast<const GT*>(L.g[i]) + e), aa = s0[o],
      bb = T(0), cc = T(0), dd = T(0);
    if constexpr (reads_s1(KIND)) bb = s1[o];
    if constexpr (KIND == K_ADAN) {
      cc = s2[o];
      if (!k.first) dd = s3[o];
    }
    update<KIND, T>(pp, gg, aa, bb, cc, dd, k);
    p[e] = pp;
    s0[o] = aa;
    if constexpr (KIND == K_ADAMW || KIND == K_ADAN) s1[o] = bb;
    if constexpr (KIND == K_SOPHIA) {
      if (k.refresh) s1[o] = bb;
    }
    if constexpr (KIND == K_ADAN) {
      s2[o] = cc;
      s3[o] = dd;
    }
  }
  graph_bump<DEV>(gs);
}

template <int KIND, typename T, typename GT>
void run_list(const FlatList& L, const FlatListArgs& a, const StepConsts<T>& k,
              const GraphStep& gs, cudaStream_t st) {
  constexpr int U = (KIND == K_ADAN) ? 1 : 2;
#ifndef MCO_LIST_MINB
#define MCO_LIST_MINB 1
#endif
  constexpr int MINB =
      (sizeof(T) == 4 && (KIND == K_ADAN || KIND == K_LION)) ? 3 : MCO_LIST_MINB;
  auto kern = gs.d ? flat_list_kernel<KIND, T, GT, U, MINB, true>
                   : flat_list_kernel<KIND, T, GT, U, MINB, false>;
  const uint64_t nv = L.vbeg[L.n], ne = L.ebeg[L.n];
  const uint64_t items = std::max<uint64_t>(std::max((nv + U - 1) / U, ne), 1);
  const int grid = grid_for(kern, items, current_device());
  kern<<<grid, kThreads, 0, st>>>(L, (T*)a.s[0], (T*)a.s[1], (T*)a.s[2], (T*)a.s[3], k, gs);
  launch_check("flat_list_kernel");
}

// tma: fp32 state and parameters on the cp.async.bulk pipeline (flat_tma.cu), the
// default variant -- tiles of list_tma_tile() elements per 16 B-aligned tensor; else
// the LDG kernel above (W-element vectors per W-aligned tensor).
template <int KIND, typename T, typename GT>
void list_chunks(const FlatListArgs& a, const StepConsts<T>& k, cudaStream_t st) {
  constexpr int W = Vec<T>::W;
  bool tma = false;
  if constexpr (std::is_same_v<T, float>) tma = std::strcmp(flat_variant_name(), "tma") == 0;
  const uint64_t unit = tma ? (uint64_t)list_tma_tile() : (uint64_t)W;  // elements per item
  const size_t align = tma ? 16 : sizeof(T) * W;
  uint64_t soff = 0;
  int last = -1;
  for (int i = 0; i < a.count; ++i)
    if (a.len[i]) last = i;
  if (last < 0) {  // nothing to update: the step still counts
    if (a.gs.d) launch_flat_graph_bump(a.gs.d, st);
    return;
  }
  FlatList L{};
  auto flush = [&](bool final_chunk) {
    if (L.n == 0) return;
    GraphStep gs = a.gs;
    gs.bump = final_chunk ? 1 : 0;  // graph mode: the step's last launch advances t
    if constexpr (std::is_same_v<T, float>) {
      if (tma) {
        float* sl[4] = {(float*)a.s[0], (float*)a.s[1], (float*)a.s[2], (float*)a.s[3]};
        launch_list_tma(a.kind, a.g_dtype, L, sl, k, gs, st);
        L = FlatList{};
        return;
      }
    }
    run_list<KIND, T, GT>(L, a, k, gs, st);
    L = FlatList{};
  };
  for (int i = 0; i < a.count; ++i) {
    const uint64_t n = a.len[i];
    if (n) {
      uint64_t items = 0;
      const int t = L.n++;
      if (tma) {
        // every stream element-aligned; each may sit at its own phase within 16 B
        // (list_tma_kernel reads / writes it shifted): the state slots must share one
        const size_t gsz = sizeof(GT);
        const auto ph = [](const void* q, size_t es) { return (int)(((uintptr_t)q % 16) / es); };
        bool ok = aligned(a.p[i], sizeof(T)) && aligned(a.g[i], gsz);
        int ss = -1;
        for (int j = 0; j < 4; ++j) {
          if (!a.s[j]) continue;
          const void* q = (const char*)a.s[j] + soff * sizeof(T);
          ok = ok && aligned(q, sizeof(T)) && (ss < 0 || ph(q, sizeof(T)) == ss);
          ss = ph(q, sizeof(T));
        }
        L.shp[t] = (uint8_t)ph(a.p[i], sizeof(T));
        L.shg[t] = (uint8_t)ph(a.g[i], gsz);
        L.shs[t] = (uint8_t)std::max(ss, 0);
        const bool shifted = L.shp[t] || L.shg[t] || L.shs[t];
        // a shifted stream's copies reach up to 16 B past the tile: keep them inside the
        // tensor (the last tile joins the scalar elements otherwise)
        if (ok) items = shifted ? (n >= 8 ? (n - 8) / unit : 0) : n / unit;
      } else {
        bool vec = aligned(a.p[i], align) && aligned(a.g[i], sizeof(GT) * W);
        for (int j = 0; j < 4; ++j)
          vec = vec && aligned(a.s[j] ? (const char*)a.s[j] + soff * sizeof(T) : nullptr, align);
        items = vec ? n / unit : 0;
      }
      L.p[t] = a.p[i];
      L.g[t] = a.g[i];
      L.soff[t] = soff;
      L.first_scalar[t] = items * unit;
      L.vbeg[t + 1] = L.vbeg[t] + items;
      L.ebeg[t + 1] = L.ebeg[t] + (n - items * unit);
      if (L.n == kListMax) flush(i == last);
    }
    soff += n;
  }
  flush(true);
}

template <int KIND>
void list_dtypes(const FlatListArgs& a, const StepConsts<float>& kf,
                 const StepConsts<double>& kd, cudaStream_t st) {
  if (a.state_dtype == MCO_F64) {
    if (a.p_dtype != MCO_F64 || a.g_dtype != MCO_F64)
      throw Error(MCO_CONTRACT, "flat step list: f64 state takes f64 params and grads");
    list_chunks<KIND, double, double>(a, kd, st);
  } else if (a.p_dtype != MCO_F32) {
    throw Error(MCO_CONTRACT, "flat step list: f32 state takes f32 params");
  } else if (a.g_dtype == MCO_F32) {
    list_chunks<KIND, float, float>(a, kf, st);
  } else if (a.g_dtype == MCO_BF16) {
    list_chunks<KIND, float, uint16_t>(a, kf, st);
  } else {
    throw Error(MCO_CONTRACT, "flat step list: f32 state takes f32 or bf16 grads");
  }
}

// ---- LOMO list form (mco_lomo_apply_list) -------------------------------------------
// p_i -= f * g_i over separate tensors in one launch per kListMax tensors: lomo_kernel's
// loads, arithmetic and stores per W-element vector (vbeg: vectors), scalar tails.
template <typename PT, typename GT>
__global__ void __launch_bounds__(kThreads)
    lomo_list_kernel(const __grid_constant__ FlatList L, double lr, double scale,
                     const double* __restrict__ sumsq, double clip) {
  using T = typename std::conditional<std::is_same<PT, double>::value, double, float>::type;
  constexpr int W = lomo_width<PT, GT>();
  __shared__ uint64_t vb[kListMax + 1], eb[kListMax + 1];
  pdl_wait();
  for (int i = threadIdx.x; i <= L.n; i += blockDim.x) vb[i] = L.vbeg[i], eb[i] = L.ebeg[i];
  __syncthreads();
  const T f = lomo_factor<T>(lr, scale, sumsq, clip);
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t nv = vb[L.n];
  int cur = 0;  // the thread's vectors only increase: step the owning tensor forward
  for (uint64_t vi = tid; vi < nv; vi += stride) {
    while (cur + 1 < L.n && vb[cur + 1] <= vi) ++cur;
    const int i = cur;
    const uint64_t e = (vi - vb[i]) * W;
    PT* p = static_cast<PT*>(L.p[i]) + e;
    const GT* g = static_cast<const GT*>(L.g[i]) + e;
    T pv[W], gv[W];
    if constexpr (W == 16) {
      ld_stream_bf16x16(p, pv);
      ld_stream_ro_bf16x16(g, gv);
    } else {
      if constexpr (std::is_same<PT, uint16_t>::value)
        ld_stream_bf16x8(p, pv);
      else
        ld_stream(p, pv);
      load_grad(g, gv);
    }
#pragma unroll
    for (int j = 0; j < W; ++j) pv[j] = pv[j] - f * gv[j];
    if constexpr (W == 16)
      st_stream_bf16x16(p, pv);
    else if constexpr (std::is_same<PT, uint16_t>::value)
      st_stream_bf16x8(p, pv);
    else
      st_stream(p, pv);
  }
  const uint64_t ne = eb[L.n];
  for (uint64_t x = tid; x < ne; x += stride) {
    const int i = list_find(eb, L.n, x);
    const uint64_t e = L.first_scalar[i] + (x - eb[i]);
    PT* p = static_cast<PT*>(L.p[i]);
    const GT* g = static_cast<const GT*>(L.g[i]);
    if constexpr (std::is_same<PT, uint16_t>::value)
      p[e] = (uint16_t)f2bf_bits(bf2f(p[e]) - f * load_grad1(g + e));
    else
      p[e] = p[e] - f * (T)load_grad1(g + e);
  }
}

template <typename PT, typename GT>
void lomo_list_chunks(int count, void* const* ps, const void* const* gs, const uint64_t* len,
                      double lr, double scale, const double* sumsq, double clip,
                      cudaStream_t st) {
  constexpr int W = lomo_width<PT, GT>();
  auto kern = lomo_list_kernel<PT, GT>;
  FlatList L{};
  auto flush = [&] {
    if (L.n == 0) return;
    const uint64_t items = std::max<uint64_t>(std::max(L.vbeg[L.n], L.ebeg[L.n]), 1);
    const int grid = grid_for(kern, items, current_device());
    launch_pdl(kern, grid, kThreads, st, L, lr, scale, sumsq, clip);
    launch_check("lomo_list_kernel");
    L = FlatList{};
  };
  for (int i = 0; i < count; ++i) {
    const uint64_t n = len[i];
    if (!n) continue;
    const bool vec = aligned(ps[i], sizeof(PT) * W) && aligned(gs[i], sizeof(GT) * W);
    const uint64_t nvec = vec ? n / W : 0;
    const int t = L.n++;
    L.p[t] = ps[i];
    L.g[t] = gs[i];
    L.soff[t] = 0;
    L.first_scalar[t] = nvec * W;
    L.vbeg[t + 1] = L.vbeg[t] + nvec;
    L.ebeg[t + 1] = L.ebeg[t] + (n - nvec * W);
    if (L.n == kListMax) flush();
  }
  flush();
}

}  // namespace

void launch_flat_step_list(const FlatListArgs& a, const StepConsts<float>& kf,
                           const StepConsts<double>& kd, cudaStream_t st) {
  switch (a.kind) {
    case MCO_ADAMW: list_dtypes<K_ADAMW>(a, kf, kd, st); break;
    case MCO_LION: list_dtypes<K_LION>(a, kf, kd, st); break;
    case MCO_ADAN: list_dtypes<K_ADAN>(a, kf, kd, st); break;
    case MCO_SOPHIA: list_dtypes<K_SOPHIA>(a, kf, kd, st); break;
    default: throw Error(MCO_CONTRACT, "FlatOptimizer: fused kind");
  }
}

void launch_lomo_list(int count, void* const* p, int p_dtype, const void* const* g, int g_dtype,
                      const uint64_t* len, double lr, double scale, const double* dev_sumsq,
                      double clip, cudaStream_t st) {
  if (p_dtype == MCO_F32 && g_dtype == MCO_F32)
    lomo_list_chunks<float, float>(count, p, g, len, lr, scale, dev_sumsq, clip, st);
  else if (p_dtype == MCO_F32 && g_dtype == MCO_BF16)
    lomo_list_chunks<float, uint16_t>(count, p, g, len, lr, scale, dev_sumsq, clip, st);
  else if (p_dtype == MCO_BF16 && g_dtype == MCO_BF16)
    lomo_list_chunks<uint16_t, uint16_t>(count, p, g, len, lr, scale, dev_sumsq, clip, st);
  else if (p_dtype == MCO_F64 && g_dtype == MCO_F64)
    lomo_list_chunks<double, double>(count, p, g, len, lr, scale, dev_sumsq, clip, st);
  else
    throw Error(MCO_CONTRACT, "lomo_apply_list: unsupported param/grad dtype pair");
}

}  // namespace mco
