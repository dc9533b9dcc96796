// AdaLomo for sm_100a (optim.cpp:192-282): factored row/column second moment,
// RMS(theta)-scaled lr, update-RMS damping, optional global grad-norm clip.
//
// The reference's six sequential passes per tensor (optim.cpp:223-274, with a
// stride-C column loop and a full-size temporary u) become three streaming
// passes over HBM plus three small finalisation kernels.  The dependency chain
// forces them: column statistics need every row before any u exists, and the
// damping needs sum(u^2) over the whole tensor before any parameter moves.
//
//   K1 stats   (tiles)   : per row sum g^2 (row partials), per column partial
//                          sums over the tile's rows, sum p^2, sum v_row_old
//   KR         (columns) : tile partials -> statistics payload (column sums, per tensor
//                          sum g^2 / p^2 / v_row_old)
//   K2 scalars (1 CTA)   : per tensor sum g^2, sum p^2 -> global clip scale s,
//                          t += 1, corr, rms_theta, lr_t, row_mean (linearity)
//   K3 moments (items)   : v_row / v_col EMAs (fp64 state) and the fp32
//                          factors a_i = v_row_i/corr, b_j = (v_col_j/corr)/row_mean
//   K4 sum u^2 (tiles)   : u = s*g / sqrt(a_i*b_j + eps); 1-D tensors update v_full
//   K5 damping (1 CTA)   : f = lr_t / max(1, rms_u / adalomo_clip)
//   K6 update  (tiles)   : p -= f * u  (u recomputed bit-identically to K4)
// Unsharded calls run K2 inside KR's scalar block and K5 in K4's last CTA (5 launches);
// the row-split sharded phases all-reduce the payloads between KR and K2 and between
// K4 and K5, so they launch all seven.
//
// Work unit = tile: rows [r0,r1) x columns [c0,c1) of one matrix (or an
// element range of a 1-D tensor), one CTA per tile, persistent grid over the
// tile table.  Threads: TR row groups x TC column lanes, one 8-wide (32 B)
// column chunk per lane, so every warp reads a contiguous 1 KB row segment.
// All reductions are fixed-order (no float atomics): results are
// bit-reproducible run to run.
#include <algorithm>
#include <atomic>
#include <cfloat>
#include <mutex>
#include <unordered_map>
#include <cmath>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include <cooperative_groups.h>

#include "adalomo.h"
#include "tma.cuh"

namespace mco {
namespace {

// Programmatic Dependent Launch (common.cuh): every AdaLomo kernel starts with
// pdl_wait() and is launched with launch_pdl.  The per-tensor hook form runs 8
// dependent launches per tensor, where the launch gaps dominate.


constexpr int kThreads = 256;
constexpr int kRB = 2;   // K1 / K6 tiles: rows per thread per loop iteration (loads in flight)
// bf16 parameters and gradients move half the bytes per row: twice the rows in flight
// (ncu, bf16 at kRB: K1 / K6 stalled on long_scoreboard at ~30 % issue, 0.5 of copy BW)
template <typename GT, typename PT>
constexpr int rows_in_flight() {
  return (sizeof(GT) == 2 && sizeof(PT) == 2) ? 2 * kRB : kRB;
}
#ifndef MCO_K1_RB_BF16
// K1 on bf16 parameters + gradients: 8 rows in flight per thread at 2 CTAs / SM (126
// registers) -- 7B bf16 13.69 -> 13.41 ms (same box; 8 rows at 3 CTAs: 13.62, 2 rows at
// 4 CTAs: 14.22)
#define MCO_K1_RB_BF16 8
#endif
#ifndef MCO_K1_RB_F32
// K1 on fp32 parameters: 4 rows in flight at 2 CTAs / SM (MCO_K1_MINB, 128 registers)
// instead of 2 at 3 -- same box: 7B multi-tensor 25.05 -> 24.55 ms, list form 25.4 ->
// 24.8, hook form 29.54 -> 29.00, C3 (13B + clip) 47.56 -> 46.77
#define MCO_K1_RB_F32 4
#endif
template <typename GT, typename PT>
constexpr int k1_rows() {
  return (MCO_K1_RB_BF16 && sizeof(GT) == 2 && sizeof(PT) == 2) ? MCO_K1_RB_BF16
         : (MCO_K1_RB_F32 && sizeof(PT) == 4)                    ? MCO_K1_RB_F32
                                                                 : rows_in_flight<GT, PT>();
}
#ifndef MCO_K1_MINB
#define MCO_K1_MINB 2  // with MCO_K1_RB_F32 = 4 (below)
#endif
#ifndef MCO_K4_MINB
#define MCO_K4_MINB 3
#endif
constexpr int kMinCtasK1 = MCO_K1_MINB;  // resident CTAs per SM (register cap)
constexpr int kMinCtasK4 = MCO_K4_MINB;
#ifndef MCO_K6_MINB
#define MCO_K6_MINB 3
#endif
#ifndef MCO_K6_MINB_BF16
// round 1: 4 (64 registers, 56 B spilled) won, 16.93 -> 16.50 ms on 7B bf16; after the
// round-2 K6 (one FMA for p - f u) 3 CTAs with 80 registers and no spills win: 7B bf16
// 13.95-14.06 -> 13.68 ms, same box (K1 / K4 caps re-measured: 3 stays best)
#define MCO_K6_MINB_BF16 3
#endif
#ifndef MCO_K1_MINB_BF16
#define MCO_K1_MINB_BF16 2  // with MCO_K1_RB_BF16 = 8 (above)
#endif
// register caps -> resident CTAs per SM (tuning knobs; bf16 rows move half the bytes,
// so more CTAs keep enough loads in flight)
template <typename GT, typename PT>
constexpr int k6_minb() {
  return sizeof(GT) == 2 ? MCO_K6_MINB_BF16 : MCO_K6_MINB;  // bf16 gradients
}
#ifndef MCO_K4_MINB_BF16
#define MCO_K4_MINB_BF16 MCO_K4_MINB
#endif
template <typename GT>
constexpr int k4_minb() {
  return sizeof(GT) == 2 ? MCO_K4_MINB_BF16 : kMinCtasK4;
}
template <typename GT, typename PT>
constexpr int k1_minb() {
  return (sizeof(GT) == 2 && sizeof(PT) == 2) ? MCO_K1_MINB_BF16 : kMinCtasK1;
}

struct Ctx {
  const Tile* tiles;
  const TensorInfo* tensors;
  double* state;      // fp64 v_row / v_col / v_full
  float* colpart;     // [nrb][C] per factored tensor
  double* rowpart;    // [kc][R]  per factored tensor
  double* tile_sc;    // 4 doubles per tile: psq, gsq, vrs, usq
  double* tens_sc;    // kTensScalars per tensor
  float* fa;          // a_i per factored tensor row
  float* fb;          // b_j per factored tensor column
  double* glob;       // [0] = clip scale s, [1] = global sum g^2
  double* pay;        // stats payload: 3 per tensor (gsq, psq, vrs) | column sums
  double* pay_usq;    // usq payload: 1 per tensor
  int64_t ntens;      // total tensors (payload layout)
  const Chunk* chunks;
  double* chunk_sc;   // per-chunk sum u^2
  float* fra;         // 1 / sqrt(a_i)  (separable form, see sep_ok)
  float* frb;         // 1 / sqrt(b_j)
  unsigned* mins;     // per tensor: min a_i, min b_j (fp32 bits; atomicMin)
};

enum { TS_GSQ = 0, TS_PSQ, TS_VRS, TS_CORR, TS_LRT, TS_ROWMEAN, TS_USQ, TS_F, kTensScalars };

template <typename GT>
__device__ __forceinline__ void load8(const GT* g, float (&r)[8]);
template <>
__device__ __forceinline__ void load8<float>(const float* g, float (&r)[8]) {
  ld_keep_ro(g, r);
}
template <>
__device__ __forceinline__ void load8<uint16_t>(const uint16_t* g, float (&r)[8]) {
  ld_stream_ro_bf16x8(g, r);
}
__device__ __forceinline__ float ld1(const float* g) { return *g; }
__device__ __forceinline__ float ld1(const uint16_t* g) { return bf2f(*g); }

// A lane's column chunk is always kCW = 8 columns; VEC selects one 256-bit
// (f32) / 128-bit (bf16) access or 8 scalar accesses (unaligned rows).
constexpr int VW = kCW;
template <bool VEC, typename GT>
__device__ __forceinline__ void load_vec(const GT* g, float (&r)[VW], int valid) {
  if constexpr (VEC) {
    if (valid == VW) {
      load8<GT>(g, r);
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < VW; ++j) r[j] = j < valid ? ld1(g + j) : 0.f;
}
// Parameters: fp32, or bf16 storage (fp32 arithmetic, RNE store -- the fp32 result
// rounded once, as LOMO's bf16 path).
__device__ __forceinline__ float ldp1(const float* p) { return *p; }
__device__ __forceinline__ float ldp1(const uint16_t* p) { return bf2f(*p); }
__device__ __forceinline__ void stp1(float* p, float v) { *p = v; }
__device__ __forceinline__ void stp1(uint16_t* p, float v) { *p = (uint16_t)f2bf_bits(v); }

template <bool VEC, typename PT>
__device__ __forceinline__ void load_p(const PT* p, float (&r)[VW], int valid) {
  if constexpr (VEC) {
    if (valid == VW) {
      if constexpr (sizeof(PT) == 4)
        ld_stream(p, r);
      else
        ld_stream_bf16x8(p, r);
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < VW; ++j) r[j] = j < valid ? ldp1(p + j) : 0.f;
}
template <bool VEC, typename PT>
__device__ __forceinline__ void store_p(PT* p, const float (&r)[VW], int valid) {
  if constexpr (VEC) {
    if (valid == VW) {
      if constexpr (sizeof(PT) == 4)
        st_stream(p, r);
      else
        st_stream_bf16x8(p, r);
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < VW; ++j)
    if (j < valid) stp1(p + j, r[j]);
}

constexpr int kLaneStride = 32;  // scalar-path tile lanes: column stride (lane_cols)
// a tile lane's 8 columns back (vector or strided scalar layout, lane_cols)
template <bool VEC, typename PT>
__device__ __forceinline__ void store_tile(PT* p, const float (&r)[VW], int valid) {
  if constexpr (VEC) {
    store_p<VEC, PT>(p, r, VW);
  } else {
#pragma unroll
    for (int j = 0; j < VW; ++j)
      if (j < valid) stp1(p + kLaneStride * j, r[j]);
  }
}

// A tile lane's 8 columns of one row.  Vector path: 8 contiguous columns, one 256-bit
// (fp32) / 128-bit (bf16) access.  Scalar path (rows off the 8-element grid: C % 8 != 0,
// or a tensor behind an odd-sized one in a flat buffer): the warp's 256 columns are dealt
// out strided -- lane l of warp w in the row group takes columns 256 w + l + 32 j -- so
// every load / store instruction of the warp covers 32 consecutive elements (coalesced,
// any alignment) instead of 32 lanes each touching its own 32 B (round 1: 8 scalar
// accesses per lane 32 B apart, 0.5 of the copy bandwidth).  `valid` = how many of the
// lane's 8 columns lie in the tile (always a prefix in either layout).
template <bool VEC>
__device__ __forceinline__ void lane_cols(const Tile& tl, int lane_c, int64_t& col, int& cs,
                                          int& valid) {
  if constexpr (VEC) {
    col = tl.c0 + (int64_t)lane_c * VW;
    cs = 1;
    valid = (int)std::min<int64_t>(VW, std::max<int64_t>(0, tl.c1 - col));
  } else {
    col = tl.c0 + (int64_t)(lane_c >> 5) * (32 * VW) + (lane_c & 31);
    cs = kLaneStride;
    valid = (int)std::min<int64_t>(VW, std::max<int64_t>(0, (tl.c1 - col + kLaneStride - 1) /
                                                                kLaneStride));
  }
}
// column offset within the tile -> (lane, element) of the layout above
template <bool VEC>
__device__ __forceinline__ void col_lane(int q, int& lane_c, int& j) {
  if constexpr (VEC) {
    lane_c = q / VW;
    j = q % VW;
  } else {
    lane_c = (q / (32 * VW)) * 32 + (q % 32);
    j = (q % (32 * VW)) / 32;
  }
}

// Held in load form until consumed: fp32 as 8 floats, bf16 as the 4 raw 32-bit words
// (half the registers), so the bf16 tile kernels can keep twice the rows in flight
// (rows_in_flight) without spilling.  On the vector path (C % 8 == 0, so a lane's chunk
// is either whole or outside the tile) a load is always a whole 8-element vector:
// callers load only lanes with valid > 0.
template <bool VEC, typename T, bool RO>
struct RowVec {
  float v[VW];
  __device__ __forceinline__ void load(const T* src, int valid) {
    if constexpr (VEC) {
      if constexpr (RO)
        load_vec<VEC, T>(src, v, VW);
      else
        load_p<VEC, T>(src, v, VW);
    } else {
#pragma unroll
      for (int j = 0; j < VW; ++j)
        v[j] = j < valid ? (RO ? ld1(src + kLaneStride * j) : ldp1(src + kLaneStride * j)) : 0.f;
    }
  }
  __device__ __forceinline__ void get(float (&r)[VW]) const {
#pragma unroll
    for (int j = 0; j < VW; ++j) r[j] = v[j];
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int j = 0; j < VW; ++j) v[j] = 0.f;
  }
};
template <bool VEC, bool RO>
struct RowVec<VEC, uint16_t, RO> {
  uint32_t w[4];
  __device__ __forceinline__ void load(const uint16_t* src, int valid) {
    if constexpr (VEC) {
      if constexpr (RO)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                     : "l"(src));
      else
        asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                     : "l"(src));
      return;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // strided scalar layout (lane_cols)
      const uint32_t lo = 2 * k < valid ? src[kLaneStride * (2 * k)] : 0u;
      const uint32_t hi = 2 * k + 1 < valid ? src[kLaneStride * (2 * k + 1)] : 0u;
      w[k] = lo | (hi << 16);
    }
  }
  __device__ __forceinline__ void get(float (&r)[VW]) const {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      r[2 * k] = __uint_as_float(w[k] << 16);
      r[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
    }
  }
  __device__ __forceinline__ void zero() { w[0] = w[1] = w[2] = w[3] = 0u; }
};

struct Ptrs {
  void* p;
  const void* g;
  int single;  // 1: p / g point at the call's only tensor
  int ntab;    // > 0: tensor t0 + i at ptab[i] / gtab[i] (list form)
  int t0;
  // calls mixing tensors that take the vector path with tensors that cannot (odd column
  // counts, rows off the 8-element grid): 1 = this launch takes only the vector-path
  // tensors, 2 = only the others, 0 = every tensor (the call is uniform)
  int filt;
  int psz, gsz;  // element bytes of the parameters / gradients
  void* ptab[kMaxTab];
  const void* gtab[kMaxTab];
};
template <typename GT>
__device__ __forceinline__ const GT* gptr(const Ptrs& P, const TensorInfo& T, int k) {
  if (P.ntab) return (const GT*)P.gtab[k - P.t0];
  return (const GT*)P.g + (P.single ? 0 : T.elem_off);
}
template <typename PT>
__device__ __forceinline__ PT* pptr(const Ptrs& P, const TensorInfo& T, int k) {
  if (P.ntab) return (PT*)P.ptab[k - P.t0];
  return (PT*)P.p + (P.single ? 0 : T.elem_off);
}

// Vector-path eligibility of tensor k, as the host decides it (launch_adalomo_phase):
// 1-D tensors run element loops on either path; a matrix needs C % 8 == 0 and its
// parameter and gradient rows at 8-element-aligned addresses.  A mixed call launches
// every tiled pass twice (VEC instance with filt 1, scalar instance with filt 2) and each
// tile is taken by exactly one of them -- same tiles, same arithmetic, same order.
__device__ __forceinline__ bool skip_tensor(const Ptrs& P, const TensorInfo& T, int k) {
  if (!P.filt) return false;
  bool v = true;
  if (T.factored) {
    const int64_t off = P.single ? 0 : T.elem_off;
    const uintptr_t pb = P.ntab ? (uintptr_t)P.ptab[k - P.t0] : (uintptr_t)P.p + off * P.psz;
    const uintptr_t gb = P.ntab ? (uintptr_t)P.gtab[k - P.t0] : (uintptr_t)P.g + off * P.gsz;
    v = T.cols % 8 == 0 && pb % (8 * P.psz) == 0 && gb % (8 * P.gsz) == 0;
  }
  return v != (P.filt == 1);
}

// ============================ K1: statistics =====================================
// MODE bit 1: gradient statistics (row sums, column partials, sum g^2, sum v_row_old);
// bit 2: parameter statistics (sum p^2).  MODE 3 is the normal pass; the host-span
// clipped form (mco_adalomo_apply_all_host) runs MODE 1 while the gradients stream in
// and MODE 2 per tensor once its parameters have arrived -- same loops and accumulation
// order, so the statistics are bit-identical to MODE 3's.
constexpr int kStatsG = 1, kStatsP = 2, kStatsAll = 3;
//
// early (hook form, one tensor after another on one stream): the previous kernel is the
// previous tensor's K6, which triggers its dependents as soon as it starts, and writes
// only that tensor's parameters -- nothing this kernel reads.  So this pass starts
// without waiting and fills the SMs K6's tail leaves idle; it waits before it exits, so
// its own completion still implies K6's (every later kernel's pdl_wait stays transitive).
template <bool VEC, typename GT, typename PT, int MODE>
__global__ void __launch_bounds__(kThreads, k1_minb<GT, PT>())
    k1_stats(Ctx c, Ptrs P, int64_t tile0, int64_t ntiles, int early) {
  constexpr bool SG = MODE & kStatsG, SP = MODE & kStatsP;
  if (!early) pdl_wait();
  __shared__ float colbuf[kThreads * VW];
  __shared__ float rowbuf[kMaxTileRows * 4];
  __shared__ double scratch[32];
  for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const Tile tl = c.tiles[tile0 + ti];
    const TensorInfo T = c.tensors[tl.tensor];
    if (skip_tensor(P, T, tl.tensor)) continue;
    const GT* g = gptr<GT>(P, T, tl.tensor);
    const PT* p = pptr<PT>(P, T, tl.tensor);
    double psq = 0.0, gsq = 0.0;
    if (T.factored) {
      const int TC = T.tc, TR = kThreads / T.tc;
      const int lane_c = threadIdx.x % TC, tr = threadIdx.x / TC;
      int64_t col;
      int cs, valid;
      lane_cols<VEC>(tl, lane_c, col, cs, valid);
      const int wrow = (threadIdx.x % TC) >> 5;  // warp index within the row group
      const int nwr = TC >> 5;
      float cacc[VW];
#pragma unroll
      for (int j = 0; j < VW; ++j) cacc[j] = 0.f;
      // RB rows per iteration: all their loads are in flight before any math
      constexpr int RB = k1_rows<GT, PT>();
      // 32-bit row indices within the tile (h <= 128), row pointers advanced by adds
      // (fp32 7B: K1 833 -> 820 us under ncu; the bf16 tile loops of K4 / K6 measured no
      // better this way and keep their 64-bit form)
      const int h = (int)(tl.r1 - tl.r0);
      const int64_t rstep = (int64_t)TR * T.cols;
      const GT* gq = g + (tl.r0 + tr) * T.cols + col;
      const PT* pq = p + (tl.r0 + tr) * T.cols + col;
      for (int lr0 = tr; lr0 < h; lr0 += RB * TR) {
        RowVec<VEC, GT, true> gr[RB];
        RowVec<VEC, PT, false> pr[RB];
#pragma unroll
        for (int b = 0; b < RB; ++b) {
          if (valid > 0 && lr0 + b * TR < h) {
            if constexpr (SG) gr[b].load(gq + b * rstep, valid);
            if constexpr (SP) pr[b].load(pq + b * rstep, valid);
          } else {
            gr[b].zero();
            pr[b].zero();
          }
        }
        gq += RB * rstep;
        pq += RB * rstep;
        float sg[RB];
#pragma unroll
        for (int b = 0; b < RB; ++b) {
          float gv[VW], pv[VW];
          if constexpr (SG) gr[b].get(gv);
          if constexpr (SP) pr[b].get(pv);
          float sp = 0.f;
          sg[b] = 0.f;
#pragma unroll
          for (int j = 0; j < VW; ++j) {  // fused multiply-adds: K1 on bf16 data is issue-bound
            if constexpr (SG) {
              cacc[j] = __fmaf_rn(gv[j], gv[j], cacc[j]);
              sg[b] = __fmaf_rn(gv[j], gv[j], sg[b]);
            }
            if constexpr (SP) sp = __fmaf_rn(pv[j], pv[j], sp);
          }
          if constexpr (SP) psq += (double)sp;
        }
        if constexpr (SG) {
          // the RB rows' sums over the warp's 256 columns in one multi-value butterfly (a
          // warp never straddles two rows: TC >= 32); lane group of row b writes it
          const float tot = warp_sum_rows<RB>(sg);
          const int lane = threadIdx.x & 31, b = warp_rows_index<RB>(lane);
          const int lr = lr0 + b * TR;
          if ((lane & (32 / RB - 1)) == 0 && lr < h) rowbuf[lr * nwr + wrow] = tot;
        }
      }
      if constexpr (!SG) {  // parameter statistics only
        const double bps = block_sum(psq, scratch);
        if (threadIdx.x == 0) c.tile_sc[(tile0 + ti) * 4 + 0] = bps;
        continue;
      }
      // column partials: fixed-order sum over the TR row groups
      if constexpr (SG) {
#pragma unroll
        for (int j = 0; j < VW; ++j) colbuf[(tr * TC + lane_c) * VW + j] = cacc[j];
      }
      __syncthreads();
      const int64_t w = tl.c1 - tl.c0;
      for (int64_t q = threadIdx.x; q < w; q += kThreads) {
        int lc, j;
        col_lane<VEC>((int)q, lc, j);
        float s = 0.f;
        for (int k = 0; k < TR; ++k) s += colbuf[(k * TC + lc) * VW + j];
        c.colpart[T.colpart_off + tl.rb * T.cols + tl.c0 + q] = s;
      }
      // row partials
      double vrs = 0.0;
      for (int64_t i = threadIdx.x; i < h; i += kThreads) {
        double s = 0.0;
        for (int k = 0; k < nwr; ++k) s += (double)rowbuf[i * nwr + k];
        c.rowpart[T.rowpart_off + (int64_t)tl.cb * T.rows + tl.r0 + i] = s;
        gsq += s;
        if (tl.cb == 0) vrs += c.state[T.vrow_off + tl.r0 + i];
      }
      const double bps = SP ? block_sum(psq, scratch) : 0.0;
      const double bgs = block_sum(gsq, scratch);
      const double bvr = block_sum(vrs, scratch);
      if (threadIdx.x == 0) {
        if constexpr (SP) c.tile_sc[(tile0 + ti) * 4 + 0] = bps;
        c.tile_sc[(tile0 + ti) * 4 + 1] = bgs;
        c.tile_sc[(tile0 + ti) * 4 + 2] = bvr;
      }
      __syncthreads();  // colbuf / rowbuf reuse by the next tile
    } else {
      for (int64_t e = tl.r0 + threadIdx.x; e < tl.r1; e += kThreads) {
        if constexpr (SG) {
          const double gv = (double)ld1(g + e);
          gsq += gv * gv;
        }
        if constexpr (SP) {
          const double pv = (double)ldp1(p + e);
          psq += pv * pv;
        }
      }
      const double bps = SP ? block_sum(psq, scratch) : 0.0;
      const double bgs = SG ? block_sum(gsq, scratch) : 0.0;
      if (threadIdx.x == 0) {
        if constexpr (SP) c.tile_sc[(tile0 + ti) * 4 + 0] = bps;
        if constexpr (SG) {
          c.tile_sc[(tile0 + ti) * 4 + 1] = bgs;
          c.tile_sc[(tile0 + ti) * 4 + 2] = 0.0;
        }
      }
    }
  }
  if (early) pdl_wait();
}

// One lane's (thread's) share of a strided fixed-order sum: x(i0) + x(i0 + stride) + ...
// over [i0, end), added in that order, with the loads issued 8 at a time so their
// latencies overlap (a one-tensor call reduces ~450 tile partials per tensor in one warp:
// 14 dependent L2 round trips per lane before).  The padding adds +0.0, which leaves
// every sum here (of squares / of non-negative statistics) bit-unchanged.
// B loads per batch (16 where one lane walks ~14 partials of a one-tensor call: one L2
// round trip instead of two); the batch size never changes the order of the additions.
template <int B = 8, typename F>
__device__ __forceinline__ double strided_sum(int64_t i0, int64_t end, int64_t stride, F x) {
  double acc = 0.0;
  for (int64_t i = i0; i < end; i += B * stride) {
    double v[B];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int64_t j = i + q * stride;
      v[q] = j < end ? x(j) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < B; ++q) acc += v[q];
  }
  return acc;
}
// three strided sums over the same index set in one walk (each in strided_sum's order):
// the loads of all three are in flight together
template <typename F>
__device__ __forceinline__ void strided_sum3(int64_t i0, int64_t end, int64_t stride, F x,
                                             double& a0, double& a1, double& a2) {
  a0 = a1 = a2 = 0.0;
  for (int64_t i = i0; i < end; i += 8 * stride) {
    double v[8][3];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t j = i + q * stride;
#pragma unroll
      for (int r = 0; r < 3; ++r) v[q][r] = j < end ? x(j, r) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      a0 += v[q][0];
      a1 += v[q][1];
      a2 += v[q][2];
    }
  }
}

// K2's / K5's work, also run inside KR / K4 by unsharded (fused) calls
__device__ void k2_body(const Ctx& c, int t0, int t1, double lr, double b2, int use_clip,
                        double clip, const double* ext_sumsq, double* red);
__device__ void k5_body(const Ctx& c, int t0, int t1, double adalomo_clip);
__device__ void k2_one(const Ctx& c, int k, double gsq, double psq, double vrs, double lr,
                       double b2, int use_clip, double clip, const double* ext_sumsq);
__device__ __forceinline__ void k5_val(const Ctx& c, int k, double us, double numel, double lrt,
                                       double adalomo_clip);

// ============================ KR: tile partials -> payload ===========================
// Blocks [0, ncolblk): one thread per column of the factored tensors in [t0,t1):
// fixed-order sum of the tile column partials.  Blocks ncolblk + i: tensor t0 + i's
// tile scalars (sum p^2, g^2, v_row_old), 256 thread-strided partials in a block_sum --
// one block per tensor, so a one-tensor call (hook form) reduces its ~450 tiles with
// 256 threads instead of one warp (KR 11.3 us -> see DESIGN.md), and every form of the
// call sums a tensor in the same order.  Everything is scaled by the tensor's shard
// weight (1, or 0 on ranks that hold a replica another rank already contributes), so an
// all-reduce of the payload yields global sums.  fuse2 (no all-reduce between the
// phases): the last tensor block to finish (ticket) runs K2's body for the call.
__device__ __forceinline__ void tensor_stats(const Ctx& c, int k, int mode, bool one,
                                             double* red, double* out = nullptr) {
  const TensorInfo T = c.tensors[k];
  const int64_t i0 = T.tile_begin + threadIdx.x;
  double ps, gs, vr;
  if (one) {  // one-tensor call (hook form): the three walks' loads in flight together
    strided_sum3(i0, T.tile_end, blockDim.x, [&](int64_t i, int r) { return c.tile_sc[i * 4 + r]; },
                 ps, gs, vr);
  } else {  // (measured: the fused walk slows multi-tensor calls slightly)
    ps = strided_sum(i0, T.tile_end, blockDim.x, [&](int64_t i) { return c.tile_sc[i * 4 + 0]; });
    gs = strided_sum(i0, T.tile_end, blockDim.x, [&](int64_t i) { return c.tile_sc[i * 4 + 1]; });
    vr = strided_sum(i0, T.tile_end, blockDim.x, [&](int64_t i) { return c.tile_sc[i * 4 + 2]; });
  }
  ps = block_sum(ps, red);
  gs = block_sum(gs, red);
  vr = block_sum(vr, red);
  if (threadIdx.x == 0) {
    if (mode & kStatsG) {
      c.pay[k * 3 + 0] = T.weight * gs;
      c.pay[k * 3 + 2] = T.weight * vr;
    }
    if (mode & kStatsP) c.pay[k * 3 + 1] = T.weight * ps;
    if (out) {  // thread 0: the payload values, for k2_one
      out[0] = T.weight * gs;
      out[1] = T.weight * ps;
      out[2] = T.weight * vr;
    }
  }
}

__global__ void __launch_bounds__(kThreads)
    kr_stats(Ctx c, int t0, int t1, const int64_t* __restrict__ col_off, int64_t ncols,
             int ncolblk, int mode, int fuse2, double lr, double b2, int use_clip, double clip,
             const double* ext_sumsq) {
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((int)blockIdx.x < ncolblk) {
    // 32 columns per CTA (one per lane, coalesced rows of the partials); the 8 warps
    // take row blocks warp, warp+8, ... and are combined in warp order: a fixed order,
    // with 8x the loads in flight of one thread walking all row blocks (the single-
    // tensor hook form launches only C/32 CTAs here)
    __shared__ double part[kThreads / 32][32];
    const int64_t gi = col_off[t0] + (int64_t)blockIdx.x * 32 + lane;
    const bool valid = gi < col_off[t0] + ncols;
    double acc = 0.0;
    int64_t slot = -1;
    double w = 0.0;
    if (valid) {
      int lo = t0, hi = t1 - 1;  // largest k with col_off[k] <= gi
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (col_off[mid] <= gi)
          lo = mid;
        else
          hi = mid - 1;
      }
      const TensorInfo& T = c.tensors[lo];
      const int64_t j = gi - col_off[lo];
      const float* src = c.colpart + T.colpart_off + j;
      const int64_t nrb = T.nrb, C = T.cols;
      auto ld = [&](int64_t rb) { return (double)src[rb * C]; };
      acc = t1 - t0 == 1 ? strided_sum<16>(warp, nrb, nw, ld) : strided_sum(warp, nrb, nw, ld);
      slot = 3 * c.ntens + T.fb_off + j;
      w = T.weight;
    }
    part[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && valid) {
      double sum = 0.0;
      for (int q = 0; q < nw; ++q) sum += part[q][lane];
      c.pay[slot] = w * sum;
    }
    return;
  }
  __shared__ double red[32];
  if (fuse2 && t1 - t0 == 1 && mode == kStatsAll) {  // one-tensor fused call (hook form)
    double v[3];
    tensor_stats(c, t0, mode, true, red, v);
    if (threadIdx.x == 0) k2_one(c, t0, v[0], v[1], v[2], lr, b2, use_clip, clip, ext_sumsq);
    return;
  }
  tensor_stats(c, t0 + (int)blockIdx.x - ncolblk, mode, t1 - t0 == 1, red);
  if (fuse2) {  // unsharded call: the last tensor block does K2's work
    __shared__ bool last;
    unsigned* ticket = reinterpret_cast<unsigned*>(c.glob + 4);
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(ticket, 1u) == (unsigned)(t1 - t0) - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      k2_body(c, t0, t1, lr, b2, use_clip, clip, ext_sumsq, red);
      if (threadIdx.x == 0) *ticket = 0u;
    }
  }
}

// tensor k's sum u^2 from K4's tile sums, by one warp (lane-strided, warp_sum)
__device__ __forceinline__ double usq_one(const Ctx& c, int k, int lane, bool one) {
  const TensorInfo T = c.tensors[k];
  // L2 reads (__ldcg): K4's tile sums, written by other CTAs of its grid
  auto ld = [&](int64_t i) { return __ldcg(&c.tile_sc[i * 4 + 3]); };
  double us = one ? strided_sum<16>(T.tile_begin + lane, T.tile_end, 32, ld)
                  : strided_sum(T.tile_begin + lane, T.tile_end, 32, ld);
  us = warp_sum(us);
  if (lane == 0) c.pay_usq[k] = T.weight * us;
  return T.weight * us;  // the payload value (lane 0)
}
__device__ __forceinline__ void usq_payload(const Ctx& c, int t0, int t1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = t0 + warp; k < t1; k += nw) usq_one(c, k, lane, t1 - t0 == 1);
}

__global__ void __launch_bounds__(1024) kr_usq(Ctx c, int t0, int t1) {
  pdl_wait();
  usq_payload(c, t0, t1);
}

// Global sum of g^2 over tensors [t0, t1) from the payload, in K2's order (same
// threads, strides and block reduction), so a clip scale computed from it equals the
// one K2 derives over the same range bit for bit.
__global__ void __launch_bounds__(kThreads) kg_sumsq(Ctx c, int t0, int t1, double* out) {
  pdl_wait();
  __shared__ double red[32];
  double G = 0;
  for (int k = t0 + threadIdx.x; k < t1; k += blockDim.x) G += c.pay[k * 3 + 0];
  G = block_sum(G, red);
  if (threadIdx.x == 0) *out = G;
}

// ============================ K2: per-tensor scalars ===============================
// One CTA of kThreads threads (k2_scalars, or KR's scalar block in fused calls).  Thread
// i handles tensors i, i + kThreads, ...: the per-tensor sums, then the global sum of g^2
// over the call's tensors (fixed order: block_sum), the clip scale and the per-tensor
// scalars.
// K2's clip rule (optim.cpp:302-303 on the global norm) and per-tensor scalars, shared by
// k2_body and k2_one so both compute them with the same operations
__device__ __forceinline__ double k2_clip_scale(double G, int use_clip, double clip,
                                                const double* ext_sumsq) {
  double s = 1.0;
  if (use_clip) {
    const double sumsq = ext_sumsq ? *ext_sumsq : G;
    const double norm = sqrt(sumsq);
    if (norm > clip && norm > 0) s = clip / norm;
  }
  return s;
}
__device__ __forceinline__ void k2_tensor(const Ctx& c, int k, double s, double lr, double b2,
                                          double gsq_k, double psq_k, double vrs_k) {
  TensorInfo* Tm = const_cast<TensorInfo*>(&c.tensors[k]);
  const TensorInfo T = *Tm;
  const int64_t t = T.t + 1;  // optim.cpp:219
  Tm->t = t;
  const double corr = 1.0 - pow(b2, (double)t);
  const double n = (double)T.numel_global;
  const double rms_theta = sqrt(psq_k / n);
  const double lr_t = lr * fmax(1e-3, rms_theta);
  double row_mean = 0.0;
  if (T.factored) {  // mean of the new v_row, by linearity of the EMA
    const double gsq = s * s * gsq_k;
    const double sum_new = b2 * vrs_k + (1 - b2) * (gsq / (double)T.cols);
    row_mean = sum_new / ((double)T.rows_global * corr);
  }
  c.tens_sc[k * kTensScalars + TS_CORR] = corr;
  c.tens_sc[k * kTensScalars + TS_LRT] = lr_t;
  c.tens_sc[k * kTensScalars + TS_ROWMEAN] = row_mean;
  c.mins[2 * k] = c.mins[2 * k + 1] = 0x7f800000u;  // +inf: K3 lowers them
}

__device__ void k2_body(const Ctx& c, int t0, int t1, double lr, double b2, int use_clip,
                        double clip, const double* ext_sumsq, double* red) {
  // per-tensor sums arrive (already all-reduced across ranks when sharded) in the payload
  // (L2 reads: in fused calls other blocks of the same grid wrote them, kr_stats)
  for (int k = t0 + threadIdx.x; k < t1; k += blockDim.x) {
    c.tens_sc[k * kTensScalars + TS_GSQ] = __ldcg(&c.pay[k * 3 + 0]);
    c.tens_sc[k * kTensScalars + TS_PSQ] = __ldcg(&c.pay[k * 3 + 1]);
    c.tens_sc[k * kTensScalars + TS_VRS] = __ldcg(&c.pay[k * 3 + 2]);
  }
  __syncthreads();
  double G = 0;
  for (int k = t0 + threadIdx.x; k < t1; k += blockDim.x) G += c.tens_sc[k * kTensScalars + TS_GSQ];
  G = block_sum(G, red);
  if (threadIdx.x == 0) {
    c.glob[0] = k2_clip_scale(G, use_clip, clip, ext_sumsq);
    c.glob[1] = G;
  }
  __syncthreads();
  const double s = c.glob[0];
  for (int k = t0 + threadIdx.x; k < t1; k += blockDim.x)
    k2_tensor(c, k, s, lr, b2, c.tens_sc[k * kTensScalars + TS_GSQ],
              c.tens_sc[k * kTensScalars + TS_PSQ], c.tens_sc[k * kTensScalars + TS_VRS]);
}

// K2 for a one-tensor fused call, by thread 0 of KR's tensor block, from the payload values
// it has just formed (gsq, psq, vrs -- what k2_body would read back): the same bits as
// k2_body (its block sum over one tensor adds only zeros) without the ticket and three
// dependent L2 round trips on the hook form's critical path.
__device__ void k2_one(const Ctx& c, int k, double gsq, double psq, double vrs, double lr,
                       double b2, int use_clip, double clip, const double* ext_sumsq) {
  c.tens_sc[k * kTensScalars + TS_GSQ] = gsq;
  c.tens_sc[k * kTensScalars + TS_PSQ] = psq;
  c.tens_sc[k * kTensScalars + TS_VRS] = vrs;
  const double G = gsq;
  const double s = k2_clip_scale(G, use_clip, clip, ext_sumsq);
  c.glob[0] = s;
  c.glob[1] = G;
  k2_tensor(c, k, s, lr, b2, gsq, psq, vrs);
}

__global__ void __launch_bounds__(kThreads)
    k2_scalars(Ctx c, int t0, int t1, double lr, double b2, int use_clip, double clip,
               const double* ext_sumsq) {
  pdl_wait();
  __shared__ double red[32];
  k2_body(c, t0, t1, lr, b2, use_clip, clip, ext_sumsq, red);
}

// ============================ K3: moments ============================================
// Item space: for each factored tensor in [t0,t1): rows then columns.
//
// Besides a_i and b_j, K3 writes their reciprocal square roots (from the fp64 values,
// rounded once) and lowers the tensor's min a / min b (fp32 bits, atomicMin: a, b >= 0,
// so the bit order is the value order -- deterministic), one atomic per warp and
// (tensor, rows|cols) group.  K4 / K6 use them for the separable form of u (sep_ok).
__global__ void __launch_bounds__(kThreads)
    k3_moments(Ctx c, int t0, int t1, const int64_t* __restrict__ item_off, int64_t item0,
               int64_t nitems, double b2) {
  pdl_wait();
  const double s = c.glob[0], s2 = s * s;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count (the min reduction below needs all 32 lanes)
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < nitems;
       base += stride) {
    const int64_t it = base + lane;
    unsigned key = 0xffffffffu, bits = 0x7f800000u;
    if (it < nitems) {
      // binary search the tensor owning this item
      const int64_t gi = item0 + it;
      int lo = t0, hi = t1 - 1;  // largest k with item_off[k] <= gi
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (item_off[mid] <= gi)
          lo = mid;
        else
          hi = mid - 1;
      }
      const TensorInfo T = c.tensors[lo];
      const int64_t local = gi - item_off[lo];
      const double corr = c.tens_sc[lo * kTensScalars + TS_CORR];
      if (local < T.rows) {  // row i: optim.cpp:239-240
        const int64_t i = local;
        double acc = 0.0;
        for (int k = 0; k < T.kc; ++k) acc += c.rowpart[T.rowpart_off + (int64_t)k * T.rows + i];
        double& vr = c.state[T.vrow_off + i];
        vr = b2 * vr + (1 - b2) * (s2 * acc / (double)T.cols);
        const double a = vr / corr;
        c.fa[T.fa_off + i] = (float)a;
        c.fra[T.fa_off + i] = (float)(1.0 / sqrt(a));
        key = 2u * (unsigned)lo;
        bits = __float_as_uint((float)a);
      } else {  // column j: optim.cpp:247-248
        const int64_t j = local - T.rows;
        const double acc = c.pay[3 * c.ntens + T.fb_off + j];  // all-reduced column sum
        double& vc = c.state[T.vcol_off + j];
        vc = b2 * vc + (1 - b2) * (s2 * acc / (double)T.rows_global);
        const double rm = c.tens_sc[lo * kTensScalars + TS_ROWMEAN];
        const double b = (vc / corr) / fmax(rm, 1e-300);
        c.fb[T.fb_off + j] = (float)b;
        c.frb[T.fb_off + j] = (float)(1.0 / sqrt(b));
        key = 2u * (unsigned)lo + 1u;
        bits = __float_as_uint((float)b);
      }
    }
    const unsigned k0 = __shfl_sync(0xffffffffu, key, 0);
    if (__all_sync(0xffffffffu, key == k0 || key == 0xffffffffu)) {
      const unsigned m = __reduce_min_sync(0xffffffffu, bits);
      if (lane == 0 && k0 != 0xffffffffu) atomicMin(&c.mins[k0], m);
    } else if (key != 0xffffffffu) {
      atomicMin(&c.mins[key], bits);
    }
  }
}

// Separable form of u in K4: when eps <= 2^-26 a_i b_j for every element of the tensor,
// eps moves a_i b_j + eps by < 2^-26 relative (u by < 2^-27), and
//   sum u_ij^2 = s^2 sum_i (1/a_i) sum_j (g_ij / sqrt(b_j))^2
// within fp32 rounding -- no per-element MUFU.RSQ (K4 reads 2-4 B per element and was
// issue-bound on it, bf16 the most).  K6 keeps the per-element form (it is bound by
// latency, not issue; u there and here agree to ~3e-7 relative, far inside the damping
// factor's use).  min a, min b >= 2^-60 keeps every
// product and the squares K4 sums far from fp32 underflow / overflow.  Otherwise (eps
// not negligible, zero rows, vanishing gradients) the per-element form below runs.
__device__ __forceinline__ bool sep_ok(const Ctx& c, int k, double eps) {
  const float ma = __uint_as_float(c.mins[2 * k]), mb = __uint_as_float(c.mins[2 * k + 1]);
  return ma >= 0x1p-60f && mb >= 0x1p-60f && (double)ma * (double)mb * 0x1p-26 >= eps;
}

// u for a factored element: u = (s*g) / sqrt(a_i*b_j + eps)   (optim.cpp:256-259),
// evaluated as (s*g) * rsqrt(.) -- MUFU.RSQ, <= 2 ulp -- instead of an IEEE sqrt and
// an IEEE division: K4 reads 4 B/element and would otherwise be issue-bound.
// K4 and K6 evaluate the identical expression, so both see the same u.  a*b + eps is
// one fused multiply-add (explicit: the library is built with --fmad=false so that the
// stored-state kernels keep the reference's operation order; AdaLomo is compared
// within the fp32 tolerance of the fp64 reference).
// rsqrt.approx.ftz: the flush-to-zero form is one MUFU.RSQ, the default form wraps it in
// a subnormal check and two scaling multiplies (3 more instructions per element in the
// issue-bound K4).  Its argument a*b + eps is never subnormal -- eps is clamped to
// FLT_MIN (ada_eps) and a, b >= 0 -- so both forms give the same bits.
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ada_eps(double eps) { return fmaxf((float)eps, FLT_MIN); }

__device__ __forceinline__ float u_fact(float g, float s, float a, float b, float eps) {
  const float gs = s * g;
  return gs * rsqrt_ftz(__fmaf_rn(a, b, eps));
}

// K6's update of one 8-element row vector, every K6 traversal (tiles, flat chunks, the
// bulk-copy pipeline): p <- fma(-f, u, p) with u = u_fact(g, s, a, b_j, eps) -- one
// rounding for p - f*u.  (A packed-pair FMUL2 / FFMA2 form halved the FP issue slots but
// measured no faster on bf16 data -- 7B: 14.2 vs 14.1 ms -- and is not kept.)
__device__ __forceinline__ void k6_row8(float (&pv)[8], const float (&gv)[8], float a,
                                        const float (&bv)[8], float sf, float ff, float eps) {
#pragma unroll
  for (int j = 0; j < 8; ++j) pv[j] = __fmaf_rn(-ff, u_fact(gv[j], sf, a, bv[j], eps), pv[j]);
}
__device__ __forceinline__ float k6_one(float p, float g, float a, float b, float sf, float ff,
                                        float eps) {
  return __fmaf_rn(-ff, u_fact(g, sf, a, b, eps), p);  // == one element of k6_row8
}

// row / col of element e of a factored tensor: e / C by multiply-high with the
// per-tensor magic (set_fast_div; exact for e < 2^31) instead of the ~20-instruction
// 32-bit udiv -- K4 is issue-bound (ncu: 68 % issue active).
__device__ __forceinline__ void row_col(uint32_t e, const TensorInfo& T, uint32_t C,
                                        uint32_t& row, uint32_t& col) {
  row = C == 1 ? e : (__umulhi(e, T.div_m) >> T.div_s);
  col = e - row * C;
}

// ============================ K4: sum u^2 ============================================
// Over the statistics tiles, like K1: each lane owns one 8-column chunk of the tile, so
// b_j (or 1/sqrt(b_j)) sits in registers for the whole tile and a row costs one a_i
// load -- no per-vector index arithmetic (the flat-chunk traversal spent ~14 address
// instructions per 8 elements, with K4 issue-bound on bf16 data).  Rows in flight: one
// stream only, so twice K1's.  The per-tile sums go to tile_sc[.][3].
#ifndef MCO_K4_RB_BF16
#define MCO_K4_RB_BF16 (4 * kRB)
#endif
#ifndef MCO_K4_RB_F32
#define MCO_K4_RB_F32 (2 * kRB)
#endif
template <typename GT>
constexpr int k4_rows() {
  return sizeof(GT) == 2 ? MCO_K4_RB_BF16 : MCO_K4_RB_F32;
}
#ifndef MCO_K6_RB_F32
#define MCO_K6_RB_F32 0  // A/B knob: K6 tiles' rows in flight on fp32 data (0: kRB)
#endif
template <typename GT, typename PT>
constexpr int k6_rows() {
  return (MCO_K6_RB_F32 && sizeof(GT) == 4 && sizeof(PT) == 4) ? MCO_K6_RB_F32
                                                               : rows_in_flight<GT, PT>();
}

// K4's tile loop (k4_usq)
template <bool VEC, typename GT>
__device__ __forceinline__ void k4_tiles(const Ctx& c, const Ptrs& P, int64_t tile0,
                                         int64_t ntiles, double b2, double eps,
                                         double* scratch) {
  const float sf = (float)c.glob[0], epsf = ada_eps(eps);
  for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const Tile tl = c.tiles[tile0 + ti];
    const TensorInfo T = c.tensors[tl.tensor];
    if (skip_tensor(P, T, tl.tensor)) continue;
    const GT* g = gptr<GT>(P, T, tl.tensor);
    double usq = 0.0;
    if (T.factored) {
      const int TC = T.tc, TR = kThreads / T.tc;
      const int lane_c = threadIdx.x % TC, tr = threadIdx.x / TC;
      int64_t col;
      int cs, valid;
      lane_cols<VEC>(tl, lane_c, col, cs, valid);
      if (valid > 0) {
        const bool sep = sep_ok(c, tl.tensor, eps);
        const float* fa = (sep ? c.fra : c.fa) + T.fa_off;
        float bv[VW];
#pragma unroll
        for (int j = 0; j < VW; ++j)
          bv[j] = j < valid ? (sep ? c.frb : c.fb)[T.fb_off + col + j * cs] : 0.f;
        constexpr int RB = k4_rows<GT>();
        const int64_t rstep = (int64_t)TR * T.cols;  // row pointers advance by adds
        uint64_t bv2[VW / 2];
#pragma unroll
        for (int j = 0; j < VW; j += 2) bv2[j / 2] = pk2(bv[j], bv[j + 1]);
        // one row loop per form of u (the per-row branch is gone from the hot loop); a_i
        // is loaded with its row, and rows past the tile read as zeros (exact zero terms)
        auto rows = [&](auto sep_tag) {
          constexpr bool SEP = decltype(sep_tag)::value;
          const GT* grow = g + (tl.r0 + tr) * T.cols + col;
          for (int64_t r0 = tl.r0 + tr; r0 < tl.r1; r0 += (int64_t)RB * TR) {
            RowVec<VEC, GT, true> gr[RB];
            float av[RB];
            const GT* gb = grow;
#pragma unroll
            for (int b = 0; b < RB; ++b, gb += rstep) {
              const int64_t r = r0 + (int64_t)b * TR;
              if (r < tl.r1) {
                gr[b].load(gb, valid);
                av[b] = fa[r];
              } else {
                gr[b].zero();
                av[b] = 0.f;
              }
            }
            grow = gb;
            float su = 0.f;
#pragma unroll
            for (int b = 0; b < RB; ++b) {
              float gv[VW];
              gr[b].get(gv);
              if constexpr (SEP) {  // a = 1/sqrt(a_i), bv = 1/sqrt(b_j): ra^2 sum_j (g rb)^2
                uint64_t rs2 = 0;  // even / odd column partials (FMUL2 / FFMA2)
#pragma unroll
                for (int j = 0; j < VW; j += 2) {
                  const uint64_t x = mul2(pk2(gv[j], gv[j + 1]), bv2[j / 2]);
                  rs2 = fma2(x, x, rs2);
                }
                float re, ro;
                up2(rs2, re, ro);
                su = __fmaf_rn(av[b] * av[b], re + ro, su);
              } else {
#pragma unroll
                for (int j = 0; j < VW; ++j) {  // s is applied once per tile (s^2 below)
                  const float x = gv[j] * rsqrt_ftz(__fmaf_rn(av[b], bv[j], epsf));
                  su = __fmaf_rn(x, x, su);
                }
              }
            }
            usq += (double)su;
          }
        };
        if (sep)
          rows(std::true_type{});
        else
          rows(std::false_type{});
      }
      usq *= (double)sf * (double)sf;  // sum (s g r)^2 = s^2 sum (g r)^2
    } else {  // optim.cpp:262-267 with fp64 state
      const double s = c.glob[0];
      const double corr = c.tens_sc[tl.tensor * kTensScalars + TS_CORR];
      for (int64_t e = tl.r0 + threadIdx.x; e < tl.r1; e += kThreads) {
        const double gs = s * (double)ld1(g + e);
        double& v = c.state[T.vfull_off + e];
        v = b2 * v + (1 - b2) * gs * gs;
        const double u = gs / sqrt(v / corr + eps);
        usq += u * u;
      }
    }
    const double b = block_sum(usq, scratch);
    if (threadIdx.x == 0) c.tile_sc[(tile0 + ti) * 4 + 3] = b;
  }
}

template <bool VEC, typename GT>
__global__ void __launch_bounds__(kThreads, k4_minb<GT>())
    k4_usq(Ctx c, Ptrs P, int64_t tile0, int64_t ntiles, double b2, double eps, int t0, int t1,
           int fuse5, double adalomo_clip) {
  pdl_wait();
  __shared__ double scratch[32];
  __shared__ bool last;
  k4_tiles<VEC, GT>(c, P, tile0, ntiles, b2, eps, scratch);
  if (fuse5) {  // unsharded call: the last CTA to finish does K5's reduction and damping
    unsigned* ticket = reinterpret_cast<unsigned*>(c.glob + 3);
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      if (t1 - t0 == 1) {  // one tensor: K5 from warp 0's sum in registers (same bits)
        if (threadIdx.x < 32) {
          const double lrt = c.tens_sc[t0 * kTensScalars + TS_LRT];  // in flight with the sum
          const double numel = (double)c.tensors[t0].numel_global;
          const double us = usq_one(c, t0, threadIdx.x, true);
          if (threadIdx.x == 0) k5_val(c, t0, us, numel, lrt, adalomo_clip);
        }
      } else {
        usq_payload(c, t0, t1);
        __syncthreads();
        k5_body(c, t0, t1, adalomo_clip);
      }
      if (threadIdx.x == 0) *ticket = 0u;
    }
  }
}

// ============================ K5: damping ==============================================
__device__ __forceinline__ void k5_val(const Ctx& c, int k, double us, double numel, double lrt,
                                       double adalomo_clip) {  // optim.cpp:269-273
  const double rms_u = sqrt(us / numel);
  const double damp = fmax(1.0, rms_u / adalomo_clip);
  c.tens_sc[k * kTensScalars + TS_USQ] = us;
  c.tens_sc[k * kTensScalars + TS_F] = lrt / damp;
}
__device__ __forceinline__ void k5_one(const Ctx& c, int k, double adalomo_clip) {
  k5_val(c, k, __ldcg(&c.pay_usq[k]), (double)c.tensors[k].numel_global,
         c.tens_sc[k * kTensScalars + TS_LRT], adalomo_clip);
}
__device__ void k5_body(const Ctx& c, int t0, int t1, double adalomo_clip) {
  for (int k = t0 + (int)threadIdx.x; k < t1; k += blockDim.x) k5_one(c, k, adalomo_clip);
}

__global__ void __launch_bounds__(1024)
    k5_damp(Ctx c, int t0, int t1, double adalomo_clip, int with_usq) {
  pdl_wait();
  if (with_usq) {  // unsharded call: KR2's reduction here, one launch less per tensor
    usq_payload(c, t0, t1);
    __syncthreads();
  }
  k5_body(c, t0, t1, adalomo_clip);
}

// ============================ K6: update ==============================================
template <bool VEC, typename GT>
__device__ __forceinline__ void chunk_vec_load(const GT* g, int64_t e, int64_t e1, float (&v)[VW]) {
  if constexpr (VEC) {
    load8<GT>(g + e, v);
  } else {
#pragma unroll
    for (int j = 0; j < VW; ++j) v[j] = (e + j < e1) ? ld1(g + e + j) : 0.f;
  }
}

template <bool VEC, typename GT, typename PT>
__global__ void __launch_bounds__(kThreads)
    k6_update(Ctx c, Ptrs P, int64_t chunk0, int64_t nchunks, double eps, int trigger) {
  pdl_wait();
  if (trigger) pdl_trigger();  // the next tensor's K1 may start (see k1_stats)
  const float sf = (float)c.glob[0], epsf = ada_eps(eps);
  // reverse chunk order: the tail of K4's gradient reads is still L2-resident
  for (int64_t k = blockIdx.x; k < nchunks; k += gridDim.x) {
    const int64_t ci = nchunks - 1 - k;
    const Chunk ch = c.chunks[chunk0 + ci];
    const TensorInfo T = c.tensors[ch.tensor];
    if (skip_tensor(P, T, ch.tensor)) continue;
    const GT* g = gptr<GT>(P, T, ch.tensor);
    PT* p = pptr<PT>(P, T, ch.tensor);
    const double f = c.tens_sc[ch.tensor * kTensScalars + TS_F];
    if (T.factored) {
      const float ff = (float)f;
      const uint32_t C = (uint32_t)T.cols;
      const float* fa = c.fa + T.fa_off;
      const float* fb = c.fb + T.fb_off;
      constexpr int U6 = 2;
      for (int64_t base = ch.e0 + (int64_t)threadIdx.x * VW; base < ch.e1;
           base += (int64_t)kThreads * VW * U6) {
        float gv[U6][VW], pv[U6][VW];
#pragma unroll
        for (int u = 0; u < U6; ++u) {
          const int64_t e = base + (int64_t)u * kThreads * VW;
          if (e < ch.e1) {
            chunk_vec_load<VEC, GT>(g, e, ch.e1, gv[u]);
            load_p<VEC, PT>(p + e, pv[u], (int)std::min<int64_t>(VW, ch.e1 - e));
          }
        }
#pragma unroll
        for (int u = 0; u < U6; ++u) {
          const int64_t e = base + (int64_t)u * kThreads * VW;
          if (e < ch.e1) {
            if constexpr (VEC) {
              uint32_t row, col;
              row_col((uint32_t)e, T, C, row, col);
              const float a = fa[row];
              const float4 b0 = *reinterpret_cast<const float4*>(fb + col);
              const float4 b1 = *reinterpret_cast<const float4*>(fb + col + 4);
              const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
              k6_row8(pv[u], gv[u], a, bv, sf, ff, epsf);
              store_p<VEC, PT>(p + e, pv[u], VW);
            } else {
#pragma unroll
              for (int j = 0; j < VW; ++j) {
                const int64_t ej = e + j;
                if (ej < ch.e1) {
                  uint32_t row, col;
                  row_col((uint32_t)ej, T, C, row, col);
                  stp1(p + ej, k6_one(pv[u][j], gv[u][j], fa[row], fb[col], sf, ff, epsf));
                }
              }
            }
          }
        }
      }
    } else {
      const double s = c.glob[0];
      const double corr = c.tens_sc[ch.tensor * kTensScalars + TS_CORR];
      for (int64_t e = ch.e0 + threadIdx.x; e < ch.e1; e += kThreads) {
        const double gs = s * (double)ld1(g + e);
        const double u = gs / sqrt(c.state[T.vfull_off + e] / corr + eps);
        stp1(p + e, (float)((double)ldp1(p + e) - f * u));
      }
    }
  }
}

// K6 on the cp.async.bulk pipeline (the chunk traversal's work, staged through shared
// memory).  Items are 4096-element pieces of the call's chunks (16 per 64 Ki chunk; the
// pieces past a short chunk's end are empty and skipped by producer and consumers alike),
// round-robin over one CTA per SM.  One producer lane issues the bulk copies of a piece's
// gradient and parameters into stage s (mbarrier complete_tx), 16 consumer warps update
// the parameters in shared memory (8 elements per thread: row / column of the vector, a_i
// and b_j from L1), and the producer writes the piece back with a bulk store, refilling
// the previous piece's stage as in lomo_tma_kernel.  Bytes in flight per SM are set by
// the stage count (6-8 pieces), not by registers: the register-resident tile K6 on bf16
// data was latency-bound at 0.8 of the copy bandwidth.  Requires every tensor of the
// call at a 16 B aligned start with a whole number of 16 B (host: k6_tma_ok).
constexpr int kK6Piece = 4096;                // elements per piece
constexpr int kK6Consumers = 512;             // 16 warps: one 8-element vector each
constexpr int kK6PPC = (int)(kChunkElems / kK6Piece);
template <typename GT, typename PT>
constexpr int k6_stage_bytes() {
  return kK6Piece * (int)(sizeof(GT) + sizeof(PT));
}
template <typename GT, typename PT>
constexpr int k6_stages() {
  return std::min(8, (200 * 1024) / k6_stage_bytes<GT, PT>());
}
template <typename GT, typename PT>
constexpr int k6_smem() {
  return k6_stages<GT, PT>() * k6_stage_bytes<GT, PT>() + 2 * k6_stages<GT, PT>() * 8;
}

__device__ __forceinline__ bool k6_piece(const Ctx& c, int64_t chunk0, int64_t k, Chunk& ch,
                                         int64_t& e0, int64_t& e1) {
  ch = c.chunks[chunk0 + k / kK6PPC];
  e0 = ch.e0 + (k % kK6PPC) * (int64_t)kK6Piece;
  e1 = std::min<int64_t>(ch.e1, e0 + kK6Piece);
  return e0 < ch.e1;
}

template <typename GT, typename PT>
__global__ void __launch_bounds__(kK6Consumers + 32, 1)
    k6_tma(Ctx c, Ptrs P, int64_t chunk0, int64_t nchunks, double eps, int trigger) {
  constexpr int NS = k6_stages<GT, PT>();
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * k6_stage_bytes<GT, PT>());
  uint64_t* done = full + NS;
  auto sp = [&](int s) { return reinterpret_cast<PT*>(smem + s * k6_stage_bytes<GT, PT>()); };
  auto sg = [&](int s) {
    return reinterpret_cast<GT*>(smem + s * k6_stage_bytes<GT, PT>() + kK6Piece * sizeof(PT));
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], kK6Consumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  if (trigger) pdl_trigger();
  const int64_t nitems = nchunks * kK6PPC;
  // next non-empty item of this CTA at or after k
  auto next = [&](int64_t k) {
    Chunk ch;
    int64_t e0, e1;
    while (k < nitems && !k6_piece(c, chunk0, k, ch, e0, e1)) k += gridDim.x;
    return k;
  };
  if (warp == kK6Consumers / 32) {  // ---------------- producer ----------------
    if (lane == 0) {
      auto issue = [&](int64_t k, int s) {
        Chunk ch;
        int64_t e0, e1;
        k6_piece(c, chunk0, k, ch, e0, e1);
        const TensorInfo& T = c.tensors[ch.tensor];
        const uint32_t n = (uint32_t)(e1 - e0);
        mbar_expect_tx(&full[s], n * (uint32_t)(sizeof(GT) + sizeof(PT)));
        bulk_g2s<false>(sp(s), pptr<PT>(P, T, ch.tensor) + e0, n * (uint32_t)sizeof(PT), &full[s], 0);
        bulk_g2s<false>(sg(s), gptr<GT>(P, T, ch.tensor) + e0, n * (uint32_t)sizeof(GT), &full[s], 0);
      };
      int64_t kf = next(blockIdx.x);
      for (int i = 0; i < NS && kf < nitems; ++i, kf = next(kf + gridDim.x)) issue(kf, i);
      int64_t i = 0;
      for (int64_t kc = next(blockIdx.x); kc < nitems; kc = next(kc + gridDim.x), ++i) {
        const int s = (int)(i % NS);
        mbar_wait(&done[s], (uint32_t)((i / NS) & 1));
        Chunk ch;
        int64_t e0, e1;
        k6_piece(c, chunk0, kc, ch, e0, e1);
        const TensorInfo& T = c.tensors[ch.tensor];
        bulk_s2g<false>(pptr<PT>(P, T, ch.tensor) + e0, sp(s), (uint32_t)(e1 - e0) * sizeof(PT), 0);
        bulk_commit();
        if (i >= 1 && kf < nitems) {  // refill the previous piece's stage
          bulk_wait_read_1();
          issue(kf, (int)((i - 1) % NS));
          kf = next(kf + gridDim.x);
        }
      }
      bulk_wait_all();
    }
    return;
  }
  // ---------------- consumers ----------------
  const float sf = (float)c.glob[0], epsf = ada_eps(eps);
  int64_t i = 0;
  for (int64_t k = next(blockIdx.x); k < nitems; k = next(k + gridDim.x), ++i) {
    const int s = (int)(i % NS);
    Chunk ch;
    int64_t e0, e1;
    k6_piece(c, chunk0, k, ch, e0, e1);
    const TensorInfo& T = c.tensors[ch.tensor];
    const double f = c.tens_sc[ch.tensor * kTensScalars + TS_F];
    mbar_wait(&full[s], (uint32_t)((i / NS) & 1));
    PT* ps = sp(s);
    const GT* gs = sg(s);
    const int n = (int)(e1 - e0);
    if (T.factored) {  // n is a multiple of 8 (C % 8 == 0): whole vectors, one row each
      const float ff = (float)f;
      const uint32_t C = (uint32_t)T.cols;
      for (int v = threadIdx.x; v * 8 < n; v += kK6Consumers) {
        uint32_t row, col;
        row_col((uint32_t)(e0 + v * 8), T, C, row, col);
        const float a = c.fa[T.fa_off + row];
        const float4 b0 = *reinterpret_cast<const float4*>(c.fb + T.fb_off + col);
        const float4 b1 = *reinterpret_cast<const float4*>(c.fb + T.fb_off + col + 4);
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        float gv[8], pv[8];
        if constexpr (sizeof(GT) == 2) {
          const uint4 w = *reinterpret_cast<const uint4*>(gs + v * 8);
          const uint32_t wa[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            gv[2 * q] = __uint_as_float(wa[q] << 16);
            gv[2 * q + 1] = __uint_as_float(wa[q] & 0xffff0000u);
          }
        } else {
          const float4 x0 = *reinterpret_cast<const float4*>(gs + v * 8);
          const float4 x1 = *reinterpret_cast<const float4*>(gs + v * 8 + 4);
          gv[0] = x0.x, gv[1] = x0.y, gv[2] = x0.z, gv[3] = x0.w;
          gv[4] = x1.x, gv[5] = x1.y, gv[6] = x1.z, gv[7] = x1.w;
        }
        if constexpr (sizeof(PT) == 2) {
          const uint4 w = *reinterpret_cast<const uint4*>(ps + v * 8);
          const uint32_t wa[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            pv[2 * q] = __uint_as_float(wa[q] << 16);
            pv[2 * q + 1] = __uint_as_float(wa[q] & 0xffff0000u);
          }
        } else {
          const float4 x0 = *reinterpret_cast<const float4*>(ps + v * 8);
          const float4 x1 = *reinterpret_cast<const float4*>(ps + v * 8 + 4);
          pv[0] = x0.x, pv[1] = x0.y, pv[2] = x0.z, pv[3] = x0.w;
          pv[4] = x1.x, pv[5] = x1.y, pv[6] = x1.z, pv[7] = x1.w;
        }
#pragma unroll
        k6_row8(pv, gv, a, bv, sf, ff, epsf);
        if constexpr (sizeof(PT) == 2) {
          uint4 w;
          w.x = f2bf2_bits(pv[0], pv[1]);
          w.y = f2bf2_bits(pv[2], pv[3]);
          w.z = f2bf2_bits(pv[4], pv[5]);
          w.w = f2bf2_bits(pv[6], pv[7]);
          *reinterpret_cast<uint4*>(ps + v * 8) = w;
        } else {
          *reinterpret_cast<float4*>(ps + v * 8) = make_float4(pv[0], pv[1], pv[2], pv[3]);
          *reinterpret_cast<float4*>(ps + v * 8 + 4) = make_float4(pv[4], pv[5], pv[6], pv[7]);
        }
      }
    } else {  // optim.cpp:262-274, fp64 state (elements of a 1-D tensor)
      const double sd = c.glob[0];
      const double corr = c.tens_sc[ch.tensor * kTensScalars + TS_CORR];
      for (int q = threadIdx.x; q < n; q += kK6Consumers) {
        const double gsd = sd * (double)ld1(gs + q);
        const double u = gsd / sqrt(c.state[T.vfull_off + e0 + q] / corr + eps);
        stp1(ps + q, (float)((double)ldp1(ps + q) - f * u));
      }
    }
    fence_proxy_async();
    mbar_arrive(&done[s]);
  }
}

// K6 over the statistics tiles (alternative traversal; identical arithmetic and result)
template <bool VEC, typename GT, typename PT>
__device__ __forceinline__ void k6_tiles(const Ctx& c, const Ptrs& P, int64_t tile0,
                                         int64_t ntiles, double eps);

template <bool VEC, typename GT, typename PT>
__global__ void __launch_bounds__(kThreads, k6_minb<GT, PT>())
    k6_update_tiles(Ctx c, Ptrs P, int64_t tile0, int64_t ntiles, double eps, int trigger) {
  pdl_wait();
  if (trigger) pdl_trigger();
  k6_tiles<VEC, GT, PT>(c, P, tile0, ntiles, eps);
}

// K6's tile loop (k6_update_tiles)
template <bool VEC, typename GT, typename PT>
__device__ __forceinline__ void k6_tiles(const Ctx& c, const Ptrs& P, int64_t tile0,
                                         int64_t ntiles, double eps) {
  const float sf = (float)c.glob[0], epsf = ada_eps(eps);
  // reverse tile order: the tail of K4's gradient reads is still L2-resident
  for (int64_t k = blockIdx.x; k < ntiles; k += gridDim.x) {
    const int64_t ti = ntiles - 1 - k;
    const Tile tl = c.tiles[tile0 + ti];
    const TensorInfo T = c.tensors[tl.tensor];
    if (skip_tensor(P, T, tl.tensor)) continue;
    const GT* g = gptr<GT>(P, T, tl.tensor);
    PT* p = pptr<PT>(P, T, tl.tensor);
    const double f = c.tens_sc[tl.tensor * kTensScalars + TS_F];
    if (T.factored) {
      const float ff = (float)f;
      const int TC = T.tc, TR = kThreads / T.tc;
      const int lane_c = threadIdx.x % TC, tr = threadIdx.x / TC;
      int64_t col;
      int cs, valid;
      lane_cols<VEC>(tl, lane_c, col, cs, valid);
      if (valid <= 0) continue;
      float bv[VW];
#pragma unroll
      for (int j = 0; j < VW; ++j) bv[j] = j < valid ? c.fb[T.fb_off + col + j * cs] : 0.f;
      const float* fa = c.fa + T.fa_off;
      constexpr int RB = k6_rows<GT, PT>();
      const int64_t rstep = (int64_t)TR * T.cols;  // row offsets advance by adds
      int64_t roff = (tl.r0 + tr) * T.cols + col;
      for (int64_t r0 = tl.r0 + tr; r0 < tl.r1; r0 += (int64_t)RB * TR) {
        RowVec<VEC, GT, true> gr[RB];
        RowVec<VEC, PT, false> pr[RB];
        int64_t o = roff;
#pragma unroll
        for (int b = 0; b < RB; ++b, o += rstep) {
          if (r0 + (int64_t)b * TR < tl.r1) {
            gr[b].load(g + o, valid);
            pr[b].load(p + o, valid);
          }
        }
        o = roff;
#pragma unroll
        for (int b = 0; b < RB; ++b, o += rstep) {
          if (r0 + (int64_t)b * TR < tl.r1) {
            float gv[VW], pv[VW];
            gr[b].get(gv);
            pr[b].get(pv);
            k6_row8(pv, gv, fa[r0 + (int64_t)b * TR], bv, sf, ff, epsf);
            store_tile<VEC, PT>(p + o, pv, valid);
          }
        }
        roff = o;
      }
    } else {
      const double s = c.glob[0];
      const double corr = c.tens_sc[tl.tensor * kTensScalars + TS_CORR];
      for (int64_t e = tl.r0 + threadIdx.x; e < tl.r1; e += kThreads) {
        const double gs = s * (double)ld1(g + e);
        const double u = gs / sqrt(c.state[T.vfull_off + e] / corr + eps);
        stp1(p + e, (float)((double)ldp1(p + e) - f * u));
      }
    }
  }
}

// ============================ one small 1-D tensor, one launch =======================
// The hook form of a norm weight (LLaMA: 4096-8192 elements, 65 of the 7B set's 291
// tensors) ran the 4-launch chain K1 -> KR(K2) -> K4(K5) -> K6 for ~20 KB of data.
// One thread-block cluster (one CTA of 256 threads per plan tile, up to 8 CTAs; a CTA
// takes tiles rank, rank + 8, ...) now runs the whole chain in one launch, with cluster
// barriers where the chain had kernel boundaries and the tile sums gathered in CTA 0's
// shared memory over DSMEM.  It reproduces the chain operation for operation -- each
// tile's block_sum in a 256-thread CTA as K1 / K4 do, KR's tensor_stats and K2's body in
// CTA 0 with 256 threads, usq_payload's lane-strided warp sum, K5's body -- so its bits
// equal the multi-kernel path's, which every other form shares.  (A first version on
// one 1024-thread CTA was issue-latency-bound on one SM: 22 us per call.)
constexpr int kSmallTiles = 32, kSmallCluster = 8, kSmallPer = kSmallTiles / kSmallCluster;
#ifndef MCO_SMALL_EARLY
#define MCO_SMALL_EARLY 1  // A/B: k_small_vec triggers its dependents before its own wait
#endif

template <typename GT, typename PT>
__global__ void __launch_bounds__(kThreads, 1)
    k_small_vec(Ctx c, Ptrs P, int k, double lr, double b2, double eps, int use_clip,
                double clip, const double* ext_sumsq, double adalomo_clip, int trigger) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), cs = (int)cl.num_blocks();
  __shared__ double red[32];
  __shared__ double sc[3][kSmallTiles];  // CTA 0: per tile sum p^2, sum g^2, sum u^2
  __shared__ double bc[3];               // s, corr, f from CTA 0
  // every CTA of the cluster must have started before any DSMEM access: arrive now,
  // wait just before the first remote write (the loads below overlap the barrier)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  // the next tensor's K1 may start now, before this kernel's own wait: it touches only its
  // own tensor and waits at its end (k1_stats early), so it overlaps the previous tensor's
  // K6 as it would without this small call in between
  if (MCO_SMALL_EARLY && trigger) pdl_trigger();
  pdl_wait();
  if (!MCO_SMALL_EARLY && trigger) pdl_trigger();
  const TensorInfo T = c.tensors[k];
  const GT* g = gptr<GT>(P, T, k);
  PT* p = pptr<PT>(P, T, k);
  const int nt = (int)(T.tile_end - T.tile_begin);
  double* sc0 = cl.map_shared_rank(&sc[0][0], 0);
  // every load first: this thread's element of each of the CTA's tiles
  float gv[kSmallPer], pv[kSmallPer];
  double vv[kSmallPer];
  int64_t ev[kSmallPer];
#pragma unroll
  for (int q = 0; q < kSmallPer; ++q) {
    const int ti = rank + q * cs;
    ev[q] = -1;
    if (ti < nt) {
      const Tile tl = c.tiles[T.tile_begin + ti];
      const int64_t e = tl.r0 + threadIdx.x;
      if (e < tl.r1) ev[q] = e;
    }
    gv[q] = ev[q] >= 0 ? ld1(g + ev[q]) : 0.f;
    pv[q] = ev[q] >= 0 ? ldp1(p + ev[q]) : 0.f;
    vv[q] = ev[q] >= 0 ? c.state[T.vfull_off + ev[q]] : 0.0;
  }
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  // K1 (1-D branch): per tile sum p^2, sum g^2 -> CTA 0
#pragma unroll
  for (int q = 0; q < kSmallPer; ++q) {
    const int ti = rank + q * cs;
    if (ti >= nt) break;  // uniform in the CTA
    double gsq = 0.0, psq = 0.0;
    if (ev[q] >= 0) {
      const double g1 = (double)gv[q], p1 = (double)pv[q];
      gsq += g1 * g1;
      psq += p1 * p1;
    }
    const double bps = block_sum(psq, red);
    const double bgs = block_sum(gsq, red);
    if (threadIdx.x == 0) {
      sc0[ti] = bps;
      sc0[kSmallTiles + ti] = bgs;
    }
  }
  cl.sync();
  if (rank == 0) {  // KR's tensor block + K2
    double ps = strided_sum(threadIdx.x, nt, kThreads, [&](int64_t i) { return sc[0][i]; });
    double gs = strided_sum(threadIdx.x, nt, kThreads, [&](int64_t i) { return sc[1][i]; });
    double vr = strided_sum(threadIdx.x, nt, kThreads, [&](int64_t) { return 0.0; });
    ps = block_sum(ps, red);
    gs = block_sum(gs, red);
    vr = block_sum(vr, red);
    if (threadIdx.x == 0) {
      c.pay[k * 3 + 0] = T.weight * gs;
      c.pay[k * 3 + 2] = T.weight * vr;
      c.pay[k * 3 + 1] = T.weight * ps;
    }
    __syncthreads();
    k2_body(c, k, k + 1, lr, b2, use_clip, clip, ext_sumsq, red);
    __syncthreads();
    if (threadIdx.x < cs) {
      double* dst = cl.map_shared_rank(&bc[0], (int)threadIdx.x);
      dst[0] = c.glob[0];
      dst[1] = c.tens_sc[k * kTensScalars + TS_CORR];
    }
  }
  cl.sync();
  const double s = bc[0], corr = bc[1];
  // K4 (1-D branch): v_full EMA, per tile sum u^2 -> CTA 0
#pragma unroll
  for (int q = 0; q < kSmallPer; ++q) {
    const int ti = rank + q * cs;
    if (ti >= nt) break;
    double usq = 0.0;
    if (ev[q] >= 0) {
      const double gs = s * (double)gv[q];
      double v = vv[q];
      v = b2 * v + (1 - b2) * gs * gs;
      c.state[T.vfull_off + ev[q]] = v;
      vv[q] = v;
      const double u = gs / sqrt(v / corr + eps);
      usq += u * u;
    }
    const double bu = block_sum(usq, red);
    if (threadIdx.x == 0) sc0[2 * kSmallTiles + ti] = bu;
  }
  cl.sync();
  if (rank == 0) {  // usq_payload + K5
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      double us = strided_sum(lane, nt, 32, [&](int64_t i) { return sc[2][i]; });
      us = warp_sum(us);
      if (lane == 0) c.pay_usq[k] = T.weight * us;
    }
    __syncthreads();
    k5_body(c, k, k + 1, adalomo_clip);
    __syncthreads();
    if (threadIdx.x < cs)
      cl.map_shared_rank(&bc[0], (int)threadIdx.x)[2] = c.tens_sc[k * kTensScalars + TS_F];
  }
  cl.sync();
  const double f = bc[2];
  // K6 (1-D branch)
#pragma unroll
  for (int q = 0; q < kSmallPer; ++q) {
    if (ev[q] >= 0) {
      const double gs = s * (double)gv[q];
      const double u = gs / sqrt(vv[q] / corr + eps);
      stp1(p + ev[q], (float)((double)pv[q] - f * u));
    }
  }
}

// The small path applies to a 1-D tensor whose plan tiles all hold <= 256 elements and
// number <= kSmallTiles (vector_chunk gives 256-element tiles up to 2 * 256 * SMs).
bool small_vec_ok(const AdaLomoPlan& pl, int k) {
  const TensorInfo& T = pl.h_tensors[k];
  if (T.factored || T.numel == 0 || T.tile_end - T.tile_begin > kSmallTiles) return false;
  for (int64_t i = T.tile_begin; i < T.tile_end; ++i)
    if (pl.h_tiles[i].r1 - pl.h_tiles[i].r0 > 256) return false;
  return true;
}

template <typename K>
int grid_for(K kernel, int64_t ntiles, int device) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;  // kernel -> resident CTAs per SM
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find((const void*)kernel);
    if (it == cache.end()) {
      MCO_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0));
      per_sm = std::max(per_sm, 1);
      cache[(const void*)kernel] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  const int64_t full = (int64_t)device_info(device).sms * per_sm;
  // balanced rounds: every CTA takes the same number of items, so the last round is
  // not a partial wave at a fraction of the bandwidth (the per-tensor hook form:
  // 512 tiles of a 4096^2 matrix on 444 resident CTAs -> 256 CTAs x 2 tiles)
  const int64_t rounds = (std::max<int64_t>(ntiles, 1) + full - 1) / full;
  return (int)std::max<int64_t>(1, (ntiles + rounds - 1) / rounds);
}

// k6_tma: every tensor of the call starts 16 B aligned and spans a whole number of 16 B,
// for parameters and gradients (bulk copies move 16 B units).
bool k6_tma_ok(const AdaLomoPlan& pl, const AdaLomoCall& call, size_t gsz, size_t psz) {
  for (int k = call.t0; k < call.t1; ++k) {
    const TensorInfo& T = pl.h_tensors[k];
    const int64_t off = call.single || call.ntab ? 0 : T.elem_off;
    const uintptr_t pb = (uintptr_t)(call.ntab ? call.ptab[k - call.t0] : call.p) + off * psz;
    const uintptr_t gb = (uintptr_t)(call.ntab ? call.gtab[k - call.t0] : call.g) + off * gsz;
    if (pb % 16 || gb % 16 || (T.numel * psz) % 16 || (T.numel * gsz) % 16) return false;
  }
  return true;
}

// Launch state shared by one phase's kernels.
struct Launch {
  Ctx c;
  Ptrs P;
  int dev;
  int64_t tile0, ntiles, chunk0, nchunks, sms;
};

Launch make_launch(const AdaLomoPlan& pl, const AdaLomoCall& call) {
  Launch L{};
  L.c = Ctx{pl.d_tiles,   pl.d_tensors, pl.d_state, pl.d_colpart, pl.d_rowpart,
            pl.d_tile_sc, pl.d_tens_sc, pl.d_fa,    pl.d_fb,      pl.d_glob,
            pl.d_payload, pl.d_payload + pl.stats_len, (int64_t)pl.h_tensors.size(),
            pl.d_chunks,  pl.d_chunk_sc, pl.d_fra,    pl.d_frb,     pl.d_mins};
  L.P.p = call.p;
  L.P.g = call.g;
  L.P.single = call.single;
  L.P.ntab = call.ntab;
  L.P.t0 = call.t0;
  L.P.filt = 0;
  L.P.psz = call.p_dtype == MCO_BF16 ? 2 : 4;
  L.P.gsz = call.g_dtype == MCO_BF16 ? 2 : 4;
  for (int i = 0; i < call.ntab; ++i) {
    L.P.ptab[i] = call.ptab[i];
    L.P.gtab[i] = call.gtab[i];
  }
  L.dev = current_device();
  L.tile0 = pl.h_tensors[call.t0].tile_begin;
  L.ntiles = pl.h_tensors[call.t1 - 1].tile_end - L.tile0;
  L.chunk0 = pl.h_tensors[call.t0].chunk_begin;
  L.nchunks = pl.h_tensors[call.t1 - 1].chunk_end - L.chunk0;
  L.sms = device_info(L.dev).sms;
  return L;
}

// pass 1 over {g, p}
template <bool VEC, typename GT, typename PT>
void launch_k1(Launch L, const AdaLomoCall& call, int filt, cudaStream_t st) {
  L.P.filt = filt;
  const int mode = call.stats_mode ? call.stats_mode : kStatsAll;
  auto go1 = [&](auto kk1) {
    launch_pdl(kk1, grid_for(kk1, L.ntiles, L.dev), kThreads, st, L.c, L.P, L.tile0, L.ntiles,
               call.early);
  };
  if (mode == kStatsG)
    go1(k1_stats<VEC, GT, PT, kStatsG>);
  else if (mode == kStatsP)
    go1(k1_stats<VEC, GT, PT, kStatsP>);
  else
    go1(k1_stats<VEC, GT, PT, kStatsAll>);
  launch_check("adalomo k1_stats");
}

// pass 2 over {g}; fuse5: K4's last CTA reduces sum u^2 and computes the damping
template <bool VEC, typename GT, typename PT>
void launch_k4(Launch L, const AdaLomoPlan& pl, const AdaLomoCall& call, int filt, int fuse5,
               cudaStream_t st) {
  L.P.filt = filt;
  auto kk4 = k4_usq<VEC, GT>;
  launch_pdl(kk4, grid_for(kk4, L.ntiles, L.dev), kThreads, st, L.c, L.P, L.tile0, L.ntiles,
             pl.cfg.beta2, pl.cfg.eps, call.t0, call.t1, fuse5, pl.cfg.adalomo_clip);
  launch_check("adalomo k4_usq");
}

// pass 3 over {g, p -> p}
template <bool VEC, typename GT, typename PT>
void launch_k6(Launch L, const AdaLomoPlan& pl, const AdaLomoCall& call, int filt,
               cudaStream_t st) {
  L.P.filt = filt;
  // K6 traversal: tiles for multi-tensor calls (the per-thread b_j and a_i loads
  // amortise over a tile) and flat chunks for the one-tensor hook form (finer work items
  // for one tensor).  The cp.async.bulk pipeline (k6_tma, 16 B aligned / sized tensors
  // only) measured slower on every form (same box, 7B: multi-tensor 27.5 vs 25.1 ms,
  // bf16 18.8 vs 14.1, hook form 33.6 vs 31.2) and is opt-in.
  // MCO_ADALOMO_K6 = "tma" / "tiles" / "chunks" forces one (A/B knob).
  static const int k6_force = [] {
    const char* e = getenv("MCO_ADALOMO_K6");
    if (!e) return 0;
    const std::string v(e);
    return v == "tiles" ? 1 : v == "chunks" ? 2 : v == "tma" ? 3 : 0;
  }();
  const bool tma_ok = VEC && !filt && k6_tma_ok(pl, call, sizeof(GT), sizeof(PT));
  const int k6 = k6_force == 3 && tma_ok               ? 3
                 : k6_force == 1 || k6_force == 2      ? k6_force
                 : call.single && VEC                  ? 2  // scalar rows: strided tiles
                                                       : 1;
  const double eps = pl.cfg.eps;
  if (k6 == 3) {
    auto kk6 = k6_tma<GT, PT>;
    constexpr int smem = k6_smem<GT, PT>();
    static std::atomic<uint64_t> attr_set{0};  // per device: dynamic smem opt-in done
    if (!(attr_set.load() & (1ull << L.dev))) {
      MCO_CUDA_CHECK(cudaFuncSetAttribute(kk6, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr_set.fetch_or(1ull << L.dev);
    }
    const int64_t nitems = L.nchunks * kK6PPC;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(L.sms, nitems));
    launch_pdl_smem(kk6, grid, kK6Consumers + 32, smem, st, L.c, L.P, L.chunk0, L.nchunks, eps,
                    call.trigger);
  } else if (k6 == 1) {
    auto kk6 = k6_update_tiles<VEC, GT, PT>;
    launch_pdl(kk6, grid_for(kk6, L.ntiles, L.dev), kThreads, st, L.c, L.P, L.tile0, L.ntiles,
               eps, call.trigger);
  } else {
    auto kk6 = k6_update<VEC, GT, PT>;
    launch_pdl(kk6, grid_for(kk6, L.nchunks, L.dev), kThreads, st, L.c, L.P, L.chunk0,
               L.nchunks, eps, call.trigger);
  }
  launch_check("adalomo k6_update");
}

// f(vec_tag, gt_tag, pt_tag) for the call's dtype pair, VEC = vec
template <typename F>
void with_types(const AdaLomoCall& call, bool vec, F&& f) {
  using T = std::true_type;
  using N = std::false_type;
  // (params, grads): (f32, f32), (f32, bf16), (bf16, bf16)
  if (call.p_dtype == MCO_F32 && call.g_dtype == MCO_F32) {
    vec ? f(T{}, float{}, float{}) : f(N{}, float{}, float{});
  } else if (call.p_dtype == MCO_F32 && call.g_dtype == MCO_BF16) {
    vec ? f(T{}, uint16_t{}, float{}) : f(N{}, uint16_t{}, float{});
  } else if (call.p_dtype == MCO_BF16 && call.g_dtype == MCO_BF16) {
    vec ? f(T{}, uint16_t{}, uint16_t{}) : f(N{}, uint16_t{}, uint16_t{});
  } else {
    throw Error(MCO_CONTRACT, "adalomo: params / grads must be f32 / f32, f32 / bf16 or bf16 / bf16");
  }
}

}  // namespace

void launch_adalomo_phase(const AdaLomoPlan& pl, const AdaLomoCall& call, int phase,
                          cudaStream_t st) {
  if (call.t1 <= call.t0) return;
  // vector path, per tensor: a factored tensor needs C % 8 == 0 and rows aligned to 8
  // elements of their type (32 B f32, 16 B bf16) for both params and grads (skip_tensor
  // is the device-side twin).  A call whose tensors all agree runs one instance of each
  // pass; a mixed call (an odd-sized tensor shifts every later flat offset off the grid)
  // runs the vector instance over the aligned tensors and the scalar one over the rest,
  // instead of sending the whole call to the scalar path (a (7,) vector ahead of two 7B
  // layers: 6.3 vs 2.5 ms before this split).
  const size_t gsz = call.g_dtype == MCO_BF16 ? 2 : 4;
  const size_t psz = call.p_dtype == MCO_BF16 ? 2 : 4;
  bool any_vec = false, any_scalar = false;
  for (int k = call.t0; k < call.t1; ++k) {
    const TensorInfo& T = pl.h_tensors[k];
    if (!T.factored) continue;
    const int64_t off = call.single || call.ntab ? 0 : T.elem_off;
    const uintptr_t pb = (uintptr_t)(call.ntab ? call.ptab[k - call.t0] : call.p);
    const uintptr_t gb = (uintptr_t)(call.ntab ? call.gtab[k - call.t0] : call.g);
    const bool v = (T.cols % 8 == 0) && ((pb + off * psz) % (8 * psz) == 0) &&
                   ((gb + off * gsz) % (8 * gsz) == 0);
    (v ? any_vec : any_scalar) = true;
  }
  const bool mixed = any_vec && any_scalar;
  const bool vec = !any_scalar;  // uniform call: its one instance
  const Launch L = make_launch(pl, call);
  const auto& cfg = pl.cfg;
  // each tiled pass: one launch (uniform) or the vector + scalar pair (mixed)
  auto each = [&](auto&& pass) {
    if (!mixed) {
      with_types(call, vec, [&](auto V, auto g, auto p) { pass(V, g, p, 0); });
    } else {
      with_types(call, true, [&](auto V, auto g, auto p) { pass(V, g, p, 1); });
      with_types(call, false, [&](auto V, auto g, auto p) { pass(V, g, p, 2); });
    }
  };

  if (phase == 1) {  // pass 1 + reduction of the tile partials into the payload
    each([&](auto V, auto g, auto p, int filt) {
      launch_k1<decltype(V)::value, decltype(g), decltype(p)>(L, call, filt, st);
    });
    const int mode = call.stats_mode ? call.stats_mode : kStatsAll;
    const int64_t ncols = pl.h_col_off[call.t1] - pl.h_col_off[call.t0];
    const int ncolblk = (mode & kStatsG) ? (int)((ncols + 31) / 32) : 0;
    // fused calls (no all-reduce between the phases): KR's scalar block does K2's work
    launch_pdl(kr_stats, ncolblk + (call.t1 - call.t0), kThreads, st, L.c, call.t0, call.t1,
               (const int64_t*)pl.d_col_off, ncols, ncolblk, mode, call.fuse_usq, call.lr,
               cfg.beta2, call.use_clip, pl.grad_clip, call.ext_sumsq);
    launch_check("adalomo kr_stats");
  } else if (phase == 2) {  // scalars, moments, pass 2
    if (!call.fuse_usq) {
      launch_pdl(k2_scalars, 1, kThreads, st, L.c, call.t0, call.t1, call.lr, cfg.beta2,
                 call.use_clip, pl.grad_clip, call.ext_sumsq);
      launch_check("adalomo k2_scalars");
    }
    const int64_t nitems = pl.h_item_off[call.t1] - pl.h_item_off[call.t0];
    if (nitems > 0) {
      const int64_t blocks = std::min<int64_t>((nitems + kThreads - 1) / kThreads, L.sms * 8);
      launch_pdl(k3_moments, (unsigned)blocks, kThreads, st, L.c, call.t0, call.t1,
                 (const int64_t*)pl.d_item_off, pl.h_item_off[call.t0], nitems, cfg.beta2);
      launch_check("adalomo k3_moments");
    }
    // K4's last-CTA reduction counts one grid: a mixed call leaves it to K5 (with_usq)
    each([&](auto V, auto g, auto p, int filt) {
      launch_k4<decltype(V)::value, decltype(g), decltype(p)>(L, pl, call, filt,
                                                             call.fuse_usq && !mixed, st);
    });
    if (!call.fuse_usq) {
      launch_pdl(kr_usq, 1, 1024, st, L.c, call.t0, call.t1);
      launch_check("adalomo kr_usq");
    }
  } else {  // damping + pass 3
    if (!call.fuse_usq || mixed) {
      launch_pdl(k5_damp, 1, 1024, st, L.c, call.t0, call.t1, cfg.adalomo_clip,
                 call.fuse_usq && mixed ? 1 : 0);
      launch_check("adalomo k5_damp");
    }
    each([&](auto V, auto g, auto p, int filt) {
      launch_k6<decltype(V)::value, decltype(g), decltype(p)>(L, pl, call, filt, st);
    });
  }
}


void launch_adalomo_gsumsq(const AdaLomoPlan& pl, int t0, int t1, double* out, cudaStream_t st) {
  Ctx c{};
  c.pay = pl.d_payload;
  launch_pdl(kg_sumsq, 1, kThreads, st, c, t0, t1, out);
  launch_check("adalomo kg_sumsq");
}

void launch_adalomo(const AdaLomoPlan& pl, const AdaLomoCall& call, cudaStream_t st) {
  static const bool small_on = [] {  // MCO_ADALOMO_SMALL=0: the 4-launch chain (A/B knob)
    const char* e = getenv("MCO_ADALOMO_SMALL");
    return !(e && atoi(e) == 0);
  }();
  if (small_on && call.t1 == call.t0 + 1 && !call.stats_mode && small_vec_ok(pl, call.t0)) {
    Launch L = make_launch(pl, call);
    const auto& cfg = pl.cfg;
    const TensorInfo& T = pl.h_tensors[call.t0];
    const unsigned cs = (unsigned)std::min<int64_t>(kSmallCluster, T.tile_end - T.tile_begin);
    auto go = [&](auto kk) {
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(cs);
      lc.blockDim = dim3(kThreads);
      lc.stream = st;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = MCO_PDL;
      attr[1].id = cudaLaunchAttributeClusterDimension;
      attr[1].val.clusterDim.x = cs;
      attr[1].val.clusterDim.y = 1;
      attr[1].val.clusterDim.z = 1;
      lc.attrs = attr;
      lc.numAttrs = 2;
      cuda_check(cudaLaunchKernelEx(&lc, kk, L.c, L.P, call.t0, call.lr, cfg.beta2, cfg.eps,
                                    call.use_clip, pl.grad_clip, call.ext_sumsq,
                                    cfg.adalomo_clip, call.trigger),
                 "cudaLaunchKernelEx (k_small_vec)");
    };
    with_types(call, false, [&](auto, auto g, auto p) {
      go(k_small_vec<decltype(g), decltype(p)>);
    });
    launch_check("adalomo k_small_vec");
    return;
  }
  AdaLomoCall c = call;
  c.fuse_usq = 1;  // no all-reduce between the phases
  for (int phase = 1; phase <= 3; ++phase) launch_adalomo_phase(pl, c, phase, st);
}

}  // namespace mco

namespace mco {

// ---- host: tile plan ------------------------------------------------------------
// Magic for e / cols with e < 2^31 (round-up method): p = 31 + ceil(log2 d),
// m = ceil(2^p / d) < 2^32, e / d = (e * m) >> p for every e < 2^31.
void set_fast_div(TensorInfo& T) {
  const uint64_t d = (uint64_t)T.cols;
  if (d <= 1) {
    T.div_m = 0;
    T.div_s = 0;
    return;
  }
  int l = 0;
  while ((1ull << l) < d) ++l;
  const int p = 31 + l;
  const unsigned __int128 m = (((unsigned __int128)1 << p) + d - 1) / d;
  T.div_m = (uint32_t)m;
  T.div_s = p - 32;
}

// Per matrix R x C: column blocks of w = min(C, 1024) columns (TC lanes x 8),
// row blocks of h <= 128 rows; h is halved (down to 8) until one tensor alone
// yields >= 2 tiles per SM, so the per-tensor hook form also fills the GPU.
// Column partials cost ceil(R/h)*C floats per tensor (written once, read once).
// Element range per CTA for a 1-D (unfactored) tensor: its passes are fp64 element
// loops (v_full EMA, sqrt, divide), latency-bound per thread, so a norm vector of
// 4096 elements is spread over ~2 CTAs per SM (>= 256 elements each) instead of one
// 64 Ki chunk on one CTA (ncu: K4 16 us, K6 21 us for a single 4096-vector).
int64_t vector_chunk(int64_t numel, int sms) {
  int64_t c = (numel + 2LL * sms - 1) / (2LL * sms);
  c = (c + 255) / 256 * 256;
  return std::min<int64_t>(std::max<int64_t>(c, 256), 1 << 16);
}

void build_adalomo_plan(AdaLomoPlan& pl, const std::vector<std::vector<int64_t>>& shapes,
                        int sms) {
  pl.h_tensors.clear();
  pl.h_tiles.clear();
  pl.h_chunks.clear();
  pl.h_item_off.assign(1, 0);
  pl.h_col_off.assign(1, 0);
  int64_t elem = 0, state = 0, colpart = 0, rowpart = 0, fa = 0, fb = 0;
  const int64_t min_tiles = 2LL * sms;
  // tile heights: "waves" (default) or "pow2" (round 1: h halved from 128 until >= 2
  // tiles per SM); MCO_ADALOMO_TILES, an A/B knob read at plan build
  const char* tk = getenv("MCO_ADALOMO_TILES");
  const bool waves = !(tk && std::string(tk) == "pow2");
  const char* wk = getenv("MCO_ADALOMO_WAVE");  // tile-kernel CTAs per SM of a wave (A/B)
  const int wave_ctas = wk ? std::max(1, atoi(wk)) : 3;
  for (size_t k = 0; k < shapes.size(); ++k) {
    const auto& s = shapes[k];
    TensorInfo T{};
    int64_t numel = 1;
    for (int64_t d : s) numel *= d;
    T.numel = numel;
    T.elem_off = elem;
    T.factored = s.size() == 2 ? 1 : 0;
    T.tile_begin = (int64_t)pl.h_tiles.size();
    if (T.factored) {
      T.rows = s[0];
      T.cols = s[1];
      if (numel >= (1LL << 31))
        throw Error(MCO_CONTRACT, "AdaLomoState: a factored tensor must have < 2^31 elements");
      set_fast_div(T);
      const int64_t w = std::min<int64_t>(T.cols, 128 * kCW);
      const int64_t chunks = (w + kCW - 1) / kCW;
      int tc = 32;
      while (tc < chunks) tc <<= 1;
      T.tc = tc;
      T.kc = (int32_t)((T.cols + w - 1) / w);
      int64_t h = kMaxTileRows;
      if (waves) {
        // whole waves: the tensor's tile count is the smallest multiple m of the resident
        // tile-kernel CTAs (3 per SM) that keeps h <= 128, so a one-tensor call (hook
        // form) runs every pass in m full rounds -- 4096^2: 444 tiles of 37 rows (one round
        // of 444 CTAs) instead of 512 tiles of 32 rows (two rounds of 256 CTAs, 1.7 per SM:
        // K1 36.7 us against a 20.5 us traffic floor, ncu)
        const int64_t wave = (int64_t)wave_ctas * sms;
        const int64_t need = ((T.rows + kMaxTileRows - 1) / kMaxTileRows) * T.kc;
        const int64_t m = std::max<int64_t>(1, (need + wave - 1) / wave);
        const int64_t nrb_max = std::max<int64_t>(1, (m * wave) / T.kc);
        h = std::max<int64_t>((T.rows + nrb_max - 1) / nrb_max, 8);
        h = std::min<int64_t>(h, kMaxTileRows);
      } else {
        while (h > 8 && ((T.rows + h - 1) / h) * T.kc < min_tiles) h >>= 1;
      }
      h = std::min<int64_t>(h, std::max<int64_t>(T.rows, 1));
      T.nrb = (T.rows + h - 1) / h;
      T.vrow_off = state;
      state += T.rows;
      T.vcol_off = state;
      state += T.cols;
      T.vfull_off = -1;
      T.colpart_off = colpart;
      colpart += T.nrb * T.cols;
      T.rowpart_off = rowpart;
      rowpart += (int64_t)T.kc * T.rows;
      T.fa_off = fa;
      fa += T.rows;
      T.fb_off = fb;
      fb += (T.cols + 7) / 8 * 8;  // 32 B aligned per tensor (float4 loads in K4 / K6)
      for (int64_t rb = 0; rb < T.nrb; ++rb)
        for (int cb = 0; cb < T.kc; ++cb) {
          Tile tl{};
          tl.tensor = (int32_t)k;
          tl.cb = cb;
          tl.rb = rb;
          tl.r0 = rb * h;
          tl.r1 = std::min(T.rows, (rb + 1) * h);
          tl.c0 = (int64_t)cb * w;
          tl.c1 = std::min(T.cols, ((int64_t)cb + 1) * w);
          pl.h_tiles.push_back(tl);
        }
      pl.h_item_off.push_back(pl.h_item_off.back() + T.rows + T.cols);
      pl.h_col_off.push_back(pl.h_col_off.back() + T.cols);
    } else {
      T.rows = numel;
      T.cols = 1;
      T.tc = 32;
      T.kc = 1;
      T.nrb = 0;
      T.vrow_off = T.vcol_off = -1;
      T.vfull_off = state;
      state += numel;
      T.colpart_off = T.rowpart_off = T.fa_off = T.fb_off = -1;
      const int64_t chunk = vector_chunk(numel, sms);
      for (int64_t e0 = 0; e0 < numel || (numel == 0 && e0 == 0); e0 += chunk) {
        Tile tl{};
        tl.tensor = (int32_t)k;
        tl.r0 = e0;
        tl.r1 = std::min(numel, e0 + chunk);
        pl.h_tiles.push_back(tl);
        if (numel == 0) break;
      }
      pl.h_item_off.push_back(pl.h_item_off.back());
      pl.h_col_off.push_back(pl.h_col_off.back());
    }
    T.tile_end = (int64_t)pl.h_tiles.size();
    T.chunk_begin = (int64_t)pl.h_chunks.size();
    const int64_t chunk = T.factored ? kChunkElems : vector_chunk(numel, sms);
    for (int64_t e0 = 0; e0 < numel; e0 += chunk)
      pl.h_chunks.push_back(Chunk{(int32_t)k, 0, e0, std::min(numel, e0 + chunk)});
    T.chunk_end = (int64_t)pl.h_chunks.size();
    T.t = 0;
    T.rows_global = T.rows;
    T.numel_global = T.numel;
    T.weight = 1.0;
    elem += numel;
    pl.h_tensors.push_back(T);
  }
  pl.state_len = state;
  pl.colpart_len = colpart;
  pl.rowpart_len = rowpart;
  pl.fa_len = fa;
  pl.fb_len = fb;
  pl.stats_len = 3 * (int64_t)pl.h_tensors.size() + fb;
  pl.usq_len = (int64_t)pl.h_tensors.size();
}

}  // namespace mco
