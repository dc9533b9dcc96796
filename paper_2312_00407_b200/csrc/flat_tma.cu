// TMA-staged variant of the fused elementwise optimizer step (AdamW / Lion /
// Adan / Sophia, fp32).  Same arithmetic (update.cuh) and therefore the same bits
// as flat_step_kernel; only the data movement differs:
//
//   producer warp (one elected lane)          consumer warps (512 threads)
//   cp.async.bulk global->smem, per stream  ->  wait full[s]; 4 elements / thread:
//   (mbarrier complete_tx)                      ld.shared, update, st.shared,
//                                               fence.proxy.async; arrive done[s]
//   wait done[s]; cp.async.bulk smem->global
//   for every written stream; then refill the
//   PREVIOUS tile's stage (its store has had a
//   tile-time to read smem) with tile
//   i - 1 + STAGES
//
// One CTA per SM; STAGES-1 tiles of every input stream are in flight per SM
// (Adan: 3 x 48 KB) independent of register pressure, which is what limits the
// LDG version of the 11-stream Adan kernel to 3 CTAs/SM.
#include <algorithm>
#include <atomic>
#include <type_traits>

#include "flat_tma.h"
#include "tma.cuh"
#include "update.cuh"

namespace mco {
namespace {

using namespace upd;
// Configuration: CW consumer warps (each thread updates one float4 per stream per
// stage, so a tile is CW*128 elements) and NS pipeline stages (capped by shared
// memory).  Default 16 warps (4 per scheduler: at 8 warps ncu showed the consumers'
// fp32 div / sqrt chains stalled on 'wait' + 'branch_resolving') and 4 stages
// (measured: fewer starve the loads, more lose bandwidth for AdamW / Sophia).
// EPT: elements per consumer thread per stream and stage (4: float4, 2: float2);
// HINT: bulk copies carry an L2 evict-first cache policy (streams are touched once).
// DS: direct stores -- the consumers copy a stage into registers, release it at once
// and write their results straight to global memory (coalesced 16 B stores) instead of
// staging them back through shared memory for the producer's bulk stores: a stage is
// busy only while it loads, so more of the pipeline's bytes are loads in flight.
template <int CW_, int NS_, int EPT_ = 4, bool HINT_ = false, bool DS_ = false>
struct TmaCfg {
  static constexpr int CW = CW_;
  static constexpr int kConsumers = CW * 32;
  static constexpr int kEPT = EPT_;
  static constexpr int kTile = CW * 32 * EPT_;  // elements per stream per stage
  static constexpr int kStages = NS_;
  static constexpr bool kHint = HINT_;
  static constexpr bool kDS = DS_;
};
constexpr int kSmemMax = 220 * 1024;

template <int KIND>
constexpr int n_in() {  // p, g, s0 [, s1 [, s2, s3]]
  return KIND == K_ADAN ? 6 : (KIND == K_LION ? 3 : 4);
}
// A stream slot holds one tile plus 16 B: a gradient at a different 16 B phase than the
// other streams is copied from its aligned-down address (flat_tma_kernel, gsh).
template <class C>
constexpr int slot_floats() {
  return C::kTile + 4;
}
template <class C, int KIND, bool MIXED>
constexpr int stage_bytes() {
  return n_in<KIND>() * slot_floats<C>() * 4 + (MIXED ? C::kTile * 2 : 0);
}
template <class C, int KIND, bool MIXED>
constexpr int stages() {
  constexpr int cap = kSmemMax / stage_bytes<C, KIND, MIXED>();
  return C::kStages < cap ? C::kStages : cap;
}
template <class C, int KIND, bool MIXED>
constexpr int smem_bytes() {
  return stages<C, KIND, MIXED>() * stage_bytes<C, KIND, MIXED>() + 2 * stages<C, KIND, MIXED>() * 8;
}

// consecutive threads read consecutive 16 B (8 B): conflict-free LDS.128 / LDS.64
template <int E>
__device__ __forceinline__ void lds(const float* s, float (&r)[E]) {
  if constexpr (E == 4) {
    const float4 x = *reinterpret_cast<const float4*>(s);
    r[0] = x.x, r[1] = x.y, r[2] = x.z, r[3] = x.w;
  } else {
    const float2 x = *reinterpret_cast<const float2*>(s);
    r[0] = x.x, r[1] = x.y;
  }
}
template <int E>
__device__ __forceinline__ void sts(float* s, const float (&r)[E]) {
  if constexpr (E == 4)
    *reinterpret_cast<float4*>(s) = make_float4(r[0], r[1], r[2], r[3]);
  else
    *reinterpret_cast<float2*>(s) = make_float2(r[0], r[1]);
}

// Gradient tile of a stage (stream slot 1), fp32 or bf16 (bf16 fills half the slot).
template <int E>
__device__ __forceinline__ void lds_grad(const float* slot, int c0, float (&r)[E]) {
  lds<E>(slot + c0, r);
}
template <int E>
__device__ __forceinline__ void lds_grad_bf16(const float* slot, int c0, float (&r)[E]) {
  const uint16_t* h = reinterpret_cast<const uint16_t*>(slot) + c0;
  if constexpr (E == 4) {
    const uint2 w = *reinterpret_cast<const uint2*>(h);
    r[0] = __uint_as_float(w.x << 16), r[1] = __uint_as_float(w.x & 0xffff0000u);
    r[2] = __uint_as_float(w.y << 16), r[3] = __uint_as_float(w.y & 0xffff0000u);
  } else {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(h);
    r[0] = __uint_as_float(w << 16), r[1] = __uint_as_float(w & 0xffff0000u);
  }
}

template <class C, int KIND, bool MIXED, typename GT, bool DEV = false>
__global__ void __launch_bounds__(C::kConsumers + 32, 1)
    flat_tma_kernel(float* p, const GT* g, float* s0, float* s1, float* s2, float* s3,
                    uint16_t* pout, uint64_t ntiles, uint64_t n, const StepConsts<float> kv,
                    const GraphStep gs, int gsh) {
  // gsh: the gradient's element phase within 16 B when it differs from every other
  // stream's (those are 16 B aligned): its tiles are copied from the aligned-down address
  // (one 16 B granule more) and read gsh elements into the slot -- same bits, no scalar
  // fallback for a gradient view at another offset than the parameters
  const StepConsts<float> k = step_consts<DEV>(kv, gs);  // DEV: graph mode (common.cuh)
  constexpr int NIN = n_in<KIND>();
  constexpr int NS = stages<C, KIND, MIXED>();
  constexpr int kTile = C::kTile, kConsumers = C::kConsumers, kConsumerWarps = C::CW;
  constexpr int kSlot = slot_floats<C>();
  extern __shared__ __align__(128) uint8_t smem[];
  float* buf = reinterpret_cast<float*>(smem);  // [NS][NIN][kSlot]
  uint16_t* obuf = reinterpret_cast<uint16_t*>(buf + NS * NIN * kSlot);  // [NS][kTile]
  uint64_t* full = reinterpret_cast<uint64_t*>(obuf + (MIXED ? NS * kTile : 0));
  uint64_t* done = full + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // stream j of a stage: 0 p, 1 g, 2 s0, 3 s1, 4 s2, 5 s3 (slot of kTile floats each;
  // a bf16 gradient tile uses the first half of its slot)
  const float* src[6] = {p, nullptr, s0, s1, s2, s3};
  const uint64_t mine =
      ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (warp == kConsumerWarps) {  // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = C::kHint ? evict_first_policy() : 0;
      const bool skip_gp = (KIND == K_ADAN) && k.first;  // g_prev unused at t == 1
      const int nload = skip_gp ? NIN - 1 : NIN;
      const uint32_t gbytes = kTile * sizeof(GT) + (gsh ? 16u : 0u);
      auto issue = [&](uint64_t i) {
        const int s = (int)(i % NS);
        const uint64_t e = (blockIdx.x + i * gridDim.x) * (uint64_t)kTile;
        mbar_expect_tx(&full[s], (uint32_t)((nload - 1) * kTile * 4) + gbytes);
        for (int j = 0; j < nload; ++j) {
          float* dst = buf + ((size_t)s * NIN + j) * kSlot;
          if (j == 1)
            bulk_g2s<C::kHint>(dst, g + e - gsh, gbytes, &full[s], pol);
          else
            bulk_g2s<C::kHint>(dst, src[j] + e, kTile * 4, &full[s], pol);
        }
      };
      for (uint64_t i = 0; i < mine && i < (uint64_t)NS; ++i) issue(i);
      if constexpr (C::kDS) {  // consumers store directly: refill each stage once released
        for (uint64_t i = 0; i + NS < mine; ++i) {
          mbar_wait(&done[(int)(i % NS)], (uint32_t)((i / NS) & 1));
          issue(i + NS);
        }
        return;
      }
      for (uint64_t i = 0; i < mine; ++i) {
        const int s = (int)(i % NS);
        mbar_wait(&done[s], (uint32_t)((i / NS) & 1));
        const uint64_t e = (blockIdx.x + i * gridDim.x) * (uint64_t)kTile;
        float* st = buf + (size_t)s * NIN * kSlot;
        bulk_s2g<C::kHint>(p + e, st, kTile * 4, pol);
        bulk_s2g<C::kHint>(s0 + e, st + 2 * kSlot, kTile * 4, pol);
        if constexpr (KIND == K_ADAMW || KIND == K_ADAN) bulk_s2g<C::kHint>(s1 + e, st + 3 * kSlot, kTile * 4, pol);
        if constexpr (KIND == K_SOPHIA) {
          if (k.refresh) bulk_s2g<C::kHint>(s1 + e, st + 3 * kSlot, kTile * 4, pol);
        }
        if constexpr (KIND == K_ADAN) {
          bulk_s2g<C::kHint>(s2 + e, st + 4 * kSlot, kTile * 4, pol);
          bulk_s2g<C::kHint>(s3 + e, st + 5 * kSlot, kTile * 4, pol);
        }
        if constexpr (MIXED) bulk_s2g<C::kHint>(pout + e, obuf + (size_t)s * kTile, kTile * 2, pol);
        bulk_commit();
        // refill the PREVIOUS tile's stage: its store group (all but the one just
        // committed) has had a tile-time to drain out of smem, so the wait is short and
        // the producer never stalls on the store it has just issued
        if (i >= 1 && i - 1 + NS < mine) {
          bulk_wait_read_1();
          issue(i - 1 + NS);
        }
      }
      bulk_wait_all();
    }
  } else {  // ---------------- consumers ----------------
    constexpr int E = C::kEPT;
    const int c0 = threadIdx.x * E;
    for (uint64_t i = 0; i < mine; ++i) {
      const int s = (int)(i % NS);
      mbar_wait(&full[s], (uint32_t)((i / NS) & 1));
      float* st = buf + (size_t)s * NIN * kSlot + c0;
      float pv[E], gv[E], a[E], b[E], c[E], d[E];
      lds<E>(st, pv);
      if (gsh == 0) {
        if constexpr (sizeof(GT) == 4)
          lds<E>(st + kSlot, gv);
        else
          lds_grad_bf16<E>(buf + (size_t)s * NIN * kSlot + kSlot, c0, gv);
      } else {  // shifted gradient tile: element-wise reads
        const GT* gslot = reinterpret_cast<const GT*>(buf + (size_t)s * NIN * kSlot + kSlot) + gsh + c0;
#pragma unroll
        for (int j = 0; j < E; ++j) gv[j] = load_grad1(gslot + j);
      }
      lds<E>(st + 2 * kSlot, a);
      if constexpr (KIND != K_LION) lds<E>(st + 3 * kSlot, b);
      if constexpr (KIND == K_ADAN) {
        lds<E>(st + 4 * kSlot, c);
        if (!k.first) lds<E>(st + 5 * kSlot, d);
      }
      if constexpr (C::kDS) mbar_arrive(&done[s]);  // the stage is in registers: release it
#pragma unroll
      for (int j = 0; j < E; ++j) {
        if constexpr (KIND == K_LION) b[j] = 0.f;
        if constexpr (KIND != K_ADAN) c[j] = d[j] = 0.f;
        if constexpr (KIND == K_ADAN) {
          if (k.first) d[j] = 0.f;
        }
        update<KIND, float>(pv[j], gv[j], a[j], b[j], c[j], d[j], k);
      }
      if constexpr (C::kDS) {
        const uint64_t e = (blockIdx.x + i * gridDim.x) * (uint64_t)kTile + c0;
        st_stream(p + e, pv);
        st_stream(s0 + e, a);
        if constexpr (KIND == K_ADAMW || KIND == K_ADAN) st_stream(s1 + e, b);
        if constexpr (KIND == K_SOPHIA) {
          if (k.refresh) st_stream(s1 + e, b);
        }
        if constexpr (KIND == K_ADAN) {
          st_stream(s2 + e, c);
          st_stream(s3 + e, d);
        }
        if constexpr (MIXED) {
          uint32_t w[E / 2];
#pragma unroll
          for (int j = 0; j < E / 2; ++j) w[j] = f2bf2_bits(pv[2 * j], pv[2 * j + 1]);
          if constexpr (E == 4)
            *reinterpret_cast<uint2*>(pout + e) = make_uint2(w[0], w[1]);
          else
            *reinterpret_cast<uint32_t*>(pout + e) = w[0];
        }
        continue;
      }
      sts<E>(st, pv);
      sts<E>(st + 2 * kSlot, a);
      if constexpr (KIND != K_LION) sts<E>(st + 3 * kSlot, b);
      if constexpr (KIND == K_ADAN) {
        sts<E>(st + 4 * kSlot, c);
        sts<E>(st + 5 * kSlot, d);
      }
      if constexpr (MIXED) {
        uint32_t* o = reinterpret_cast<uint32_t*>(obuf + (size_t)s * kTile + c0);
#pragma unroll
        for (int j = 0; j < E / 2; ++j) o[j] = f2bf2_bits(pv[2 * j], pv[2 * j + 1]);
      }
      fence_proxy_async();  // generic-proxy smem writes -> visible to the bulk store
      mbar_arrive(&done[s]);
    }
    // tail (< one tile): plain loads / stores by the consumer threads of CTA 0
    if (blockIdx.x == 0) {
      for (uint64_t e = ntiles * kTile + threadIdx.x; e < n; e += kConsumers) {
        float pp = p[e], gg = load_grad1(g + e), aa = s0[e], bb = 0.f, cc = 0.f, dd = 0.f;
        if constexpr (KIND != K_LION) bb = s1[e];
        if constexpr (KIND == K_ADAN) {
          cc = s2[e];
          if (!k.first) dd = s3[e];
        }
        update<KIND, float>(pp, gg, aa, bb, cc, dd, k);
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
        if constexpr (MIXED) pout[e] = (uint16_t)f2bf_bits(pp);
      }
    }
    graph_bump<DEV>(gs);  // thread 0 is a consumer
  }
}

// ---- LOMO on the same pipeline -----------------------------------------------------
// p -= f * g (optim.cpp:185-190): two input streams of one element type (fp32, or bf16
// parameters with bf16 gradients -- fp32 arithmetic, RNE store, as lomo_kernel), p
// stored back.  Each consumer thread moves 16 B per stream per stage.
constexpr int kLomoWarps = 16;
constexpr int kLomoConsumers = kLomoWarps * 32;

template <typename ET>
constexpr int lomo_tile() {
  return kLomoConsumers * (16 / (int)sizeof(ET));
}

template <typename ET, int NS>
__global__ void __launch_bounds__(kLomoConsumers + 32, 1)
    lomo_tma_kernel(ET* p, const ET* g, uint64_t ntiles, uint64_t n, double lr, double scale,
                    const double* sumsq, double clip, int gsh) {
  // gsh: the gradient's element phase within 16 B when it differs from the parameters'
  // (flat_tma_kernel): copied from the aligned-down address, read shifted
  constexpr int EPT = 16 / (int)sizeof(ET);
  constexpr int kTile = lomo_tile<ET>();
  constexpr int kStage = 2 * kTile + EPT;  // p tile | g tile + 16 B
  constexpr uint32_t kBytes = kTile * sizeof(ET);
  extern __shared__ __align__(128) uint8_t smem[];
  ET* buf = reinterpret_cast<ET*>(smem);  // [NS][kStage]
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + NS * kStage);
  uint64_t* done = full + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], kLomoConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // the clip's sum of squares comes from the previous kernel
  const uint64_t mine =
      ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (warp == kLomoWarps) {  // ---------------- producer ----------------
    if (lane == 0) {
      const uint32_t gbytes = kBytes + (gsh ? 16u : 0u);
      auto issue = [&](uint64_t i) {
        const int s = (int)(i % NS);
        const uint64_t e = (blockIdx.x + i * gridDim.x) * (uint64_t)kTile;
        mbar_expect_tx(&full[s], kBytes + gbytes);
        bulk_g2s<false>(buf + (size_t)s * kStage, p + e, kBytes, &full[s], 0);
        bulk_g2s<false>(buf + (size_t)s * kStage + kTile, g + e - gsh, gbytes, &full[s], 0);
      };
      for (uint64_t i = 0; i < mine && i < (uint64_t)NS; ++i) issue(i);
      for (uint64_t i = 0; i < mine; ++i) {
        const int s = (int)(i % NS);
        mbar_wait(&done[s], (uint32_t)((i / NS) & 1));
        const uint64_t e = (blockIdx.x + i * gridDim.x) * (uint64_t)kTile;
        bulk_s2g<false>(p + e, buf + (size_t)s * kStage, kBytes, 0);
        bulk_commit();
        if (i >= 1 && i - 1 + NS < mine) {  // refill the previous tile's stage
          bulk_wait_read_1();
          issue(i - 1 + NS);
        }
      }
      bulk_wait_all();
    }
  } else {  // ---------------- consumers ----------------
    const float f = lomo_factor<float>(lr, scale, sumsq, clip);
    const int c0 = threadIdx.x * EPT;
    for (uint64_t i = 0; i < mine; ++i) {
      const int s = (int)(i % NS);
      mbar_wait(&full[s], (uint32_t)((i / NS) & 1));
      ET* sp = buf + (size_t)s * kStage + c0;
      const ET* sg = sp + kTile;
      if constexpr (sizeof(ET) == 4) {
        float4 pv = *reinterpret_cast<const float4*>(sp);
        float4 gv;
        if (gsh == 0)
          gv = *reinterpret_cast<const float4*>(sg);
        else
          gv = make_float4(sg[gsh], sg[gsh + 1], sg[gsh + 2], sg[gsh + 3]);
        pv.x = pv.x - f * gv.x;
        pv.y = pv.y - f * gv.y;
        pv.z = pv.z - f * gv.z;
        pv.w = pv.w - f * gv.w;
        *reinterpret_cast<float4*>(sp) = pv;
      } else {
        uint4 pw = *reinterpret_cast<const uint4*>(sp);
        uint4 gw;
        if (gsh == 0) {
          gw = *reinterpret_cast<const uint4*>(sg);
        } else {
          const uint16_t* h = reinterpret_cast<const uint16_t*>(sg) + gsh;
          gw.x = (uint32_t)h[0] | ((uint32_t)h[1] << 16);
          gw.y = (uint32_t)h[2] | ((uint32_t)h[3] << 16);
          gw.z = (uint32_t)h[4] | ((uint32_t)h[5] << 16);
          gw.w = (uint32_t)h[6] | ((uint32_t)h[7] << 16);
        }
        uint32_t* pa = &pw.x;
        const uint32_t* ga = &gw.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float lo = __uint_as_float(pa[k] << 16) - f * __uint_as_float(ga[k] << 16);
          const float hi = __uint_as_float(pa[k] & 0xffff0000u) -
                           f * __uint_as_float(ga[k] & 0xffff0000u);
          pa[k] = f2bf2_bits(lo, hi);
        }
        *reinterpret_cast<uint4*>(sp) = pw;
      }
      fence_proxy_async();
      mbar_arrive(&done[s]);
    }
    if (blockIdx.x == 0) {  // tail (< one tile)
      for (uint64_t e = ntiles * kTile + threadIdx.x; e < n; e += kLomoConsumers) {
        if constexpr (sizeof(ET) == 4)
          p[e] = p[e] - f * g[e];
        else
          p[e] = (ET)f2bf_bits(bf2f(p[e]) - f * bf2f(g[e]));
      }
    }
  }
}

template <typename ET, int NS>
void run_lomo_tma(void* p, const void* g, uint64_t n, double lr, double scale,
                  const double* sumsq, double clip, cudaStream_t st) {
  auto kern = lomo_tma_kernel<ET, NS>;
  constexpr int smem = NS * (2 * lomo_tile<ET>() * (int)sizeof(ET) + 16) + 2 * NS * 8;
  const int dev = current_device();
  static std::atomic<uint64_t> attr_set{0};
  if (!(attr_set.load() & (1ull << dev))) {
    MCO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set.fetch_or(1ull << dev);
  }
  const int gsh = (int)(((uintptr_t)g % 16) / sizeof(ET));
  uint64_t ntiles = n / lomo_tile<ET>();
  // a shifted gradient's copies reach 16 - gsh * sizeof(ET) bytes past the tile
  if (gsh && ntiles && (n - ntiles * lomo_tile<ET>()) * sizeof(ET) < 16 - gsh * sizeof(ET))
    --ntiles;
  const int grid = (int)std::max<uint64_t>(
      1, std::min<uint64_t>(ntiles ? ntiles : 1, (uint64_t)device_info(dev).sms));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kLomoConsumers + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = MCO_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MCO_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, (ET*)p, (const ET*)g, ntiles, n, lr, scale,
                                    sumsq, clip, gsh));
  launch_check("lomo_tma_kernel");
}

template <class C, int KIND, bool MIXED, typename GT, bool DEV>
void run_kern(const FlatArgs& a, const StepConsts<float>& k, cudaStream_t st) {
  auto kern = flat_tma_kernel<C, KIND, MIXED, GT, DEV>;
  constexpr int smem = smem_bytes<C, KIND, MIXED>();
  const int dev = current_device();
  static std::atomic<uint64_t> attr_set{0};  // per device: dynamic smem opt-in done
  if (!(attr_set.load() & (1ull << dev))) {
    MCO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set.fetch_or(1ull << dev);
  }
  const int gsh = (int)(((uintptr_t)a.g % 16) / sizeof(GT));
  uint64_t ntiles = a.n / C::kTile;
  // a shifted gradient's copies reach 16 - gsh * sizeof(GT) bytes past the tile: the last
  // tile needs that many valid bytes after it, else it joins the scalar tail
  if (gsh && ntiles && (a.n - ntiles * C::kTile) * sizeof(GT) < 16 - gsh * sizeof(GT)) --ntiles;
  const int grid = (int)std::max<uint64_t>(
      1, std::min<uint64_t>(ntiles ? ntiles : 1, (uint64_t)device_info(dev).sms));
  kern<<<grid, C::kConsumers + 32, smem, st>>>((float*)a.p, (const GT*)a.g, (float*)a.s[0],
                                               (float*)a.s[1], (float*)a.s[2], (float*)a.s[3],
                                               a.p_out_bf16, ntiles, a.n, k, a.gs, gsh);
  launch_check("flat_tma_kernel");
}

// graph mode (a.dk set) is instantiated for the default configurations only (4 stages;
// Adan's 3)
template <class C, int KIND, bool MIXED, typename GT>
void run(const FlatArgs& a, const StepConsts<float>& k, cudaStream_t st) {
  if constexpr (std::is_same_v<C, TmaCfg<16, 4>> ||
                (KIND == K_ADAN && std::is_same_v<C, TmaCfg<16, 3>>)) {
    if (a.gs.d) return run_kern<C, KIND, MIXED, GT, true>(a, k, st);
  }
  if (a.gs.d) throw Error(MCO_CONFIG, "flat_tma: graph mode runs the default configuration");
  run_kern<C, KIND, MIXED, GT, false>(a, k, st);
}

template <class C, int KIND>
void dispatch(const FlatArgs& a, const StepConsts<float>& k, cudaStream_t st) {
  if (a.g_dtype == MCO_BF16) {
    if (a.p_out_bf16)
      run<C, KIND, true, uint16_t>(a, k, st);
    else
      run<C, KIND, false, uint16_t>(a, k, st);
  } else {
    if (a.p_out_bf16)
      run<C, KIND, true, float>(a, k, st);
    else
      run<C, KIND, false, float>(a, k, st);
  }
}

template <class C>
void launch_cfg(const FlatArgs& a, const StepConsts<float>& k, cudaStream_t st) {
  switch (a.kind) {
    case MCO_ADAMW: dispatch<C, K_ADAMW>(a, k, st); break;
    case MCO_LION: dispatch<C, K_LION>(a, k, st); break;
    case MCO_ADAN: dispatch<C, K_ADAN>(a, k, st); break;
    case MCO_SOPHIA: dispatch<C, K_SOPHIA>(a, k, st); break;
    default: throw Error(MCO_CONTRACT, "flat_tma: unsupported kind");
  }
}

// ---- list form on the pipeline (mco_flat_step_list, kernels.h FlatList) -------------
// FlatList.vbeg holds tile prefix sums here: tile t belongs to tensor list_find(t) and
// starts at element (t - vbeg[i]) * kTile of it; the producer resolves every tile's
// addresses (p_i, g_i, state + soff_i), the consumers run exactly the flat kernel's
// update.  Scalar elements (tensor tails) are spread over the consumer threads of every
// CTA afterwards.
//
// Streams off the 16 B grid (round 2): a tensor's parameters, gradients and state may
// each sit at their own element phase within 16 B -- separate parameter allocations
// against a state at the running sum of the preceding lengths, which an odd-sized tensor
// shifts.  Such a stream's tile is copied from its aligned-down address, one 16 B
// granule longer, into a slot 16 B larger, and read / written `sh` elements in.  Its
// write-back is a bulk store of the tile's 16 B-aligned interior plus element stores of
// the partial granules at both ends by the consumer threads that hold them (thread 0 the
// first 4 - sh elements, the last thread the last sh): every element is written by
// exactly one tile, and the granule a tile shares with its neighbour is only read by the
// neighbour, never written from its stale copy.
struct ListStage {  // per stage, written by the producer before the stage is armed
  float* p;          // this tile's first parameter
  uint64_t so;       // its state offset
  int shp, shg, shs;  // stream phases (elements within 16 B)
};

template <int E>
__device__ __forceinline__ void lds_sh(const float* s, int sh, float (&r)[E]) {
  if (sh == 0) {
    lds<E>(s, r);
  } else {
#pragma unroll
    for (int j = 0; j < E; ++j) r[j] = s[sh + j];
  }
}
template <int E>
__device__ __forceinline__ void sts_sh(float* s, int sh, const float (&r)[E]) {
  if (sh == 0) {
    sts<E>(s, r);
  } else {
#pragma unroll
    for (int j = 0; j < E; ++j) s[sh + j] = r[j];
  }
}
// the partial 16 B granules of a shifted written stream: global element c0 + j of the
// tile goes out directly when it lies before the first / after the last aligned granule
template <int E, int kTile>
__device__ __forceinline__ void edge_st(float* dst, int c0, int sh, const float (&r)[E]) {
  if (sh == 0) return;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int cidx = c0 + j;
    if (cidx < 4 - sh || cidx >= kTile - sh) dst[cidx] = r[j];
  }
}

// SH: the launch has shifted streams (an instantiation apart, so that aligned lists keep
// the unshifted kernel: the runtime phase checks cost 6 % on 24 aligned 4096^2 tensors)
template <class C, int KIND, typename GT, bool DEV, bool SH>
__global__ void __launch_bounds__(C::kConsumers + 32, 1)
    list_tma_kernel(const __grid_constant__ FlatList L, float* s0, float* s1, float* s2,
                    float* s3, const StepConsts<float> kv, const GraphStep gs) {
  const StepConsts<float> k = step_consts<DEV>(kv, gs);
  constexpr int NIN = n_in<KIND>();
  constexpr int NS = stages<C, KIND, false>();
  constexpr int kTile = C::kTile, kConsumers = C::kConsumers, kConsumerWarps = C::CW;
  constexpr int kSlot = slot_floats<C>();
  static_assert(C::kEPT == 4, "edge stores assume 4 elements per consumer thread");
  extern __shared__ __align__(128) uint8_t smem[];
  float* buf = reinterpret_cast<float*>(smem);  // [NS][NIN][kSlot]
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + NS * NIN * kSlot);
  uint64_t* done = full + NS;
  __shared__ uint64_t tb[kListMax + 1], eb[kListMax + 1];
  __shared__ ListStage meta[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i <= L.n; i += blockDim.x) tb[i] = L.vbeg[i], eb[i] = L.ebeg[i];
  __syncthreads();
  const uint64_t ntiles = tb[L.n];
  const uint64_t mine =
      ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (warp == kConsumerWarps) {  // ---------------- producer ----------------
    if (lane == 0) {
      const bool skip_gp = (KIND == K_ADAN) && k.first;  // g_prev unused at t == 1
      const int nload = skip_gp ? NIN - 1 : NIN;
      // tensor cursors of the load and store sequences: a CTA's tiles only increase, so
      // the owning tensor is found by stepping forward, not by a binary search per tile
      int q_ld = 0, q_st = 0;
      auto where = [&](uint64_t i, int& cur, float*& p, const GT*& g, uint64_t& so, int& q) {
        const uint64_t t = blockIdx.x + i * gridDim.x;
        while (cur + 1 < L.n && tb[cur + 1] <= t) ++cur;  // largest q with tb[q] <= t
        q = cur;
        const uint64_t e = (t - tb[q]) * (uint64_t)kTile;
        p = static_cast<float*>(L.p[q]) + e;
        g = static_cast<const GT*>(L.g[q]) + e;
        so = L.soff[q] + e;
      };
      auto issue = [&](uint64_t i) {
        const int s = (int)(i % NS);
        float* p;
        const GT* g;
        uint64_t so;
        int q;
        where(i, q_ld, p, g, so, q);
        const int sp = SH ? L.shp[q] : 0, sg = SH ? L.shg[q] : 0, ss = SH ? L.shs[q] : 0;
        if constexpr (SH) meta[s] = ListStage{p, so, sp, sg, ss};  // ordered before the arrive
        const float* src[6] = {p - sp, nullptr, s0 + so - ss, s1 + so - ss, s2 + so - ss,
                               s3 + so - ss};
        const uint32_t gbytes = kTile * sizeof(GT) + (sg ? 16u : 0u);
        const uint32_t pbytes = kTile * 4 + (sp ? 16u : 0u);
        const uint32_t sbytes = kTile * 4 + (ss ? 16u : 0u);
        mbar_expect_tx(&full[s], pbytes + gbytes + (uint32_t)(nload - 2) * sbytes);
        for (int j = 0; j < nload; ++j) {
          float* dst = buf + ((size_t)s * NIN + j) * kSlot;
          if (j == 1)
            bulk_g2s<false>(dst, g - sg, gbytes, &full[s], 0);
          else
            bulk_g2s<false>(dst, src[j], j == 0 ? pbytes : sbytes, &full[s], 0);
        }
      };
      // the tile's 16 B-aligned interior of a written stream (all of it when unshifted)
      auto store = [&](float* dst, const float* slot, int sh) {
        if (sh == 0)
          bulk_s2g<false>(dst, slot, kTile * 4, 0);
        else
          bulk_s2g<false>(dst + (4 - sh), slot + 4, (kTile - 4) * 4, 0);
      };
      for (uint64_t i = 0; i < mine && i < (uint64_t)NS; ++i) issue(i);
      for (uint64_t i = 0; i < mine; ++i) {
        const int s = (int)(i % NS);
        mbar_wait(&done[s], (uint32_t)((i / NS) & 1));
        float* p;
        const GT* g;
        uint64_t so;
        int q;
        where(i, q_st, p, g, so, q);
        const int sp = SH ? L.shp[q] : 0, ss = SH ? L.shs[q] : 0;
        float* st = buf + (size_t)s * NIN * kSlot;
        store(p, st, sp);
        store(s0 + so, st + 2 * kSlot, ss);
        if constexpr (KIND == K_ADAMW || KIND == K_ADAN) store(s1 + so, st + 3 * kSlot, ss);
        if constexpr (KIND == K_SOPHIA) {
          if (k.refresh) store(s1 + so, st + 3 * kSlot, ss);
        }
        if constexpr (KIND == K_ADAN) {
          store(s2 + so, st + 4 * kSlot, ss);
          store(s3 + so, st + 5 * kSlot, ss);
        }
        bulk_commit();
        if (i >= 1 && i - 1 + NS < mine) {  // refill the previous tile's stage (flat kernel)
          bulk_wait_read_1();
          issue(i - 1 + NS);
        }
      }
      bulk_wait_all();
    }
  } else {  // ---------------- consumers ----------------
    constexpr int E = C::kEPT;
    const int c0 = threadIdx.x * E;
    for (uint64_t i = 0; i < mine; ++i) {
      const int s = (int)(i % NS);
      mbar_wait(&full[s], (uint32_t)((i / NS) & 1));
      ListStage m{nullptr, 0, 0, 0, 0};
      if constexpr (SH) m = meta[s];
      float* st = buf + (size_t)s * NIN * kSlot + c0;
      float pv[E], gv[E], a[E], b[E], c[E], d[E];
      lds_sh<E>(st, m.shp, pv);
      if (m.shg == 0) {
        if constexpr (sizeof(GT) == 4)
          lds<E>(st + kSlot, gv);
        else
          lds_grad_bf16<E>(buf + (size_t)s * NIN * kSlot + kSlot, c0, gv);
      } else {
        const GT* gslot = reinterpret_cast<const GT*>(buf + (size_t)s * NIN * kSlot + kSlot) + m.shg + c0;
#pragma unroll
        for (int j = 0; j < E; ++j) gv[j] = load_grad1(gslot + j);
      }
      lds_sh<E>(st + 2 * kSlot, m.shs, a);
      if constexpr (KIND != K_LION) lds_sh<E>(st + 3 * kSlot, m.shs, b);
      if constexpr (KIND == K_ADAN) {
        lds_sh<E>(st + 4 * kSlot, m.shs, c);
        if (!k.first) lds_sh<E>(st + 5 * kSlot, m.shs, d);
      }
#pragma unroll
      for (int j = 0; j < E; ++j) {
        if constexpr (KIND == K_LION) b[j] = 0.f;
        if constexpr (KIND != K_ADAN) c[j] = d[j] = 0.f;
        if constexpr (KIND == K_ADAN) {
          if (k.first) d[j] = 0.f;
        }
        update<KIND, float>(pv[j], gv[j], a[j], b[j], c[j], d[j], k);
      }
      sts_sh<E>(st, m.shp, pv);
      sts_sh<E>(st + 2 * kSlot, m.shs, a);
      if constexpr (KIND != K_LION) sts_sh<E>(st + 3 * kSlot, m.shs, b);
      if constexpr (KIND == K_ADAN) {
        sts_sh<E>(st + 4 * kSlot, m.shs, c);
        sts_sh<E>(st + 5 * kSlot, m.shs, d);
      }
      if constexpr (SH) {  // partial granules of shifted written streams, to global memory
        edge_st<E, kTile>(m.p, c0, m.shp, pv);
        edge_st<E, kTile>(s0 + m.so, c0, m.shs, a);
        if constexpr (KIND == K_ADAMW || KIND == K_ADAN) edge_st<E, kTile>(s1 + m.so, c0, m.shs, b);
        if constexpr (KIND == K_SOPHIA) {
          if (k.refresh) edge_st<E, kTile>(s1 + m.so, c0, m.shs, b);
        }
        if constexpr (KIND == K_ADAN) {
          edge_st<E, kTile>(s2 + m.so, c0, m.shs, c);
          edge_st<E, kTile>(s3 + m.so, c0, m.shs, d);
        }
      }
      fence_proxy_async();
      mbar_arrive(&done[s]);
    }
    // scalar elements: consumers of every CTA
    const uint64_t ne = eb[L.n];
    for (uint64_t x = (uint64_t)blockIdx.x * kConsumers + threadIdx.x; x < ne;
         x += (uint64_t)gridDim.x * kConsumers) {
      const int q = list_find(eb, L.n, x);
      const uint64_t e = L.first_scalar[q] + (x - eb[q]), o = L.soff[q] + e;
      float* p = static_cast<float*>(L.p[q]);
      float pp = p[e], gg = load_grad1(static_cast<const GT*>(L.g[q]) + e), aa = s0[o],
            bb = 0.f, cc = 0.f, dd = 0.f;
      if constexpr (KIND != K_LION) bb = s1[o];
      if constexpr (KIND == K_ADAN) {
        cc = s2[o];
        if (!k.first) dd = s3[o];
      }
      update<KIND, float>(pp, gg, aa, bb, cc, dd, k);
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
    graph_bump<DEV>(gs);  // thread 0 is a consumer
  }
}

using ListCfg = TmaCfg<16, 4>;
// Adan on 3 stages, as the flat step: 350M decoder's 241 tensors 2.536 -> 2.412 ms
using ListCfgAdan = TmaCfg<16, 3>;

template <int KIND, typename GT, bool DEV, bool SH>
void run_list_tma_sh(const FlatList& L, float* const* s, const StepConsts<float>& k,
                     const GraphStep& gs, cudaStream_t st) {
  using C = std::conditional_t<KIND == K_ADAN, ListCfgAdan, ListCfg>;  // same tile size
  auto kern = list_tma_kernel<C, KIND, GT, DEV, SH>;
  constexpr int smem = smem_bytes<C, KIND, false>();
  const int dev = current_device();
  static std::atomic<uint64_t> attr_set{0};
  if (!(attr_set.load() & (1ull << dev))) {
    MCO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set.fetch_or(1ull << dev);
  }
  const uint64_t nt = L.vbeg[L.n], ne = L.ebeg[L.n];
  const uint64_t want = std::max<uint64_t>({nt, (ne + C::kConsumers - 1) / C::kConsumers, 1});
  const int grid = (int)std::min<uint64_t>(want, (uint64_t)device_info(dev).sms);
  kern<<<grid, C::kConsumers + 32, smem, st>>>(L, s[0], s[1], s[2], s[3], k, gs);
  launch_check("list_tma_kernel");
}

template <int KIND, typename GT, bool DEV>
void run_list_tma(const FlatList& L, float* const* s, const StepConsts<float>& k,
                  const GraphStep& gs, cudaStream_t st) {
  bool sh = false;
  for (int i = 0; i < L.n && !sh; ++i)
    sh = L.vbeg[i + 1] > L.vbeg[i] && (L.shp[i] || L.shg[i] || L.shs[i]);
  if (sh)
    run_list_tma_sh<KIND, GT, DEV, true>(L, s, k, gs, st);
  else
    run_list_tma_sh<KIND, GT, DEV, false>(L, s, k, gs, st);
}

template <int KIND, typename GT>
void list_tma_dev(const FlatList& L, float* const* s, const StepConsts<float>& k,
                  const GraphStep& gs, cudaStream_t st) {
  if (gs.d)
    run_list_tma<KIND, GT, true>(L, s, k, gs, st);
  else
    run_list_tma<KIND, GT, false>(L, s, k, gs, st);
}

template <typename GT>
void list_tma_kind(int kind, const FlatList& L, float* const* s, const StepConsts<float>& k,
                   const GraphStep& gs, cudaStream_t st) {
  switch (kind) {
    case MCO_ADAMW: list_tma_dev<K_ADAMW, GT>(L, s, k, gs, st); break;
    case MCO_LION: list_tma_dev<K_LION, GT>(L, s, k, gs, st); break;
    case MCO_ADAN: list_tma_dev<K_ADAN, GT>(L, s, k, gs, st); break;
    case MCO_SOPHIA: list_tma_dev<K_SOPHIA, GT>(L, s, k, gs, st); break;
    default: throw Error(MCO_CONTRACT, "list_tma: unsupported kind");
  }
}

}  // namespace

bool flat_tma_eligible(const FlatArgs& a, int cfg) {
  if (a.state_dtype != MCO_F32 || a.p_dtype != MCO_F32) return false;
  if (a.g_dtype != MCO_F32 && a.g_dtype != MCO_BF16) return false;
  auto al = [](const void* q) { return q == nullptr || ((uintptr_t)q % 16) == 0; };
  // every stream but the gradient 16 B aligned; the gradient element-aligned (its 16 B
  // phase may differ: flat_tma_kernel's gsh)
  bool ok = al(a.p) && al(a.p_out_bf16) && ((uintptr_t)a.g % (a.g_dtype == MCO_BF16 ? 2 : 4)) == 0;
  for (int i = 0; i < 4; ++i) ok = ok && al(a.s[i]);
  return ok && a.n >= (uint64_t)tma_tile(cfg) + (al(a.g) ? 0 : (uint64_t)tma_tile(cfg));
}

#define MCO_UNPAREN(...) __VA_ARGS__
#define MCO_TMA_CONFIGS(X)        \
  X(0, (TmaCfg<16, 4>))             \
  X(1, (TmaCfg<16, 3>))             \
  X(2, (TmaCfg<16, 5>))             \
  X(3, (TmaCfg<24, 4>))             \
  X(4, (TmaCfg<8, 4>))              \
  X(5, (TmaCfg<16, 8, 2>))          \
  X(6, (TmaCfg<16, 4, 4, true>))    \
  X(7, (TmaCfg<24, 6, 2>))          \
  X(8, (TmaCfg<16, 4, 4, false, true>)) \
  X(9, (TmaCfg<16, 2>))

int tma_tile(int cfg) {
  switch (cfg) {
#define X(id, cfg) \
  case id: return MCO_UNPAREN cfg::kTile;
    MCO_TMA_CONFIGS(X)
#undef X
  }
  throw Error(MCO_CONFIG, "flat_tma: unknown configuration");
}

void launch_flat_tma(const FlatArgs& a, const StepConsts<float>& k, cudaStream_t st, int cfg) {
  switch (cfg) {
#define X(id, cfg) \
  case id: launch_cfg<MCO_UNPAREN cfg>(a, k, st); return;
    MCO_TMA_CONFIGS(X)
#undef X
  }
  throw Error(MCO_CONFIG, "flat_tma: unknown configuration");
}

bool lomo_tma_eligible(const void* p, int p_dtype, const void* g, int g_dtype, uint64_t n) {
  if (p_dtype != g_dtype || (p_dtype != MCO_F32 && p_dtype != MCO_BF16)) return false;
  const size_t es = p_dtype == MCO_F32 ? 4 : 2;
  // parameters 16 B aligned; the gradient element-aligned (its phase may differ: gsh)
  if (((uintptr_t)p % 16) || ((uintptr_t)g % es)) return false;
  const uint64_t tile = p_dtype == MCO_F32 ? lomo_tile<float>() : lomo_tile<uint16_t>();
  return n >= tile * (((uintptr_t)g % 16) ? 2 : 1);
}

void launch_lomo_tma(void* p, int p_dtype, const void* g, uint64_t n, double lr, double scale,
                     const double* sumsq, double clip, cudaStream_t st, int stages) {
  const bool f32 = p_dtype == MCO_F32;
  switch (stages) {
    case 4:
      f32 ? run_lomo_tma<float, 4>(p, g, n, lr, scale, sumsq, clip, st)
          : run_lomo_tma<uint16_t, 4>(p, g, n, lr, scale, sumsq, clip, st);
      break;
    case 12:
      f32 ? run_lomo_tma<float, 12>(p, g, n, lr, scale, sumsq, clip, st)
          : run_lomo_tma<uint16_t, 12>(p, g, n, lr, scale, sumsq, clip, st);
      break;
    default:
      f32 ? run_lomo_tma<float, 8>(p, g, n, lr, scale, sumsq, clip, st)
          : run_lomo_tma<uint16_t, 8>(p, g, n, lr, scale, sumsq, clip, st);
  }
}

int list_tma_tile() { return ListCfg::kTile; }

void launch_list_tma(int kind, int g_dtype, const FlatList& L, float* const* s,
                     const StepConsts<float>& k, const GraphStep& gs, cudaStream_t st) {
  if (g_dtype == MCO_BF16)
    list_tma_kind<uint16_t>(kind, L, s, k, gs, st);
  else
    list_tma_kind<float>(kind, L, s, k, gs, st);
}

}  // namespace mco
