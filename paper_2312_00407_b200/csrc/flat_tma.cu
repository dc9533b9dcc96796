// TMA-staged variant of the fused elementwise optimizer step (AdamW / Lion /
// Adan / Sophia, fp32).  Same arithmetic (update.cuh) and therefore the same bits
// as flat_step_kernel; only the data movement differs:
//
//   producer warp (one elected lane)          consumer warps (256 threads)
//   cp.async.bulk global->smem, per stream  ->  wait full[s]; 8 elements / thread:
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

#include "flat_tma.h"
#include "update.cuh"

namespace mco {
namespace {

using namespace upd;
constexpr int kTile = 2048;  // elements per stream per stage (8 KB of fp32)
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kSmemBudget = 200 * 1024;

template <int KIND>
constexpr int n_in() {  // p, g, s0 [, s1 [, s2, s3]]
  return KIND == K_ADAN ? 6 : (KIND == K_LION ? 3 : 4);
}
template <int KIND, bool MIXED>
constexpr int stages() {
  constexpr int per = n_in<KIND>() * kTile * 4 + (MIXED ? kTile * 2 : 0);
  constexpr int s = kSmemBudget / per;
  return s > 8 ? 8 : s;
}
template <int KIND, bool MIXED>
constexpr int smem_bytes() {
  return stages<KIND, MIXED>() * (n_in<KIND>() * kTile * 4 + (MIXED ? kTile * 2 : 0)) +
         2 * stages<KIND, MIXED>() * 8;
}

__device__ __forceinline__ uint32_t sa(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(sa(dst)),
      "l"(src), "r"(bytes), "r"(sa(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(sa(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void lds8(const float* s, float (&r)[8]) {
  const float4 x = reinterpret_cast<const float4*>(s)[0], y = reinterpret_cast<const float4*>(s)[1];
  r[0] = x.x, r[1] = x.y, r[2] = x.z, r[3] = x.w, r[4] = y.x, r[5] = y.y, r[6] = y.z, r[7] = y.w;
}
__device__ __forceinline__ void sts8(float* s, const float (&r)[8]) {
  reinterpret_cast<float4*>(s)[0] = make_float4(r[0], r[1], r[2], r[3]);
  reinterpret_cast<float4*>(s)[1] = make_float4(r[4], r[5], r[6], r[7]);
}

template <int KIND, bool MIXED>
__global__ void __launch_bounds__(kConsumers + 32, 1)
    flat_tma_kernel(float* p, const float* g, float* s0, float* s1, float* s2, float* s3,
                    uint16_t* pout, uint64_t ntiles, uint64_t n, const StepConsts<float> k) {
  constexpr int NIN = n_in<KIND>();
  constexpr int NS = stages<KIND, MIXED>();
  extern __shared__ __align__(128) uint8_t smem[];
  float* buf = reinterpret_cast<float*>(smem);  // [NS][NIN][kTile]
  uint16_t* obuf = reinterpret_cast<uint16_t*>(buf + NS * NIN * kTile);  // [NS][kTile]
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

  // stream j of a stage: 0 p, 1 g, 2 s0, 3 s1, 4 s2, 5 s3
  const float* src[6] = {p, g, s0, s1, s2, s3};
  const uint64_t mine =
      ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (warp == kConsumerWarps) {  // ---------------- producer ----------------
    if (lane == 0) {
      const bool skip_gp = (KIND == K_ADAN) && k.first;  // g_prev unused at t == 1
      const int nload = skip_gp ? NIN - 1 : NIN;
      auto issue = [&](uint64_t i) {
        const int s = (int)(i % NS);
        const uint64_t e = (blockIdx.x + i * gridDim.x) * (uint64_t)kTile;
        mbar_expect_tx(&full[s], (uint32_t)(nload * kTile * 4));
        for (int j = 0; j < nload; ++j)
          bulk_g2s(buf + ((size_t)s * NIN + j) * kTile, src[j] + e, kTile * 4, &full[s]);
      };
      for (uint64_t i = 0; i < mine && i < (uint64_t)NS; ++i) issue(i);
      for (uint64_t i = 0; i < mine; ++i) {
        const int s = (int)(i % NS);
        mbar_wait(&done[s], (uint32_t)((i / NS) & 1));
        const uint64_t e = (blockIdx.x + i * gridDim.x) * (uint64_t)kTile;
        float* st = buf + (size_t)s * NIN * kTile;
        bulk_s2g(p + e, st, kTile * 4);
        bulk_s2g(s0 + e, st + 2 * kTile, kTile * 4);
        if constexpr (KIND == K_ADAMW || KIND == K_ADAN) bulk_s2g(s1 + e, st + 3 * kTile, kTile * 4);
        if constexpr (KIND == K_SOPHIA) {
          if (k.refresh) bulk_s2g(s1 + e, st + 3 * kTile, kTile * 4);
        }
        if constexpr (KIND == K_ADAN) {
          bulk_s2g(s2 + e, st + 4 * kTile, kTile * 4);
          bulk_s2g(s3 + e, st + 5 * kTile, kTile * 4);
        }
        if constexpr (MIXED) bulk_s2g(pout + e, obuf + (size_t)s * kTile, kTile * 2);
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
    const int c8 = threadIdx.x * 8;
    for (uint64_t i = 0; i < mine; ++i) {
      const int s = (int)(i % NS);
      mbar_wait(&full[s], (uint32_t)((i / NS) & 1));
      float* st = buf + (size_t)s * NIN * kTile + c8;
      float pv[8], gv[8], a[8], b[8], c[8], d[8];
      lds8(st, pv);
      lds8(st + kTile, gv);
      lds8(st + 2 * kTile, a);
      if constexpr (KIND != K_LION) lds8(st + 3 * kTile, b);
      if constexpr (KIND == K_ADAN) {
        lds8(st + 4 * kTile, c);
        if (!k.first) lds8(st + 5 * kTile, d);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if constexpr (KIND == K_LION) b[j] = 0.f;
        if constexpr (KIND != K_ADAN) c[j] = d[j] = 0.f;
        if constexpr (KIND == K_ADAN) {
          if (k.first) d[j] = 0.f;
        }
        update<KIND, float>(pv[j], gv[j], a[j], b[j], c[j], d[j], k);
      }
      sts8(st, pv);
      sts8(st + 2 * kTile, a);
      if constexpr (KIND != K_LION) sts8(st + 3 * kTile, b);
      if constexpr (KIND == K_ADAN) {
        sts8(st + 4 * kTile, c);
        sts8(st + 5 * kTile, d);
      }
      if constexpr (MIXED) {
        uint32_t* o = reinterpret_cast<uint32_t*>(obuf + (size_t)s * kTile + c8);
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = f2bf2_bits(pv[2 * j], pv[2 * j + 1]);
      }
      fence_proxy_async();  // generic-proxy smem writes -> visible to the bulk store
      mbar_arrive(&done[s]);
    }
    // tail (< one tile): plain loads / stores by the consumer threads of CTA 0
    if (blockIdx.x == 0) {
      for (uint64_t e = ntiles * kTile + threadIdx.x; e < n; e += kConsumers) {
        float pp = p[e], gg = g[e], aa = s0[e], bb = 0.f, cc = 0.f, dd = 0.f;
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
  }
}

template <int KIND, bool MIXED>
void run(const FlatArgs& a, const StepConsts<float>& k, cudaStream_t st) {
  auto kern = flat_tma_kernel<KIND, MIXED>;
  constexpr int smem = smem_bytes<KIND, MIXED>();
  static bool attr = false;
  if (!attr) {
    MCO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const uint64_t ntiles = a.n / kTile;
  const int grid = (int)std::max<uint64_t>(
      1, std::min<uint64_t>(ntiles ? ntiles : 1, (uint64_t)device_info(current_device()).sms));
  kern<<<grid, kConsumers + 32, smem, st>>>((float*)a.p, (const float*)a.g, (float*)a.s[0],
                                            (float*)a.s[1], (float*)a.s[2], (float*)a.s[3],
                                            a.p_out_bf16, ntiles, a.n, k);
  launch_check("flat_tma_kernel");
}

template <int KIND>
void dispatch(const FlatArgs& a, const StepConsts<float>& k, cudaStream_t st) {
  if (a.p_out_bf16)
    run<KIND, true>(a, k, st);
  else
    run<KIND, false>(a, k, st);
}

}  // namespace

bool flat_tma_eligible(const FlatArgs& a) {
  if (a.state_dtype != MCO_F32 || a.p_dtype != MCO_F32 || a.g_dtype != MCO_F32) return false;
  auto al = [](const void* q) { return q == nullptr || ((uintptr_t)q % 16) == 0; };
  bool ok = al(a.p) && al(a.g) && al(a.p_out_bf16);
  for (int i = 0; i < 4; ++i) ok = ok && al(a.s[i]);
  return ok && a.n >= (uint64_t)kTile;
}

void launch_flat_tma(const FlatArgs& a, const StepConsts<float>& k, cudaStream_t st) {
  switch (a.kind) {
    case MCO_ADAMW: dispatch<K_ADAMW>(a, k, st); break;
    case MCO_LION: dispatch<K_LION>(a, k, st); break;
    case MCO_ADAN: dispatch<K_ADAN>(a, k, st); break;
    case MCO_SOPHIA: dispatch<K_SOPHIA>(a, k, st); break;
    default: throw Error(MCO_CONTRACT, "flat_tma: unsupported kind");
  }
}

}  // namespace mco
