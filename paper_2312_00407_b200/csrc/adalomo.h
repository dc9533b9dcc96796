// AdaLomo tile plan (host) and launch interface.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace mco {

constexpr int kCW = 8;            // columns per lane chunk
constexpr int kMaxTileRows = 128;  // bounds fp32 column partial length and smem

struct Tile {
  int32_t tensor;
  int32_t cb;  // column block
  int64_t rb;  // row block
  int64_t r0, r1, c0, c1;  // 1-D tensors: [r0, r1) is the element range
};

// Work unit of the two streaming passes after the statistics (K4, K6): a flat
// element range of one tensor; row / column recovered per 8-wide vector.
struct Chunk {
  int32_t tensor, pad;
  int64_t e0, e1;
};
constexpr int64_t kChunkElems = 1 << 16;

struct TensorInfo {
  int64_t numel, rows, cols;
  int32_t factored, tc;  // tc: column lanes per row group (32/64/128)
  int32_t kc;            // column blocks
  uint32_t div_m;        // row = umulhi(e, div_m) >> div_s  (e / cols, e < 2^31; cols > 1)
  int32_t div_s, pad0;
  int64_t nrb;           // row blocks
  int64_t elem_off;      // offset in the registry-order flat buffer
  int64_t vrow_off, vcol_off, vfull_off;  // fp64 state offsets
  int64_t colpart_off, rowpart_off, fa_off, fb_off;
  int64_t tile_begin, tile_end;
  int64_t chunk_begin, chunk_end;
  int64_t t;  // per-entry step counter (optim.hpp:93), advanced on the device
  // row-split sharding: statistics normalise by the global shape; the payload
  // contribution is scaled by `weight` (0 on ranks holding a duplicate replica)
  int64_t rows_global, numel_global;
  double weight;
};

struct AdaLomoPlan {
  mco_config cfg{};
  int device = 0;
  // global grad-norm clip of the gradients before the AdaLomo update (BASELINE C3, beyond
  // the reference: its AdaLomoState ignores clip_threshold, which is LOMO's,
  // optim.hpp:28).  Opt-in through mco_adalomo_set_grad_clip only.
  int grad_clip_on = 0;
  double grad_clip = 0.0;
  std::vector<TensorInfo> h_tensors;
  std::vector<Tile> h_tiles;
  std::vector<Chunk> h_chunks;
  std::vector<int64_t> h_item_off;  // per tensor prefix of (rows + cols) for factored
  std::vector<int64_t> h_col_off;   // per tensor prefix of cols for factored
  int64_t state_len = 0, colpart_len = 0, rowpart_len = 0, fa_len = 0, fb_len = 0;
  int64_t stats_len = 0, usq_len = 0;  // payload: [3 per tensor | column sums] + [usq]
  // device
  Tile* d_tiles = nullptr;
  Chunk* d_chunks = nullptr;
  double* d_chunk_sc = nullptr;  // per-chunk sum u^2
  TensorInfo* d_tensors = nullptr;
  int64_t* d_item_off = nullptr;
  int64_t* d_col_off = nullptr;
  double* d_payload = nullptr;  // stats_len + usq_len doubles
  double* d_state = nullptr;
  float* d_colpart = nullptr;
  double* d_rowpart = nullptr;
  double* d_tile_sc = nullptr;
  double* d_tens_sc = nullptr;
  float* d_fa = nullptr;
  float* d_fb = nullptr;
  float* d_fra = nullptr;     // 1/sqrt(a_i), 1/sqrt(b_j): separable form of u
  float* d_frb = nullptr;
  unsigned* d_mins = nullptr;  // 2 per tensor: min a, min b (fp32 bits)
  double* d_glob = nullptr;
};

constexpr int kMaxTab = 64;  // tensors per list call (pointer table in the kernel params)

struct AdaLomoCall {
  int t0, t1;  // tensor range [t0, t1)
  void* p;
  int p_dtype;  // MCO_F32 or MCO_BF16 (bf16 storage: fp32 arithmetic, RNE store)
  const void* g;
  int g_dtype;
  int single;
  double lr;
  int use_clip;
  const double* ext_sumsq;  // device global sum g^2 (hook form), or null
  // phases run back to back (no all-reduce between them): KR's scalar block does K2's
  // work and K4's last CTA K5's -- 5 launches per call instead of 7
  int fuse_usq;
  // phase 1 statistics: 0 / 3 all, 1 gradient statistics only, 2 sum p^2 only
  int stats_mode;
  // hook form, tensor after tensor on one stream: K6 triggers its dependents early and
  // the next tensor's K1 starts without waiting (adalomo.cu k1_stats).  early may only be
  // set when the previous kernel in the stream is a K6 of another tensor.
  int trigger, early;
  // list form: tensor t0 + i lives at ptab[i] / gtab[i] (separate allocations, the
  // per-parameter tensors of a model); ntab = 0 -> flat buffers / single tensor
  int ntab;
  void* ptab[kMaxTab];
  const void* gtab[kMaxTab];
};

// Build the host tile plan for `shapes` (registry order) on a device with `sms` SMs.
void build_adalomo_plan(AdaLomoPlan& pl, const std::vector<std::vector<int64_t>>& shapes,
                        int sms);
// phase 1: K1 + payload reduction; phase 2: K2, K3, K4 + usq payload; phase 3: K5, K6.
// Between phases a sharded caller all-reduces the payload (row-split tensors).
void launch_adalomo_phase(const AdaLomoPlan& pl, const AdaLomoCall& call, int phase,
                          cudaStream_t st);
void launch_adalomo(const AdaLomoPlan& pl, const AdaLomoCall& call, cudaStream_t st);
// out = sum over tensors [t0, t1) of the payload's sum g^2, in K2's reduction order.
void launch_adalomo_gsumsq(const AdaLomoPlan& pl, int t0, int t1, double* out, cudaStream_t st);

}  // namespace mco
