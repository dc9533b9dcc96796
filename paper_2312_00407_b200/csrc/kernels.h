// Host-side launch interface of the sm_100a kernels (used by abi.cpp).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mco {

// FlatOptimizer state (SoA, optim.cpp:74-98).  s[0..3] are, per kind:
//   adamw  m, v          lion   m
//   adan   m, v, n, gp   sophia m, h
struct FlatArgs {
  int kind;
  int state_dtype;  // MCO_F32 / MCO_F64
  void* p;
  int p_dtype;
  const void* g;
  int g_dtype;
  void* s[4];
  uint16_t* p_out_bf16;  // mixed step only
  uint64_t n;
  // graph mode (common.cuh): the step scalars come from the device step counter;
  // gs.d null = the by-value scalars of launch_flat_step
  GraphStep gs;
};

// Launch one fused read-grad / update-state / write-param pass.
// `kd` / `kf` carry the per-step scalars (only the one matching state_dtype is used).
void launch_flat_step(const FlatArgs& a, const StepConsts<float>& kf,
                      const StepConsts<double>& kd, cudaStream_t st);

// Sophia with an fp64 first moment ("precise-m", state MCO_F32M64; sophia_m64.cu).
void launch_sophia_m64(float* p, const void* g, int g_dtype, double* m, float* h, uint64_t n,
                       const StepConsts<double>& kd, cudaStream_t st);

// List form: separate parameter / gradient tensors over the flat state (tensor i's state
// at the sum of the preceding lengths).  One launch per kListMax tensors.
#ifndef MCO_LIST_MAX
#define MCO_LIST_MAX 40
#endif
constexpr int kListMax = MCO_LIST_MAX;
struct FlatList {  // one launch (kernel parameter)
  int n;
  uint64_t vbeg[kListMax + 1];      // prefix sums: vector-path vectors
  uint64_t ebeg[kListMax + 1];      // prefix sums: scalar-path elements
  uint64_t first_scalar[kListMax];  // first element on the scalar path
  void* p[kListMax];
  const void* g[kListMax];
  uint64_t soff[kListMax];          // state offset (elements)
  // TMA list form: each stream's element phase within 16 B (params, grads, state) --
  // streams off the 16 B grid are copied from their aligned-down address (list_tma_kernel)
  uint8_t shp[kListMax], shg[kListMax], shs[kListMax];
};
struct FlatListArgs {
  int kind;
  int state_dtype;
  int p_dtype;
  int g_dtype;
  int count;
  void* const* p;
  const void* const* g;
  const uint64_t* len;
  void* s[4];  // state slots at the list's first element
  GraphStep gs;
};
// LOMO over separate tensors (FlatList vbeg = vectors, no state), one launch per
// kListMax tensors; dev_sumsq != null: the global-norm clip scale from the device sum.
void launch_lomo_list(int count, void* const* p, int p_dtype, const void* const* g, int g_dtype,
                      const uint64_t* len, double lr, double scale, const double* dev_sumsq,
                      double clip, cudaStream_t st);
void launch_flat_step_list(const FlatListArgs& a, const StepConsts<float>& kf,
                           const StepConsts<double>& kd, cudaStream_t st);

// Graph mode: a step with no elements still counts (t += 1 on the device).
void launch_flat_graph_bump(FlatGraphDev* d, cudaStream_t st);

// Flat-kernel variant (tuning knob; "ldg" default, "tma", ...).  Throws CONFIG on an
// unknown name.
void set_flat_variant(const char* name);
const char* flat_variant_name();

// LOMO p -= f*g with f = lr*scale (host) or derived from a device Σg² (clip).
void launch_lomo(void* p, int p_dtype, const void* g, int g_dtype, uint64_t n, double lr,
                 double scale, const double* dev_sumsq, double clip, cudaStream_t st);

// Deterministic Σx² -> *out (double).  ws: >= sumsq_ws_bytes() device bytes
// private to the stream; counter word must start at zero (kernel re-arms it).
size_t sumsq_ws_bytes();
void launch_sumsq(const void* x, int dtype, uint64_t n, double* out, int accumulate, void* ws,
                  cudaStream_t st);

// Synthetic input generator.
void launch_synth(void* dst, int dtype, uint64_t n, uint64_t key, int64_t cols, int scale_log2,
                  int zero_log2, int rowcol, cudaStream_t st);
uint64_t synth_key(uint64_t seed, uint32_t role, uint32_t tensor, uint32_t step);

}  // namespace mco
