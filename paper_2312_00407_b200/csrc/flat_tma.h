// TMA-staged flat optimizer step (flat_tma.cu).
#pragma once

#include "kernels.h"

namespace mco {

// cfg (consumer warps, stages[, elements per thread, L2 hint]): 0 = (16, 4) default,
// 1 = (16, 3), 2 = (16, 5), 3 = (24, 4), 4 = (8, 4), 5 = (16, 8, 2), 6 = (16, 4, 4,
// evict-first), 7 = (24, 6, 2).  A tile is 32 * EPT elements per consumer warp.
int tma_tile(int cfg);
// fp32 state / params, fp32 or bf16 grads, 16 B aligned buffers, at least one tile.
bool flat_tma_eligible(const FlatArgs& a, int cfg);
void launch_flat_tma(const FlatArgs& a, const StepConsts<float>& k, cudaStream_t st, int cfg);

// LOMO p -= f*g on the TMA pipeline: fp32/fp32 or bf16/bf16, 16 B aligned, >= one tile.
bool lomo_tma_eligible(const void* p, int p_dtype, const void* g, int g_dtype, uint64_t n);
void launch_lomo_tma(void* p, int p_dtype, const void* g, uint64_t n, double lr, double scale,
                     const double* sumsq, double clip, cudaStream_t st, int stages);

// List form on the pipeline (flat_list.cu): L.vbeg = tile prefix sums (list_tma_tile()
// elements per tile; tensors 16 B aligned in p, g and state), L.ebeg = scalar elements.
int list_tma_tile();
void launch_list_tma(int kind, int g_dtype, const FlatList& L, float* const* s,
                     const StepConsts<float>& k, const GraphStep& gs, cudaStream_t st);

}  // namespace mco
