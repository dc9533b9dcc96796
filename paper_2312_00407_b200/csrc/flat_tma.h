// TMA-staged flat optimizer step (flat_tma.cu).
#pragma once

#include "kernels.h"

namespace mco {

// fp32 state / params / grads, 16 B aligned buffers, at least one 2048-element tile.
bool flat_tma_eligible(const FlatArgs& a);
void launch_flat_tma(const FlatArgs& a, const StepConsts<float>& k, cudaStream_t st);

}  // namespace mco
