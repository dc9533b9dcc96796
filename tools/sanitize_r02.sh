#!/bin/bash
# compute-sanitizer over the round-2 kernels (one B200): the shifted-gradient TMA reads
# (flat_tma_kernel / lomo_tma_kernel gsh: aligned-down copies one granule longer), the
# AdaLomo per-tensor vector/scalar split, KR's per-tensor blocks with the ticketed K2,
# K4's packed-pair form, and the one-launch cluster kernel for small 1-D tensors (DSMEM).
export MCO_UNDER_SANITIZER=1
for tool in memcheck racecheck synccheck; do
  echo "## $tool: shifted gradient reads (flat kinds + LOMO, every phase pair, fp32)"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_flat.py -q -x \
      -k "phase_shift and ((8192 and f32) or lomo)" 2>&1 | grep -E "passed|failed|SUMMARY|rror|azard" | head -8
  echo "## $tool: list form (shifted streams, cursor lookup) and Sophia precise-m (bulk-copy pipeline)"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_flat_list.py tests/test_gpu_flat.py -q -x \
      -k "(not random and not variants and not tiny and not phase_shift and not sampled and not f64 and not host_span) or precise_m or different_phases" 2>&1 | grep -E "passed|failed|SUMMARY|rror|azard" | head -8
  echo "## $tool: AdaLomo (mixed alignment incl. the strided scalar tiles, hook form incl. k_small_vec, CUDA-graph replay, reference parity)"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_fused.py -q -x \
      -k "mixed_alignment or hook_form_replays or adalomo_matches_reference or list_form_equals" 2>&1 | grep -E "passed|failed|SUMMARY|rror|azard" | head -8
done
