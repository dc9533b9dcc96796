#!/bin/bash
# compute-sanitizer over the TMA pipeline kernels (flat_tma_kernel, lomo_tma_kernel), the
# PDL-chained AdaLomo kernels and the overlapped ZeRO step (one B200).
for tool in memcheck racecheck synccheck; do
  echo "## $tool: flat_tma_kernel (variant tests, every kind, tails, mixed output)"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_flat.py -q -x \
      -k "(variants or bf16_grads_both or phase_peeling or tiny_gradients) and tma and not tma_ and not tma24 and not tma8 and not 1048581" 2>&1 | grep -E "passed|failed|SUMMARY|rror|azard" | head -8
  echo "## $tool: lomo_tma_kernel (fp32 / bf16, device clip)"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_fused.py -q -x \
      -k "lomo_variants and tma and not tma_ and not 1048581" 2>&1 | grep -E "passed|failed|SUMMARY|rror|azard" | head -8
  echo "## $tool: graph mode (device step counter, last-CTA bump) and list form"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_graph.py tests/test_gpu_flat_list.py -q -x \
      -k "not 10000000 and not f64" 2>&1 | grep -E "passed|failed|SUMMARY|rror|azard" | head -8
  echo "## $tool: AdaLomo (PDL chain; hook and multi-tensor forms)"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_fused.py -q -x \
      -k "adalomo and not reference" 2>&1 | grep -E "passed|failed|SUMMARY|rror|azard" | head -8
done
echo "## memcheck: overlapped ZeRO step (side stream, per-bucket kernels)"
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_overlap.py -q -x -k "equals_flat" 2>&1 | grep -E "passed|failed|SUMMARY|rror" | head -5
