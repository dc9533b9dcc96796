#!/bin/bash
# compute-sanitizer over the TMA pipeline kernel and the overlapped ZeRO step (one B200).
for tool in memcheck racecheck synccheck; do
  echo "## $tool: flat_tma_kernel (variant tests, every kind, tails, mixed output)"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_flat.py -q -x \
      -k "variants and tma and not tma_s3 and not tma24 and not tma8 and not 1048581" 2>&1 | grep -E "passed|failed|SUMMARY|rror|azard" | head -8
done
echo "## memcheck: overlapped ZeRO step (side stream, per-bucket kernels)"
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_overlap.py -q -x -k "equals_flat" 2>&1 | grep -E "passed|failed|SUMMARY|rror" | head -5
