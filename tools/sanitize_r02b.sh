#!/bin/bash
# compute-sanitizer over the late round-2 AdaLomo one-tensor paths: KR's tensor block
# running K2 from registers (k2_one), K4's last CTA running K5 from warp 0's sum (k5_val),
# the 16-deep partial walks -- through the hook form, its CUDA-graph replay, the list form
# and the reference-parity tests -- and the LOMO host path's kept resident gradient.
export MCO_UNDER_SANITIZER=1
for tool in memcheck racecheck synccheck; do
  echo "## $tool: AdaLomo hook form / list form / reference parity, LOMO host cache"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_fused.py -q -x \
      -k "hook_form or adalomo_matches_reference or list_form_equals or rank1 or resident_gradient or host_path" 2>&1 | grep -E "passed|failed|SUMMARY|rror|azard" | head -8
done
