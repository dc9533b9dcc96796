#!/bin/bash
# AdaLomo hook form: where the time goes (tools/hook_parts.py), with and without the
# one-launch small-vector kernel.
mkdir -p gpurun_out
python tools/hook_parts.py > gpurun_out/hook_parts.jsonl 2>&1
MCO_ADALOMO_SMALL=0 python tools/hook_parts.py >> gpurun_out/hook_parts.jsonl 2>&1
cat gpurun_out/hook_parts.jsonl
