#!/bin/bash
# db race fix: the teacher-forced per-layer test repeated (it caught the race
# intermittently), then the A/B timing script.
set -u
for i in 1 2 3 4 5; do
  timeout 600 python -m pytest tests/test_bench_parity_gpu.py -q -s -k "teacher_forced and vgg16-1" 2>&1 | grep -oE "db3 [0-9.e+-]+|db4 [0-9.e+-]+|[0-9]+ (passed|failed)" | tr '\n' ' '; echo
done
TAG=r02zh bash tools/r02zb.sh
