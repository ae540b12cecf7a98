#!/bin/bash
# Halo weight-gradient kernel: focused parity first (teacher-forced per-layer
# dW2, ResNet tests), then the A/B timing script.
set -u
timeout 900 python -m pytest tests/test_bench_parity_gpu.py -q -s -x -k "teacher_forced and vgg16-1" 2>&1 | grep -oE "dW1 [0-9.e+-]+|dW2 [0-9.e+-]+|dW3 [0-9.e+-]+|[0-9]+ (passed|failed)" | tr '\n' ' '; echo
TAG=r02zk bash tools/r02zb.sh
