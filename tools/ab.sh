#!/bin/bash
# A/B of the step's feature switches on one box (same clocks): bench.py lines
# per variant, interleaved twice.  Usage (under gpurun): bash tools/ab.sh <tag> "<ENV=1 ...>" ...
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "base" "$@"; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    line=$(env $envs timeout 300 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | tail -1)
    echo "$rep|$v|$line" >> gpurun_out/${TAG}_ab.txt
    python -c "import json,sys; d=json.loads(sys.argv[2]); print(sys.argv[1], round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$v" "$line"
  done
done
