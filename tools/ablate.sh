for m in 0 64 72 4 8 512 2 0x240; do
  PPB_PROBE_SKIP=$m python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$m', round(d['ms_per_step'],4))"
done
