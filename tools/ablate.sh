# Step-time ablations (timing probes: results are wrong).  PPB_PROBE_SKIP is a
# bitmask of session op kinds (1<<kind, session.h OpKind); PPB_PROBE_NO_REDUCE
# drops the split-K reduction kernels.
run() { python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$1', round(d['ms_per_step'],4))"; }
run base
PPB_PROBE_NO_REDUCE=1 run no_reduce
PPB_PROBE_SKIP=64 run no_bias
PPB_PROBE_SKIP=512 run no_pool
PPB_PROBE_SKIP=1024 run no_merge
PPB_PROBE_SKIP=8 run no_wgrad
PPB_PROBE_SKIP=4 run no_dgrad
PPB_PROBE_SKIP=2 run no_fwd
PPB_PROBE_SKIP=0x690 run no_small
