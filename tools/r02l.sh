set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_train_gpu.py tests/test_dropin_gpu.py tests/test_schedule_sim.py -q -x > gpurun_out/r02l_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02l_tests.txt
timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err; echo "bench rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e'], d['clocks'])" gpurun_out/r02l_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:'im2col' --clock-control none --csv --log-file gpurun_out/r02l_ew.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ew rc=$?"
python tools/ew_ncu.py gpurun_out/r02l_ew.csv
