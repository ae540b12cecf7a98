set -u
mkdir -p gpurun_out
for cfg in "vgg16 --n 1 --Z 1 --m 4" "vgg16 --n 2 --Z 2 --m 4" "mlp784 --n 2 --Z 3 --m 4" "wide_mlp --n 2 --Z 2 --m 4"; do
  timeout 600 python tools/sim_crosscheck.py $cfg >> gpurun_out/r02i_simcheck.jsonl 2> gpurun_out/r02i_simcheck.err; echo "sim $cfg rc=$?"
done
tail -3 gpurun_out/r02i_simcheck.err
for k in 2 4 8; do
  PPB_BENCH_PLAN_DEVICES=$k timeout 600 python bench.py --workload wide_mlp --no-cpu-baseline --steps 20 > gpurun_out/r02i_bench_wide_mlp_n$k.json 2> gpurun_out/r02i_bench_wide_mlp_n$k.err; echo "wide n=$k rc=$?"
done
timeout 1800 python -m pytest tests/test_bench_parity_gpu.py -q -x -k "wide_mlp" > gpurun_out/r02i_wide_parity.txt 2>&1; echo "wide parity rc=$?"; tail -2 gpurun_out/r02i_wide_parity.txt
