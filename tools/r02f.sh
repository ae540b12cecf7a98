set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_train_gpu.py -q -x > gpurun_out/r02f_train.txt 2>&1; echo "train rc=$?"; tail -3 gpurun_out/r02f_train.txt
timeout 1200 python -m pytest tests/test_bench_parity_gpu.py -q -x -k "proposed or microbatched or (vgg16_b512_bench_config and 1)" > gpurun_out/r02f_parity.txt 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r02f_parity.txt
for mm in "1 stash_all" "4 stash_all" "4 proposed" "2 proposed" "8 proposed"; do set -- $mm
  timeout 300 python bench.py --no-cpu-baseline --steps 50 --m $1 --memory $2 > gpurun_out/r02f_bench_m$1_$2.json 2> gpurun_out/r02f_bench_m$1_$2.err; echo "bench m=$1 $2 rc=$?"
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); c=d['config']; print(d['ms_per_step'], c['stash_bytes']/2**20, c['device_bytes']/2**20)" gpurun_out/r02f_bench_m$1_$2.json
done
