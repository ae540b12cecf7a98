set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_conv_gpu.py tests/test_cnn_gpu.py -q -x > gpurun_out/r02k_conv.txt 2>&1; echo "conv rc=$?"; tail -2 gpurun_out/r02k_conv.txt
timeout 300 python tools/profile_ops.py vgg16 > gpurun_out/r02k_ops.jsonl 2>&1; echo "ops rc=$?"
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/r02k_bench_$i.json 2> gpurun_out/r02k_bench_$i.err; echo "bench rc=$?"; python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks'])" gpurun_out/r02k_bench_$i.json; done
timeout 600 python tools/overlap_trace.py vgg16 4 proposed > gpurun_out/r02k_overlap_m4_proposed.jsonl 2>&1; echo "ovl rc=$?"; tail -1 gpurun_out/r02k_overlap_m4_proposed.jsonl | cut -c1-600
timeout 600 python tools/overlap_trace.py vgg16 4 stash_all > gpurun_out/r02k_overlap_m4_stash_all.jsonl 2>&1; echo "ovl2 rc=$?"; tail -1 gpurun_out/r02k_overlap_m4_stash_all.jsonl | cut -c1-600
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:'pool_fwd|conv_merge|dense_conv|splitk_epilogue|colsum|bias_update|loss_head|im2col|reduce_mask|finalize' --clock-control none --csv --log-file gpurun_out/r02k_ew.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ew rc=$?"
python tools/ew_ncu.py gpurun_out/r02k_ew.csv > gpurun_out/r02k_ew_summary.jsonl; cat gpurun_out/r02k_ew_summary.jsonl
