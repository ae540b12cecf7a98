set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_schedule_sim.py tests/test_train_gpu.py -q -x -k "streaming or executor_order or mlp_config_loss" > gpurun_out/r02m_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02m_tests.txt
timeout 900 python -m pytest tests/test_cnn_gpu.py tests/test_bench_parity_gpu.py -q -x -k "lenet or vgg16_b512_bench_config" > gpurun_out/r02m_cnn.txt 2>&1; echo "cnn rc=$?"; tail -3 gpurun_out/r02m_cnn.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:'im2col' --clock-control none --csv --log-file gpurun_out/r02m_ew.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ew rc=$?"
python tools/ew_ncu.py gpurun_out/r02m_ew.csv
