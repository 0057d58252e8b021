mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bench_launch.py -x -q > gpurun_out/launch_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/launch_test.log
tail -30 gpurun_out/launch_test.log
