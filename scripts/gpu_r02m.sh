mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi_rank.py tests/test_gpu_engine.py -x -q > gpurun_out/mix_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/mix_test.log
tail -15 gpurun_out/mix_test.log
