mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_period.py tests/test_gpu_wide.py -x -q > gpurun_out/period_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/period_test.log
tail -4 gpurun_out/period_test.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_period -c 1 -o gpurun_out/ncu_C4_period python bench.py --config C4 --hops 512 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/ncu_C4.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_C4.log
