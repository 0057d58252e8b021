# period tiles (C4): tests, then C4 bench with and without them
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_period.py tests/test_gpu_wide.py -x -q > gpurun_out/period_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/period_test.log
tail -15 gpurun_out/period_test.log
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --latency-hops 0 > gpurun_out/bench_C4_period.json 2> gpurun_out/bench_C4_period.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_C4_period.err
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --latency-hops 0 --no-cpu --no-e2e --tune wide_period=0 > gpurun_out/bench_C4_noperiod.json 2> gpurun_out/bench_C4_noperiod.err; echo "bench rc=$?"
