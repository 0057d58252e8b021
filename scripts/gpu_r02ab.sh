# pinned selection staging: engine tests, latency legs C5 / C3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_bank_pass.py tests/test_gpu_edge.py -x -q > gpurun_out/ab_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_tests.log
for cfg in C5 C3; do
  timeout 600 python bench.py --config $cfg --hops 300 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 300 > gpurun_out/ab_${cfg}.json 2> gpurun_out/ab_${cfg}.err
done
tail -2 gpurun_out/ab_tests.log
