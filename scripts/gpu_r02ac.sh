# deferred selection upload: full GPU suite, latency legs C5 / C3
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ac_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ac_tests.log
for cfg in C5 C3; do
  timeout 600 python bench.py --config $cfg --hops 300 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 300 > gpurun_out/ac_${cfg}.json 2> gpurun_out/ac_${cfg}.err
done
tail -2 gpurun_out/ac_tests.log
