# one-chunk host calls on the engine stream + contiguous copies: latency legs, engine tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_bank_pass.py tests/test_gpu_configs.py -x -q > gpurun_out/z_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/z_tests.log
for cfg in C5 C3 C2 C4; do
  timeout 600 python bench.py --config $cfg --hops 1000 --steps 2 --warmup 3 --no-cpu --no-e2e --latency-hops 300 > gpurun_out/z_lat_${cfg}.json 2> gpurun_out/z_lat_${cfg}.err
done
tail -3 gpurun_out/z_tests.log
