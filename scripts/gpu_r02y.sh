# entry-grouped one-hop kernel: parity, latency A/B (C5, C3), ncu of the C5 hop kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_bank_pass.py -x -q > gpurun_out/y_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/y_tests.log
for cfg in C5 C3; do
  for o in 1 0; do
    timeout 600 python bench.py --config $cfg --hops 2000 --steps 2 --warmup 3 --no-cpu --no-e2e --latency-hops 300 --tune entry_order=$o > gpurun_out/y_lat_${cfg}_o$o.json 2> gpurun_out/y_lat_${cfg}_o$o.err
  done
done
timeout 900 ncu --set full --clock-control none -k regex:tvolap_hop_kernel -s 10 -c 1 -o gpurun_out/y_hop_C5 -f python bench.py --config C5 --hops 64 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 30 > gpurun_out/y_ncu_C5.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:tvolap_hop_kernel -s 10 -c 1 -o gpurun_out/y_hop_C3 -f python bench.py --config C3 --hops 64 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 30 > gpurun_out/y_ncu_C3.log 2>&1
tail -3 gpurun_out/y_tests.log
