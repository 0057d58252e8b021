mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_period -c 1 -o gpurun_out/ncu_C4_period3 python bench.py --config C4 --hops 512 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/ncu_C4.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_mac -c 1 -o gpurun_out/ncu_C2_wide python bench.py --config C2 --hops 1024 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/ncu_C2.log 2>&1; echo "ncu rc=$?"
