mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bank_mac -c 1 -o gpurun_out/ncu_C5_bank python bench.py --hops 1733 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/ncu_C5_bank.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bank_mac -c 1 -o gpurun_out/ncu_C3_bank python bench.py --config C3 --hops 1000 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/ncu_C3_bank.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C5.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
