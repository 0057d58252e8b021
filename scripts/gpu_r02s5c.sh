# session 5: full GPU suite on the new bank-pass defaults (64-hop tiles, CTAs walk all tiles), launch list + ncu captures
python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/s5c_gputest.txt; cat gpurun_out/s5c_gputest.txt
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/s5c_bench_C5.json 2> gpurun_out/s5c_bench_C5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s5c_launches_C5.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/s5c_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bank_mac -c 1 -o gpurun_out/s5c_ncu_C5_bank python bench.py --hops 1733 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/s5c_ncu_C5_bank.log 2>&1; echo "ncu C5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bank_mac -c 1 -o gpurun_out/s5c_ncu_C3_bank python bench.py --config C3 --hops 1000 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/s5c_ncu_C3_bank.log 2>&1; echo "ncu C3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bank_k5 -c 1 -o gpurun_out/s5c_ncu_C5_k5 python bench.py --hops 1733 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/s5c_ncu_C5_k5.log 2>&1; echo "ncu k5 rc=$?"
ls -la gpurun_out/*.ncu-rep
