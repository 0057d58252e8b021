mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -3 gpurun_out/gputest.log
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_period -c 1 -o gpurun_out/ncu_C4_period6 python bench.py --config C4 --hops 512 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/ncu_C4.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_C4.csv python bench.py --config C4 --hops 1024 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/ncu_launch_C4.log 2>&1; echo "launch rc=$?"
