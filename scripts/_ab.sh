timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2h_pytest.log 2>&1
tail -3 gpurun_out/r2h_pytest.log
python scripts/bank_pass_ab.py > gpurun_out/r2h_ab_q.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_launches_C3.csv python bench.py --config C3 --hops 1733 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/r2h_ncu.log 2>&1
