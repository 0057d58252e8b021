nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_bw scripts/l2_bw.cu && /tmp/l2_bw > gpurun_out/r2g_l2bw.jsonl 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2g_pytest.log 2>&1
tail -3 gpurun_out/r2g_pytest.log
python bench.py --config C3 > gpurun_out/r2g_bench_C3.json 2> gpurun_out/r2g_bench_C3.err
ncu --set full --clock-control none --import-source on -k regex:bank_mac -c 1 -o gpurun_out/r2g_ncu_C3 python bench.py --config C3 --hops 1000 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/r2g_ncu_C3.log 2>&1
