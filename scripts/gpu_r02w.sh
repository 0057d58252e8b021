mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"wide_forward_warp|bank_k5" -c 2 -o gpurun_out/ncu_C5_k1k5 python bench.py --hops 1733 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/ncu_C5_k1k5.log 2>&1; echo "ncu rc=$?"
