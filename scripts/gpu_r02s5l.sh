# session 5: ncu of the ring kernel (C3)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hop_ring -s 10 -c 1 -o gpurun_out/s5l_ncu_C3_ring python bench.py --config C3 --hops 64 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 30 > gpurun_out/s5l_ncu.log 2>&1; echo "rc=$?"
