# session 6: ncu --set full of the C5 one-hop kernel on two-warp CTAs (64 threads)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tvolap_hop_kernel -s 10 -c 1 -o gpurun_out/s6e_hop_C5 -f python bench.py --config C5 --hops 64 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 30 > gpurun_out/s6e_ncu_C5.log 2>&1; echo ncu rc=$?
ls -la gpurun_out/s6e_hop_C5.ncu-rep
