# ncu --set full of the streaming one-hop kernel (process(), one hop per call) for C5 and C3
mkdir -p gpurun_out
for c in C4 C2; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tvolap_hop_kernel -s 10 -c 1 -o gpurun_out/ncu_${c}_hop python bench.py --config $c --hops 64 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 30 > gpurun_out/ncu_${c}_hop.log 2>&1; echo "$c rc=$?"
done
