# copy latencies; one-hop kernel cluster size A/B (p) on C5 / C3
mkdir -p gpurun_out
python scripts/copy_lat.py > gpurun_out/aa_copy.txt 2>&1
for cfg in C5 C3; do for p in 2 4; do
  timeout 600 python bench.py --config $cfg --hops 300 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 200 --tune p=$p > gpurun_out/aa_${cfg}_p$p.json 2> gpurun_out/aa_${cfg}_p$p.err
done; done
cat gpurun_out/aa_copy.txt
