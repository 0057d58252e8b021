# round-2 config lines (C1-C4) on the current kernels
mkdir -p gpurun_out
for c in C4 C3 C2 C1; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
