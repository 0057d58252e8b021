# session 6: bank K5 partial-sum loop unrolled by 2 (8 loads in flight per thread instead of 4), same box, alternating builds
B="timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --latency-hops 0"
LIB=paper_2310_00319_b200/lib
for t in "C3 base" "C3 unroll" "C3 base" "C3 unroll" "C5 base" "C5 unroll" "C5 base" "C5 unroll"; do
  set -- $t
  cp $LIB/alt_$2.bin $LIB/libtvolap_b200.so
  $B --config $1 > gpurun_out/s6i.json 2> gpurun_out/s6i.err
  python -c "
import json
d=json.load(open('gpurun_out/s6i.json'))
print('$t', '%.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], d['clocks']['sm_mhz'])
"
done
cp $LIB/alt_unroll.bin $LIB/libtvolap_b200.so
timeout 300 python -m pytest tests/test_gpu_bank_pass.py -x -q 2>&1 | tail -2
