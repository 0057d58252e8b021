mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_edge.py tests/test_gpu_bank_pass.py -x -q > gpurun_out/edge_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/edge_test.log
tail -3 gpurun_out/edge_test.log
for c in C5 C3; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --latency-hops 0 --no-cpu > gpurun_out/e2e_${c}_ramp2.json 2> gpurun_out/e2e_${c}_ramp2.err
  python -c "
import json;d=json.load(open('gpurun_out/e2e_${c}_ramp2.json'));print('$c value %.4g e2e %.4g'%(d['value'], d['e2e']['value']), 'e2e ms %.1f'%d['e2e']['ms_per_step'], 'dev ms %.1f'%d['ms_per_step'], 'same', d['e2e']['matches_device_path'])"
done
