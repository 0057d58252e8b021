# e2e pipeline chunk sweep (pinned host buffers) on C5 and C3
mkdir -p gpurun_out
for c in C5 C3; do for lg in 25 26 27; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --latency-hops 0 --no-cpu --tune pipe_log2=$lg > gpurun_out/e2e_${c}_$lg.json 2> gpurun_out/e2e_${c}_$lg.err
  python -c "
import json;d=json.load(open('gpurun_out/e2e_${c}_$lg.json'));print('$c pipe_log2=$lg value %.4g e2e %.4g'%(d['value'], d['e2e']['value']), 'e2e ms %.1f'%d['e2e']['ms_per_step'], 'dev ms %.1f'%d['ms_per_step'])"
done; done
