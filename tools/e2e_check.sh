# e2e pipelining check on configs 3 and 5 (dev helper), 2 runs each
for r in 1 2; do for c in config3 config5; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-fused --steps 8 > gpurun_out/e2e_$c.json 2>/dev/null; python -c "
import json; l=[x for x in open('gpurun_out/e2e_$c.json') if x.startswith('{')]; d=json.loads(l[-1]); e=d['e2e']; print('$c', round(d['ms_per_step'],3), 'e2e', round(e['ms_per_step'],2), 'serial', round(e['serial_ms_per_step'],2))" >> gpurun_out/e2e_check.log; done; done
