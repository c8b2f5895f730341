# A/B on another config (dev helper): tools/ab_config.sh CONFIG variant...
cfg=$1; shift
for r in 1 2 3; do for v in default "$@"; do
  if [ "$v" = default ]; then unset ADPS_LIB; else export ADPS_LIB=$PWD/paper_2605_06876_b200/_variants/libadps_$v.so; fi
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-fused > gpurun_out/abc_$v.log 2>&1
  python -c "
import json; l=[x for x in open('gpurun_out/abc_$v.log') if x.startswith('{')]; d=json.loads(l[-1]); s=d['stages_ms']
print('$v', round(d['ms_per_step'],3), 'cap', round(s['merge_cap']*1000), 'groups', round(s['merge_groups']*1000))" >> gpurun_out/abc.log
done; done
