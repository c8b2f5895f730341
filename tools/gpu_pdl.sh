# PDL: full GPU suite, then the step with and without programmatic dependent launch, and the render
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pdl_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pdl_tests.log
for r in 1 2 3; do
  for p in 1 0; do
    ADPS_PDL=$p timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-fused > gpurun_out/pdl_${p}_${r}.json 2>/dev/null
    python -c "
import json,sys
l=[x for x in open('gpurun_out/pdl_${p}_${r}.json') if x.startswith('{')]
d=json.loads(l[-1]); print('pdl=$p', round(d['ms_per_step'],4), 'render', round(d['render']['ms_per_view'],4))" >> gpurun_out/pdl_ab.log
  done
done
