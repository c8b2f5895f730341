# quick: step parity subset + bench x3 (step ms, roofline)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rows.py -x -q > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
rm -f gpurun_out/quick_ab.log
for i in 1 2 3; do timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-fused > gpurun_out/qab_$i.json 2>/dev/null; python -c "
import json; l=[x for x in open('gpurun_out/qab_$i.json') if x.startswith('{')]; d=json.loads(l[-1]); print(round(d['ms_per_step'],4), 'roof', round(d['roofline']['frac'],3), 'minmax_ms', round(d['stages_ms']['minmax'],4))" >> gpurun_out/quick_ab.log; done
