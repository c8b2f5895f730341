tail -1 /tmp/gpurun_q.txt; tail -2 gpurun_out/gputest_q.log
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print("ms/step", round(d['ms_per_step'], 4), "value", round(d['value']))
print(json.dumps({k: round(v, 4) for k, v in d['stages_ms'].items()}))
PY
tail -25 gpurun_out/timeline_q.log
python tools/launch_summary.py gpurun_out/launches_q.csv "$1" | head -${2:-25}
