#!/bin/bash
# A/B the default build against dev variants (tools/build_variant.py) on the GPU box.
# usage: tools/ab_bench.sh variant1 variant2 ...
for v in default "$@"; do
  if [ "$v" = default ]; then unset ADPS_LIB; else export ADPS_LIB=$PWD/paper_2605_06876_b200/_variants/libadps_$v.so; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-fused > gpurun_out/ab_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/ab_{sys.argv[1]}.log") if x.startswith("{")]
if not l:
    print(sys.argv[1], "FAILED"); sys.exit()
d = json.loads(l[-1]); s = d["stages_ms"]
print(f"{sys.argv[1]:10s} step={d['ms_per_step']:.3f}ms minmax={s['minmax']:.3f} tile_ccl={s['tile_ccl']:.3f} tile_gates={s['merge_tile_gates']:.3f} roof={d['roofline']['frac']:.3f} border={s["border_merge"]:.3f} cap={s["merge_cap"]:.3f} groups={s["merge_groups"]:.3f}")
PY
done
