# A/B variants x3 runs each (tools/ab_bench.sh form, step ms only)
for r in 1 2 3; do bash tools/ab_bench.sh "$@"; done > gpurun_out/ab3.log 2>&1
