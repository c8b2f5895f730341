# one GPU iteration: the step's parity tests, an A/B of dev variants, a short bench with the fused variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rows.py -x -q > gpurun_out/gputest_i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_i.log
bash tools/ab_bench.sh "$@" > gpurun_out/ab_i.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err
