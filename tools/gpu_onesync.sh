# one-sync emit: its parity tests, then an A/B of the step (one call vs two calls)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rows.py tests/test_gpu_parity.py -x -q -k "one_sync or determinism or end_to_end or child_parent or no_write or fused_render" > gpurun_out/onesync_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/onesync_tests.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-fused > gpurun_out/ab_one_$i.json 2> gpurun_out/ab_one_$i.err
timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-fused --two-call > gpurun_out/ab_two_$i.json 2> gpurun_out/ab_two_$i.err
done
