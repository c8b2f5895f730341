# quick GPU iteration: parity tests of the step, a short bench, the host/GPU timeline and a launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rows.py -x -q > gpurun_out/gputest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_q.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 300 python tools/step_timeline.py config3 > gpurun_out/timeline_q.log 2>&1
python tools/profile_step.py config3 > gpurun_out/plain_q.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_q.csv python tools/profile_step.py config3 > gpurun_out/ncu_q.log 2>&1
