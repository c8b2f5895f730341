mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -k "merge or step or scale or determinism or sharded" > gpurun_out/merge_tests.log 2>&1; echo "rc=$?" >> gpurun_out/merge_tests.log
for i in 1 2 3; do timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-fused > gpurun_out/ab_m_$i.json 2>/dev/null; done
python tools/profile_step.py config3 > gpurun_out/plain_q.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_q.csv python tools/profile_step.py config3 > gpurun_out/ncu_q.log 2>&1
