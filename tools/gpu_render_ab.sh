# render binning: its tests, the render-dependent parity tests, per-view render time, a launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_render.py -x -q > gpurun_out/render_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/render_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "render or end_to_end or drop_in or determinism" > gpurun_out/render_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/render_parity.log
timeout 300 python tools/render_ab.py config3 16 > gpurun_out/render_ab.log 2>&1
python tools/profile_render.py config3 4 > gpurun_out/prof_render_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_render.csv python tools/profile_render.py config3 4 > gpurun_out/ncu_render.log 2>&1
