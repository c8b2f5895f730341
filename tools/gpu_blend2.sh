mkdir -p gpurun_out
for b in 1 0 1 0; do ADPS_BLEND2=$b timeout 300 python tools/render_ab.py config3 16 2>&1 | sed "s/^/blend2=$b /" >> gpurun_out/blend2.log; done
ADPS_BLEND2=1 timeout 900 python -m pytest tests/test_gpu_render.py tests/test_gpu_rows.py -x -q -k "render or fused or binning or depth" > gpurun_out/blend2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/blend2_tests.log
