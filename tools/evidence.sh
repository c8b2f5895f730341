# GPU-box evidence run (dev helper): bench line, reference arm, launch list, top-4 ncu captures into gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/ev4_smi.txt
timeout 600 python bench.py > gpurun_out/ev4_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/ev4_bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/ev4_launches.csv python tools/profile_step.py config3 > gpurun_out/ev4_ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:minmax2_kernel|tile_bits_kernel|pair_tiles_kernel|tile_words_kernel" -c 4 -o gpurun_out/ev4_top python tools/profile_step.py --timing > gpurun_out/ev4_ncu_top.log 2>&1
ls -la gpurun_out
