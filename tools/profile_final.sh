# launch list + full captures of the top kernels of one warm config-3 step (profiles/)
mkdir -p gpurun_out
python tools/profile_step.py config3 > gpurun_out/plain_p.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_p.csv python tools/profile_step.py config3 > gpurun_out/ncu_p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"minmax2|tile_bits_kernel|pair_tiles|tile_words_t|border_kernel|child_init|cap_select|group_small" -c 8 -o gpurun_out/prof_p python tools/profile_step.py config3 > gpurun_out/ncu_p2.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_p2.log
