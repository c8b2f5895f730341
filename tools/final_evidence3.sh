# final refresh on the final code (dev helper): bench lines, launch list with DRAM bytes, full ncu captures
mkdir -p gpurun_out/bench_all3
for c in config3 config2 config4; do timeout 1200 python bench.py --config $c > gpurun_out/bench_all3/$c.json 2> gpurun_out/bench_all3/$c.err; echo "$c rc=$?" >> gpurun_out/bench_all3/status.txt; done
timeout 900 python bench.py --config config5 --no-cpu-baseline --steps 10 > gpurun_out/bench_all3/config5.json 2> gpurun_out/bench_all3/config5.err; echo "config5 rc=$?" >> gpurun_out/bench_all3/status.txt
for c in config3_p5 config3_dc100; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_all3/$c.json 2> gpurun_out/bench_all3/$c.err; echo "$c rc=$?" >> gpurun_out/bench_all3/status.txt; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_f.csv python tools/profile_step.py config3 \
  > gpurun_out/ncu_f.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_f.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"minmax2|tile_bits_kernel|pair_tiles|tile_words_t|border_kernel|child_init|cap_huge|group_small" -c 8 -o gpurun_out/prof_f python tools/profile_step.py config3 > gpurun_out/ncu_f2.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/ncu_f2.log
