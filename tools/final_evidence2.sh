# refresh after the cluster cap (dev helper): config3 bench lines, launch list
mkdir -p gpurun_out/bench_all2
for c in config3 config2 config4; do timeout 1200 python bench.py --config $c > gpurun_out/bench_all2/$c.json 2> gpurun_out/bench_all2/$c.err; echo "$c rc=$?" >> gpurun_out/bench_all2/status.txt; done
timeout 900 python bench.py --config config5 --no-cpu-baseline --steps 10 > gpurun_out/bench_all2/config5.json 2> gpurun_out/bench_all2/config5.err; echo "config5 rc=$?" >> gpurun_out/bench_all2/status.txt
for c in config3_p5 config3_dc100; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_all2/$c.json 2> gpurun_out/bench_all2/$c.err; echo "$c rc=$?" >> gpurun_out/bench_all2/status.txt; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_e.csv python tools/profile_step.py config3 \
  > gpurun_out/ncu_e.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_e.log
