# every config's bench line on the final code (dev helper)
mkdir -p gpurun_out/bench_all4
for c in config3 config2 config4; do timeout 1200 python bench.py --config $c > gpurun_out/bench_all4/$c.json 2> gpurun_out/bench_all4/$c.err; echo "$c rc=$?" >> gpurun_out/bench_all4/status.txt; done
timeout 900 python bench.py --config config5 --no-cpu-baseline --steps 10 > gpurun_out/bench_all4/config5.json 2> gpurun_out/bench_all4/config5.err; echo "config5 rc=$?" >> gpurun_out/bench_all4/status.txt
for c in config3_p5 config3_dc100; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_all4/$c.json 2> gpurun_out/bench_all4/$c.err; echo "$c rc=$?" >> gpurun_out/bench_all4/status.txt; done
