# every BASELINE config on one B200 (bench lines for profiles/), plus the workload variants
mkdir -p gpurun_out/bench_all
run() { name=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/bench_all/$name.json 2> gpurun_out/bench_all/$name.err; echo "$name rc=$?" >> gpurun_out/bench_all/status.txt; }
run config3 --config config3
run config3_reference --config config3 --impl reference --steps 5 --warmup 1
run config2 --config config2
run config2_reference --config config2 --impl reference --steps 5 --warmup 1
run config4 --config config4
run config3_p5 --config config3_p5 --no-cpu-baseline
run config3_dc100 --config config3_dc100 --no-cpu-baseline
run config5 --config config5 --no-cpu-baseline --steps 10
