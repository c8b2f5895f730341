# end-of-round evidence on one B200 (dev helper): every BASELINE config, the
# step's launch list with DRAM bytes, the multi-rank functional check
mkdir -p gpurun_out
bash tools/bench_all.sh
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_d.csv python tools/profile_step.py config3 \
  > gpurun_out/ncu_d.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_d.log
ADPS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/multirank.json 2> gpurun_out/multirank.err
echo "multirank rc=$?" >> gpurun_out/multirank.err
