# compute-sanitizer, ONE tool per gpurun call (tools/sanitize.sh memcheck|racecheck|synccheck|initcheck)
# on the smoke step and on one config-2 step (renders resident, as the bench)
tool=$1
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize/${tool}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/sanitize/${tool}_smoke.log
timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/profile_step.py config2 > gpurun_out/sanitize/${tool}_config2.log 2>&1
echo "config2 rc=$?" >> gpurun_out/sanitize/${tool}_config2.log
