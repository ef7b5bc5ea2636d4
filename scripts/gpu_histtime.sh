mkdir -p gpurun_out
ADAPT_HIST_TIMING=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/histtime.log 2>&1; echo rc=$?
grep hist-timing gpurun_out/histtime.log | tail -12
