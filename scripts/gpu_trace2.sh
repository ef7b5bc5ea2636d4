mkdir -p gpurun_out
ADAPT_TRACE_HOST=2 timeout 300 python bench.py --rows 12500000 --steps 1 --warmup 2 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/trace2_proxy.log 2>&1; echo rc=$?
grep "host:" gpurun_out/trace2_proxy.log | tail -12
