mkdir -p gpurun_out
ADAPT_TRACE_HOST=2 timeout 300 python bench.py --steps 1 --warmup 2 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/trace3_full.log 2>&1; echo rc=$?
grep "\[adapt\]" gpurun_out/trace3_full.log | tail -30
