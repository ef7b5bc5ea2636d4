mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_c4.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ingest_kernel -c 1 -o gpurun_out/prof_ingest python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_ingest.log 2>&1; echo "ncu ingest rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_pass -s 3 -c 1 -o gpurun_out/prof_hist python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_hist.log 2>&1; echo "ncu hist rc=$?"
ls -la gpurun_out
