# one round trip: parity tests, bench, ncu of the top kernels
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
bash scripts/gpu_tests.sh
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?"; tail -c 1800 gpurun_out/bench_c4.log
for spec in "ingest_kernel 0" "hist_pass 0" "hist_pass 8" "select_kernel 0"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_$1_$2 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_$1_$2.log 2>&1; echo "ncu $1 $2 rc=$?"
done
