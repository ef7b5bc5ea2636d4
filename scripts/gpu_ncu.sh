mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
K=${NCU_KERNEL:-hist_pass}
S=${NCU_SKIP:-0}
C=${NCU_COUNT:-1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -o gpurun_out/prof_${K}_${S} python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/ncu_${K}.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_${K}.log
