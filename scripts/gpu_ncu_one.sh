mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
K=${NCU_KERNEL:-hist_pass}; S=${NCU_SKIP:-3}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/prof_${K}_${S} python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-records ${BENCH_ARGS:---no-c5 --no-kfold --no-c2} > gpurun_out/ncu_${K}_${S}.log 2>&1; echo "ncu $K $S rc=$?"
