# round evidence: tests, driver-style bench, reference arm, launch list, ncu full captures
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
bash scripts/gpu_tests.sh
bash scripts/gpu_bench_full.sh
for spec in partition_kernel:4 hist_kernel:4 label_bin:0 discover_kernel:0 select_kernel_c:0 split_kernel:10; do
  NCU_KERNEL=${spec%%:*} NCU_SKIP=${spec##*:} bash scripts/gpu_ncu_one.sh
done
# C5: the select launch over 1e9 vectors with the trained depth-16 tree (bottom blocks)
NCU_KERNEL=select_kernel_d NCU_SKIP=0 BENCH_ARGS="--no-kfold --no-c2" bash scripts/gpu_ncu_one.sh
mv gpurun_out/prof_select_kernel_d_0.ncu-rep gpurun_out/prof_select_kernel_c5.ncu-rep 2>/dev/null
# K-fold: the batched held-out evaluation and the multi-root histogram pass
NCU_KERNEL=kfold_eval_many NCU_SKIP=0 BENCH_ARGS="--no-c5" bash scripts/gpu_ncu_one.sh
ls gpurun_out
