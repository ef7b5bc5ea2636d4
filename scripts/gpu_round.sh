# round evidence: tests, driver-style bench, reference arm, launch list, ncu full captures
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
bash scripts/gpu_tests.sh
bash scripts/gpu_bench_full.sh
for spec in partition_kernel:4 hist_kernel:4 label_bin:0 discover_kernel:0 select_kernel:0 split_kernel:10; do
  NCU_KERNEL=${spec%%:*} NCU_SKIP=${spec##*:} bash scripts/gpu_ncu_one.sh
done
ls gpurun_out
