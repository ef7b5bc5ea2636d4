# the driver-style bench (default flags) + clocks + launch list of one step
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
nproc > gpurun_out/host_cores.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host_cores.txt
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -c 4000 gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"; tail -c 1500 gpurun_out/bench_reference.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
