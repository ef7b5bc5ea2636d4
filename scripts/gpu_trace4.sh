mkdir -p gpurun_out
BA="--no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy"
timeout 600 python bench.py $BA > gpurun_out/bp_c4.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bp_c4.log').read().strip().splitlines()[-1]); print('C4', d['ms_per_step'], json.dumps(d.get('c3_train'))[:400])"
timeout 600 python bench.py --config C3 --steps 20 --warmup 3 $BA > gpurun_out/bp_c3.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bp_c3.log').read().strip().splitlines()[-1]); print('C3', d['ms_per_step'], d['train_samples_per_s'])"
ADAPT_TRACE_HOST=2 timeout 600 python bench.py --steps 1 --warmup 1 $BA > gpurun_out/trace_c4.log 2>&1; grep "\[adapt\]" gpurun_out/trace_c4.log | tail -40
