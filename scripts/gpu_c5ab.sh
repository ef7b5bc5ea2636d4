# select tests + C5 A/B (heap kernel vs previous deep kernel) + synccheck on the ingest
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "select or c1_full or c3_full or c4_slice" > gpurun_out/pytest_sel.log 2>&1; echo "sel tests rc=$?"; tail -2 gpurun_out/pytest_sel.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k c5 > gpurun_out/pytest_c5.log 2>&1; echo "c5 fullsize rc=$?"; tail -2 gpurun_out/pytest_c5.log
for v in new old; do
  if [ $v = old ]; then export ADAPT_SEL_D=1; else unset ADAPT_SEL_D; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-records --no-kfold --no-c2 --no-proxy > gpurun_out/bench_c5_$v.log 2>&1
  python -c "
import json;l=[x for x in open('gpurun_out/bench_c5_$v.log') if x.startswith('{')][-1];d=json.loads(l);c=d['select_c5']
print('$v', 'select C4 ms', d['phase_ms_per_step']['select'], 'C5 trained', c['trained']['ms_per_batch'], c['trained']['roofline']['frac'], 'complete', c['complete']['ms_per_batch'], c['complete']['roofline']['frac'])"
done
unset ADAPT_SEL_D
timeout 600 compute-sanitizer --tool synccheck --target-processes all --log-file gpurun_out/sanitize_synccheck.log python -m pytest tests/test_gpu_parity.py -q -x -k "c1_full or c2_three_regions or c3_full or degenerate_cases_general or random_small_tables or select_synthetic_complete_tree or select_deep_irregular" > gpurun_out/sanitize_synccheck.out 2>&1; echo "synccheck rc=$?"; tail -1 gpurun_out/sanitize_synccheck.out; grep "ERROR SUMMARY" gpurun_out/sanitize_synccheck.log
