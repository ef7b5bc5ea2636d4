# full-size parity (C4, C5 against the oracle goldens) + synccheck rerun + degenerate general path
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; tail -15 gpurun_out/pytest_fullsize.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "degenerate" > gpurun_out/pytest_degen.log 2>&1; echo "degen rc=$?"; tail -3 gpurun_out/pytest_degen.log
SEL="c1_full or c2_three_regions or c3_full or degenerate_cases_general or random_small_tables or select_synthetic_complete_tree or select_deep_irregular"
for tool in synccheck racecheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 50 --log-file gpurun_out/sanitize_$tool.log \
    python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL" > gpurun_out/sanitize_$tool.out 2>&1
  echo "$tool rc=$?"; tail -1 gpurun_out/sanitize_$tool.out; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize_$tool.log | sort | uniq -c
done
