# compute-sanitizer memcheck / racecheck / synccheck over the C1-C3 parity tests
# (SURVEY §5 race detection): the hot kernels' mbarrier/TMA ingest, cp.async
# split tiles, warp-aggregated smem cursors and shared-memory histograms
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
SEL="c1_full or c2_three_regions or c3_full or degenerate_cases_general or random_small_tables or select_synthetic_complete_tree or select_deep_irregular"
# SAN_TAG=_2lvl with ADAPT_TWO_LEVEL=1: the same tests through the two-level
# schedule (TAG pass, tagged histograms, MOVE4)
T=${SAN_TAG:-}
for tool in ${SAN_TOOLS:-memcheck racecheck synccheck}; do
  timeout ${SAN_TIMEOUT:-1200} compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    --log-file gpurun_out/sanitize${T}_$tool.log \
    python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL" > gpurun_out/sanitize${T}_$tool.out 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitize${T}_$tool.out; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/sanitize${T}_$tool.log | sort | uniq -c | head
done
