# bench every .variants/<name> on the same box, twice, interleaved
mkdir -p gpurun_out
for round in 1 2; do
  for d in .variants/*/; do
    v=$(basename $d)
    (cd $d && timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 > /root/repo/gpurun_out/var_${v}_$round.log 2>&1)
  done
done
echo variants done
