# build tuning variants of libadapt.so into .variants/<name>/ (copies of the
# package + bench + synth); usage: bash scripts/make_variants.sh "name:DEFS" ...
set -e
cd /root/repo
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  d=.variants/$name; rm -rf $d; mkdir -p $d
  cp -r bench.py synth include paper_2303_08873_b200 $d/
  rm -f $d/paper_2303_08873_b200/libadapt.so
  (cd $d && ADAPT_NVCC_DEFS="$defs" python paper_2303_08873_b200/build.py --force > /dev/null)
  echo "built $name ($defs)"
done
