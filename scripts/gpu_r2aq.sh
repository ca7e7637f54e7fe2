out=gpurun_out; mkdir -p $out; f=$out/r2aq_sanitizers.txt
echo "# compute-sanitizer over scripts/sanitize.py (every kernel family, exact reductions incl. direct-limb / nonfinite paths, stream set, flops sweep, GMRES cycle; CG/BiCGSTAB with the split p-update pass), round 2 final" > $f
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> $f
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize.py 2>&1 | grep -E "run done|SUMMARY" >> $f
done
cat $f
