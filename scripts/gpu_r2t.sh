out=gpurun_out; mkdir -p $out; f=$out/r2_sanitizers.txt
echo "# compute-sanitizer over scripts/sanitize.py (every kernel family, exact reductions incl. direct-limb / nonfinite paths, stream set, flops sweep, GMRES cycle), round 2" > $f
for t in memcheck racecheck synccheck; do
  echo "== $t" >> $f
  timeout 900 compute-sanitizer --tool $t python scripts/sanitize.py 2>&1 | grep -E "sanitize run done|ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Race|hazard" | head -20 >> $f
done
echo "" >> $f
echo "# peer-memory communicator (exact digit-post allreduce), 2 processes on cuda:0 under memcheck: scripts/peer_sanitize.py" >> $f
for r in 0 1; do
  MASTER_ADDR=127.0.0.1 MASTER_PORT=29533 RANK=$r WORLD_SIZE=2 LBK_PEER_TIMEOUT=600 timeout 900 \
    compute-sanitizer --tool memcheck python scripts/peer_sanitize.py > $out/r2t_peer$r.log 2>&1 &
done
wait
for r in 0 1; do grep -E "^rank|ERROR SUMMARY" $out/r2t_peer$r.log | tr '\n' ' ' >> $f; echo >> $f; done
cat $f
