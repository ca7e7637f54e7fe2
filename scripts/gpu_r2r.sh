out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_solver.py -q -k "gmres" > $out/r2r.log 2>&1; echo "rc=$?" >> $out/r2r.log
tail -15 $out/r2r.log
