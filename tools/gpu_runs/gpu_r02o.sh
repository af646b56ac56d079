# r02o: speculative list-head geometry (GPU suite; A/B on/off; profile)
set -x
O=gpurun_out/r02o; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
for rep in 1 2; do
MPGABOR_SPECGEO=0 timeout 300 python tools/ab_run.py "spec0" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
MPGABOR_SPECGEO=1 timeout 300 python tools/ab_run.py "spec1" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
done
timeout 300 python tools/prof_multi.py C2 100000 > $O/prof_c2.log 2>&1
echo done
