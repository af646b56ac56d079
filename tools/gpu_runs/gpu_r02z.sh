set -x
O=gpurun_out/r02z; mkdir -p $O
timeout 300 python tools/prof_multi.py C2,C3,C4 100000 > $O/prof.log 2>&1
timeout 300 python tools/ab_run.py "scanctr" C2,C4 f64 1 >> $O/ab.log 2>&1
echo done
