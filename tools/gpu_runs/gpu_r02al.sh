set -x
O=gpurun_out/r02al; mkdir -p $O
timeout 600 python tools/ab_run.py "tw64" C4 f64 1 128,512,64,2 >> $O/ab.log 2>&1
timeout 600 python tools/ab_run.py "tw128" C4 f64 1 128,512,128,2 >> $O/ab.log 2>&1
timeout 600 python tools/ab_run.py "tw32" C4 f64 1 128,512,32,2 >> $O/ab.log 2>&1
timeout 600 python tools/ab_run.py "tw128" C3 f64 1 64,512,128,0 >> $O/ab.log 2>&1
echo done
