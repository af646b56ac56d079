# r02bb: the round's item bases by warp 1 while warp 0 runs the energy chain (default build)
# against the single-warp form (sw0: -DMPG_SCAN_W1=0)
set -x
O=gpurun_out/r02bb; mkdir -p $O
L=$PWD/paper_2202_12380_b200
timeout 900 python -m pytest tests -m gpu -x -q -k "multi or batch or tiny or tie or full_run or launch_conf or reset or pedantic" > $O/pytest_sel.log 2>&1
for r in 1 2; do
  timeout 300 python tools/ab_run.py "w1scan" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
  MPGABOR_LIB=$L/libmpgabor_sw0.so timeout 300 python tools/ab_run.py "sw0" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
done
timeout 300 python tools/ab_run.py "w1scan" C3,C4 f64 1 >> $O/ab.log 2>&1
MPGABOR_LIB=$L/libmpgabor_sw0.so timeout 300 python tools/ab_run.py "sw0" C3,C4 f64 1 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "w1scan" C1,C2 f32 3 >> $O/ab.log 2>&1
MPGABOR_LIB=$L/libmpgabor_sw0.so timeout 300 python tools/ab_run.py "sw0" C1,C2 f32 3 >> $O/ab.log 2>&1
echo done
