# r02bc: publication by the first warps, one 16-byte chunk per thread (default build) against warp 0 alone (pw0)
set -x
O=gpurun_out/r02bc; mkdir -p $O
L=$PWD/paper_2202_12380_b200
timeout 900 python -m pytest tests -m gpu -x -q -k "multi or batch or tiny or tie or full_run or launch_conf or reset or pedantic" > $O/pytest_sel.log 2>&1
for r in 1 2; do
  timeout 300 python tools/ab_run.py "pushw" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
  MPGABOR_LIB=$L/libmpgabor_pw0.so timeout 300 python tools/ab_run.py "pw0" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
done
timeout 300 python tools/ab_run.py "pushw" C3,C4 f64 1 >> $O/ab.log 2>&1
MPGABOR_LIB=$L/libmpgabor_pw0.so timeout 300 python tools/ab_run.py "pw0" C3,C4 f64 1 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "pushw" C1,C2 f32 3 >> $O/ab.log 2>&1
MPGABOR_LIB=$L/libmpgabor_pw0.so timeout 300 python tools/ab_run.py "pw0" C1,C2 f32 3 >> $O/ab.log 2>&1
echo done
