# r02bd: the picked atoms written by warp 1 after its item bases (default build) against warp 0 after the energy chain (aw0)
set -x
O=gpurun_out/r02bd; mkdir -p $O
L=$PWD/paper_2202_12380_b200
timeout 900 python -m pytest tests -m gpu -x -q -k "multi or batch or tiny or tie or full_run or launch_conf or reset or pedantic" > $O/pytest_sel.log 2>&1
for r in 1 2; do
  timeout 300 python tools/ab_run.py "atomsw1" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
  MPGABOR_LIB=$L/libmpgabor_aw0.so timeout 300 python tools/ab_run.py "aw0" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
done
timeout 300 python tools/ab_run.py "atomsw1" C3,C4 f64 1 >> $O/ab.log 2>&1
MPGABOR_LIB=$L/libmpgabor_aw0.so timeout 300 python tools/ab_run.py "aw0" C3,C4 f64 1 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "atomsw1" C1,C2 f32 3 >> $O/ab.log 2>&1
MPGABOR_LIB=$L/libmpgabor_aw0.so timeout 300 python tools/ab_run.py "aw0" C1,C2 f32 3 >> $O/ab.log 2>&1
echo done
