# r02ax: software-pipelined publication (default build) against the plain loop (pu0)
set -x
O=gpurun_out/r02ax; mkdir -p $O
L=$PWD/paper_2202_12380_b200
for r in 1 2 3; do
  timeout 300 python tools/ab_run.py "pipe" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
  MPGABOR_LIB=$L/libmpgabor_pu0.so timeout 300 python tools/ab_run.py "pu0" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
done
timeout 300 python tools/ab_run.py "pipe" C1,C2 f32 3 >> $O/ab.log 2>&1
MPGABOR_LIB=$L/libmpgabor_pu0.so timeout 300 python tools/ab_run.py "pu0" C1,C2 f32 3 >> $O/ab.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "multi or batch or tiny or tie or full_run" > $O/pytest_sel.log 2>&1
echo done
