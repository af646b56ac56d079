# r02at: walk-window size sweep (MPG_NE = 6 / 8 default / 10 / 12, B = 8), whole decompositions
set -x
O=gpurun_out/r02at; mkdir -p $O
L=$PWD/paper_2202_12380_b200
for r in 1 2; do
  timeout 300 python tools/ab_run.py "ne8" C1,C2 f64 3 >> $O/ab.log 2>&1
  for v in ne6 ne10 ne12; do
    MPGABOR_LIB=$L/libmpgabor_$v.so timeout 300 python tools/ab_run.py "$v" C1,C2 f64 3 >> $O/ab.log 2>&1
  done
done
timeout 300 python tools/ab_run.py "ne8" C3,C4 f64 1 >> $O/ab.log 2>&1
for v in ne6 ne10 ne12; do
  MPGABOR_LIB=$L/libmpgabor_$v.so timeout 300 python tools/ab_run.py "$v" C3,C4 f64 1 >> $O/ab.log 2>&1
done
echo done
