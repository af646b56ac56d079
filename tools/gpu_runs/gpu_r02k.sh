# r02k: bisect of the C1/C2 regression (same box)
set -x
O=gpurun_out/r02k; mkdir -p $O
L=$PWD/paper_2202_12380_b200
for v in head r0 r1 r2 r3; do
  MPGABOR_LIB=$L/libmpgabor_$v.so timeout 300 python tools/ab_run.py "$v" C1,C2 f64 3 >> $O/ab.log 2>&1
done
echo done
