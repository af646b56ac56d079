# r02p: list-target A/B on the grid configs (C3, C4) and C2
set -x
O=gpurun_out/r02p; mkdir -p $O
L=$PWD/paper_2202_12380_b200
timeout 300 python tools/ab_run.py "t48" C2,C3 f64 2 >> $O/ab.log 2>&1
for v in t32 t64 t96; do
MPGABOR_LIB=$L/libmpgabor_$v.so timeout 300 python tools/ab_run.py "$v" C2,C3 f64 2 >> $O/ab.log 2>&1
done
timeout 300 python tools/ab_run.py "t48" C4 f64 1 >> $O/ab.log 2>&1
for v in t64 t96; do
MPGABOR_LIB=$L/libmpgabor_$v.so timeout 300 python tools/ab_run.py "$v" C4 f64 1 >> $O/ab.log 2>&1
done
echo done
