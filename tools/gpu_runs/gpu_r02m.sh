# r02m: walk changes (pick positions in registers, branch-free E chain)
set -x
O=gpurun_out/r02m; mkdir -p $O
L=$PWD/paper_2202_12380_b200
for rep in 1 2; do
for v in head walk2 walk2nobf; do
MPGABOR_LIB=$L/libmpgabor_$v.so timeout 300 python tools/ab_run.py "$v" C1,C2 f64 3 >> $O/ab.log 2>&1
done
done
MPGABOR_LIB=$L/libmpgabor_walk2.so timeout 300 python tools/prof_multi.py C2 100000 > $O/prof_c2.log 2>&1
MPGABOR_LIB=$L/libmpgabor_walk2.so timeout 300 python tools/ab_run.py "walk2" C3,C4 f64 1 >> $O/ab.log 2>&1
echo done
