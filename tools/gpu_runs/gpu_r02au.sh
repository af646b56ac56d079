# r02au: one 32-bin tile per work item (MPG_TPI32 = 1) against the default 2
set -x
O=gpurun_out/r02au; mkdir -p $O
L=$PWD/paper_2202_12380_b200
for r in 1 2; do
  timeout 300 python tools/ab_run.py "tpi2" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
  MPGABOR_LIB=$L/libmpgabor_tpi1.so timeout 300 python tools/ab_run.py "tpi1" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
done
echo done
