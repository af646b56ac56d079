# r02e: NE/BMAX A/B on C2/C3, L2-prefetch A/B on C4, C4 phase split, C2 ncu source capture
set -x
O=gpurun_out/r02e; mkdir -p $O
L=paper_2202_12380_b200
for v in "" _ne16 _ne16b8; do
  MPGABOR_LIB=$PWD/$L/libmpgabor$v.so timeout 300 python tools/ab_run.py "base$v" C2 f64 3 >> $O/ab_ne.log 2>&1
done
for v in "" _ne16 _ne16b8; do
  MPGABOR_LIB=$PWD/$L/libmpgabor$v.so timeout 300 python tools/ab_run.py "base$v" C1,C3 f64 2 >> $O/ab_ne.log 2>&1
done
for pf in 0 4 8; do
  MPGABOR_L2PF=$pf timeout 300 python tools/ab_run.py "l2pf$pf" C4 f64 2 >> $O/ab_l2pf.log 2>&1
done
timeout 300 python tools/prof_multi.py C4 100000 > $O/prof_c4.log 2>&1
MPGABOR_L2PF=0 timeout 300 python tools/prof_multi.py C4 100000 > $O/prof_c4_nopf.log 2>&1
timeout 300 python tools/prof_multi.py C2 100000 > $O/prof_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mp_multi -s 1 -c 1 -o $O/ncu_c2_multi python tools/ncu_one.py C2 f64 > $O/ncu_c2.log 2>&1
echo done
