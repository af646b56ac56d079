# r02aq: DGT launch shape A/B (threads per CTA, resident CTAs, TMA staging on/off)
O=gpurun_out/r02aq; mkdir -p $O
L=$PWD/paper_2202_12380_b200
for i in 1 2; do
for v in base t128m4 t128m5 t256m3 t128m5ns t256m3ns; do
  lib=$L/libmpgabor_$v.so; [ $v = base ] && lib=$L/libmpgabor.so
  for c in C4 C2; do
    MPGABOR_LIB=$lib timeout 300 python tools/dgt_time.py $c f64 > $O/dgt_${c}_${v}_$i.log 2>&1
  done
done
done
echo done
