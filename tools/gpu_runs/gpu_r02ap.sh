# r02ap: DGT with the signal range staged by a TMA bulk copy -- parity, A/B times
set -x
O=gpurun_out/r02ap; mkdir -p $O
L=$PWD/paper_2202_12380_b200
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dgt or C4 or C3" > $O/pytest_dgt.log 2>&1
for i in 1 2; do
for c in C4 C2; do
  timeout 300 python tools/dgt_time.py $c f64 > $O/dgt_${c}_stage_$i.log 2>&1
  MPGABOR_LIB=$L/libmpgabor_nostage.so timeout 300 python tools/dgt_time.py $c f64 > $O/dgt_${c}_nostage_$i.log 2>&1
  MPGABOR_LIB=$L/libmpgabor_minb3.so timeout 300 python tools/dgt_time.py $c f64 > $O/dgt_${c}_minb3_$i.log 2>&1
done
done
timeout 300 python tools/dgt_time.py C4 f32 > $O/dgt_C4_f32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgt_ct -s 0 -c 1 -o $O/ncu_dgt_ct_m128 python tools/dgt_time.py C4 f64 > $O/ncu_dgt.log 2>&1
ncu -i $O/ncu_dgt_ct_m128.ncu-rep --page source --csv > $O/dgt_ct_src.csv 2>&1
ncu -i $O/ncu_dgt_ct_m128.ncu-rep --page raw --csv > $O/dgt_ct_raw.csv 2>&1
echo done
