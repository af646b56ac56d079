# r02ao: compile-time-size DGT kernel -- parity (both DGT paths), A/B times, full GPU suite
set -x
O=gpurun_out/r02ao; mkdir -p $O
L=$PWD/paper_2202_12380_b200
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k dgt > $O/pytest_dgt.log 2>&1
for c in C4 C2; do
  timeout 300 python tools/dgt_time.py $c f64 > $O/dgt_${c}_ct.log 2>&1
  MPGABOR_DGT_RT=1 timeout 300 python tools/dgt_time.py $c f64 > $O/dgt_${c}_rt.log 2>&1
  MPGABOR_LIB=$L/libmpgabor_minb3.so timeout 300 python tools/dgt_time.py $c f64 > $O/dgt_${c}_minb3.log 2>&1
done
timeout 300 python tools/dgt_time.py C4 f32 > $O/dgt_C4_f32_ct.log 2>&1
MPGABOR_DGT_RT=1 timeout 300 python tools/dgt_time.py C4 f32 > $O/dgt_C4_f32_rt.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgt_ct -s 0 -c 1 -o $O/ncu_dgt_ct_m128 python tools/dgt_time.py C4 f64 > $O/ncu_dgt.log 2>&1
ncu -i $O/ncu_dgt_ct_m128.ncu-rep --page source --csv > $O/dgt_ct_src.csv 2>&1
ncu -i $O/ncu_dgt_ct_m128.ncu-rep --page raw --csv > $O/dgt_ct_raw.csv 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
echo done
