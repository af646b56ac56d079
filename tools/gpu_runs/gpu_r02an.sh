# r02an: smoke on the restored tree; DGT per-dictionary times and a source-level ncu capture
# of the C4 M=128 DGT launch; source-level capture of the C2 multi-selection kernel
set -x
O=gpurun_out/r02an; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 300 python tools/dgt_time.py C4 f64 > $O/dgt_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgt_stockham -s 0 -c 1 -o $O/ncu_dgt_c4_m128 python tools/dgt_time.py C4 f64 > $O/ncu_dgt.log 2>&1
ncu -i $O/ncu_dgt_c4_m128.ncu-rep --page source --csv --print-source cuda,sass > $O/dgt_src.csv 2>&1
ncu -i $O/ncu_dgt_c4_m128.ncu-rep --page source --csv > $O/dgt_src_cuda.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mp_multi -s 1 -c 1 -o $O/ncu_c2_multi python tools/ncu_one.py C2 f64 > $O/ncu_c2.log 2>&1
ncu -i $O/ncu_c2_multi.ncu-rep --page source --csv > $O/c2_src_cuda.csv 2>&1
echo done
