# r02av: per-source-line instruction counts of the C2 multi-selection kernel
set -x
O=gpurun_out/r02av; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mp_multi -s 1 -c 1 -o $O/ncu_c2_multi python tools/ncu_one.py C2 f64 > $O/ncu_c2.log 2>&1
ncu -i $O/ncu_c2_multi.ncu-rep --page source --csv --print-source cuda > $O/src_cuda.csv 2>/dev/null
ncu -i $O/ncu_c2_multi.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ls -la $O
echo done
