set -x
O=gpurun_out/r02y; mkdir -p $O
L=$PWD/paper_2202_12380_b200
timeout 300 python tools/prof_multi.py C2,C4 100000 > $O/prof_main.log 2>&1
MPGABOR_LIB=$L/libmpgabor_unr1.so timeout 300 python tools/prof_multi.py C2,C4 100000 > $O/prof_unr1.log 2>&1
echo done
