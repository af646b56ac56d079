set -x
O=gpurun_out/r02w; mkdir -p $O
L=$PWD/paper_2202_12380_b200
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 300 python tools/dgt_time.py C4 f64 > $O/dgt_minb3.log 2>&1
MPGABOR_LIB=$L/libmpgabor_minb2.so timeout 300 python tools/dgt_time.py C4 f64 > $O/dgt_minb2.log 2>&1
timeout 300 python tools/ab_run.py "rank2" C1,C2 f64 3 >> $O/ab.log 2>&1
echo done
