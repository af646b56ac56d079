# r02l: head vs current (regressions removed), DGT timing, GPU suite
set -x
O=gpurun_out/r02l; mkdir -p $O
L=$PWD/paper_2202_12380_b200
for rep in 1 2; do
MPGABOR_LIB=$L/libmpgabor_head.so timeout 300 python tools/ab_run.py "head" C1,C2 f64 3 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "cur" C1,C2 f64 3 >> $O/ab.log 2>&1
done
MPGABOR_LIB=$L/libmpgabor_head.so timeout 300 python tools/ab_run.py "head" C3,C4 f64 1 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "cur" C3,C4 f64 1 >> $O/ab.log 2>&1
timeout 300 python tools/dgt_time.py C4 f64 > $O/dgt_c4.log 2>&1
timeout 300 python tools/dgt_time.py C2 f64 > $O/dgt_c2.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
echo done
