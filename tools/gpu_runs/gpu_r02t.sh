# r02t: candidate-list rebuild after the publication (pre-emptive below CL_LOW entries)
set -x
O=gpurun_out/r02t; mkdir -p $O
L=$PWD/paper_2202_12380_b200
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
for rep in 1 2; do
MPGABOR_LIB=$L/libmpgabor_head.so timeout 300 python tools/ab_run.py "head" C1,C2 f64 3 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "rbafter" C1,C2 f64 3 >> $O/ab.log 2>&1
done
MPGABOR_LIB=$L/libmpgabor_head.so timeout 300 python tools/ab_run.py "head" C3,C4 f64 1 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "rbafter" C3,C4 f64 1 >> $O/ab.log 2>&1
timeout 300 python tools/prof_multi.py C2,C4 100000 > $O/prof.log 2>&1
echo done
