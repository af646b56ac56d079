# r02h: two-level histogram rebuild; thread-count / items-in-flight variants
set -x
O=gpurun_out/r02h; mkdir -p $O
L=paper_2202_12380_b200
timeout 900 python -m pytest tests -m gpu -x -q -k "multi or grid or fulllength or batch or tiny or tie" > $O/pytest_gpu.log 2>&1
timeout 300 python tools/prof_multi.py C2 100000 > $O/prof_c2.log 2>&1
timeout 300 python tools/prof_multi.py C4 100000 > $O/prof_c4.log 2>&1
timeout 300 python tools/ab_run.py "hist2" C1,C2 f64 3 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "hist2" C3,C4 f64 1 >> $O/ab.log 2>&1
MPGABOR_LIB=$PWD/$L/libmpgabor_lb256if2.so timeout 300 python tools/ab_run.py "lb256if2" C1,C2 f64 3 0,256,0,0 >> $O/ab.log 2>&1
MPGABOR_LIB=$PWD/$L/libmpgabor_lb384if2.so timeout 300 python tools/ab_run.py "lb384if2" C1,C2 f64 3 0,384,0,0 >> $O/ab.log 2>&1
MPGABOR_LIB=$PWD/$L/libmpgabor_lb256if2.so timeout 300 python tools/ab_run.py "lb256if2" C3,C4 f64 1 0,256,0,0 >> $O/ab.log 2>&1
echo done
