# r02n: GPU suite, DGT timing (twiddle powers, staged W^m), profile, A/B
set -x
O=gpurun_out/r02n; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 300 python tools/dgt_time.py C4 f64 > $O/dgt_c4.log 2>&1
timeout 300 python tools/dgt_time.py C2 f64 > $O/dgt_c2.log 2>&1
timeout 300 python tools/prof_multi.py C2 100000 > $O/prof_c2.log 2>&1
timeout 300 python tools/ab_run.py "cur" C1,C2 f64 3 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "cur" C3,C4 f64 1 >> $O/ab.log 2>&1
echo done
