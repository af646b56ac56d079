# r02i: GPU suite, DGT timing (fold loads batched, padding written once), A/B, configs table with floors
set -x
O=gpurun_out/r02i; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 300 python tools/dgt_time.py C4 f64 > $O/dgt_c4.log 2>&1
timeout 300 python tools/dgt_time.py C2 f64 > $O/dgt_c2.log 2>&1
timeout 300 python tools/ab_run.py "r02i" C1,C2 f64 3 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "r02i" C3,C4 f64 1 >> $O/ab.log 2>&1
MPGABOR_L2PF=0 timeout 300 python tools/ab_run.py "r02i_nopf" C3,C4 f64 1 >> $O/ab.log 2>&1
echo done
