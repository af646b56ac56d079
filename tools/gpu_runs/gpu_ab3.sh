# r02f: GPU suite (Stockham DGT, counter exchange), DGT timing, grid exchange / L2 prefetch A/B
set -x
O=gpurun_out/r02f; mkdir -p $O
L=paper_2202_12380_b200
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 300 python tools/dgt_time.py C4 f64 > $O/dgt_c4.log 2>&1
timeout 300 python tools/dgt_time.py C2 f64 > $O/dgt_c2.log 2>&1
timeout 300 python tools/ab_run.py "counter_pf" C3,C4 f64 2 >> $O/ab_gx.log 2>&1
MPGABOR_L2PF=0 timeout 300 python tools/ab_run.py "counter_nopf" C3,C4 f64 2 >> $O/ab_gx.log 2>&1
MPGABOR_L2PF=0 MPGABOR_LIB=$PWD/$L/libmpgabor_stamps.so timeout 300 python tools/ab_run.py "stamps_nopf" C3,C4 f64 2 >> $O/ab_gx.log 2>&1
timeout 300 python tools/prof_multi.py C4 100000 > $O/prof_c4.log 2>&1
MPGABOR_L2PF=0 timeout 300 python tools/prof_multi.py C4 100000 > $O/prof_c4_nopf.log 2>&1
echo done
