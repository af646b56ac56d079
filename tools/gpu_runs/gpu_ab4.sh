# r02g: GPU suite (histogram rebuild), phase profiles with wait histogram, A/B vs r02f, DGT ncu
set -x
O=gpurun_out/r02g; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 300 python tools/prof_multi.py C2 100000 > $O/prof_c2.log 2>&1
timeout 300 python tools/prof_multi.py C4 100000 > $O/prof_c4.log 2>&1
timeout 300 python tools/ab_run.py "hist" C1,C2 f64 3 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "hist" C3,C4 f64 2 >> $O/ab.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgt_stockham -c 8 -o $O/ncu_dgt_c4 python tools/dgt_time.py C4 f64 > $O/ncu_dgt.log 2>&1
echo done
