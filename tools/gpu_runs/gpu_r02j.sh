# r02j: same-box A/B: HEAD library vs node-histogram rebuild vs rank-count rebuild
set -x
O=gpurun_out/r02j; mkdir -p $O
L=$PWD/paper_2202_12380_b200
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv >> $O/smi.txt
for rep in 1 2; do
  MPGABOR_LIB=$L/libmpgabor_head.so timeout 300 python tools/ab_run.py "head" C1,C2 f64 3 >> $O/ab.log 2>&1
  timeout 300 python tools/ab_run.py "hist" C1,C2 f64 3 >> $O/ab.log 2>&1
  MPGABOR_LIB=$L/libmpgabor_rank.so timeout 300 python tools/ab_run.py "rank" C1,C2 f64 3 >> $O/ab.log 2>&1
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv >> $O/smi.txt
timeout 300 python tools/prof_multi.py C2 100000 > $O/prof_c2.log 2>&1
timeout 300 python tools/prof_multi.py C4 100000 > $O/prof_c4.log 2>&1
MPGABOR_LIB=$L/libmpgabor_head.so timeout 300 python tools/ab_run.py "head" C3,C4 f64 1 >> $O/ab.log 2>&1
timeout 300 python tools/ab_run.py "hist" C3,C4 f64 1 >> $O/ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "multi or grid or fulllength or batch or tiny or tie" > $O/pytest_gpu.log 2>&1
echo done
