# r02bj: window ranking with 4 (default) / 8 / 16 lanes per published entry (cluster kernels)
set -x
O=gpurun_out/r02bj; mkdir -p $O
L=$PWD/paper_2202_12380_b200
for r in 1 2; do
  for v in rl4 rl8 rl16; do
    MPGABOR_LIB=$L/libmpgabor_$v.so timeout 300 python tools/ab_run.py "$v" C0,C1,C2 f64 3 >> $O/ab.log 2>&1
  done
done
for v in rl4 rl16; do
  MPGABOR_LIB=$L/libmpgabor_$v.so timeout 300 python tools/ab_run.py "$v" C1,C2 f32 3 >> $O/ab.log 2>&1
done
MPGABOR_LIB=$L/libmpgabor_rl16.so timeout 600 python -m pytest tests -m gpu -x -q -k "multi or batch or tiny or tie or full_run or launch_conf" > $O/pytest_rl16.log 2>&1
echo done
