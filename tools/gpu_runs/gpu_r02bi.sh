# r02bi: candidates per round (mpgabor_set_batch B = 3..8) on the grid configurations C3 / C4
set -x
O=gpurun_out/r02bi; mkdir -p $O
for b in 8 6 5 4 3; do
  timeout 300 python tools/ab_run.py "B$b" C4 f64 1 - $b >> $O/ab.log 2>&1
done
for b in 8 6 5 4; do
  timeout 300 python tools/ab_run.py "B$b" C3,C2 f64 2 - $b >> $O/ab.log 2>&1
done
echo done
