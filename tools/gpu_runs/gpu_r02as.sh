# r02as: DGT fork/join over side streams (A/B against in-line launches), the new
# tiny-signal grid-mode tests, DGT parity, and a short bench
set -x
T=r02as
O=gpurun_out/$T; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "tiny or dgt or batch_equals or deterministic or decompose_host" > $O/pytest_sel.log 2>&1
for r in 1 2; do
  for s in 0 1; do
    MPGABOR_DGT_STREAMS=$s timeout 300 python tools/dgt_time.py C4 f64 > $O/dgt_C4_s${s}_$r.log 2>&1
    MPGABOR_DGT_STREAMS=$s timeout 300 python tools/dgt_time.py C2 f64 > $O/dgt_C2_s${s}_$r.log 2>&1
  done
done
MPGABOR_DGT_STREAMS=1 timeout 300 python tools/dgt_time.py C4 f32 > $O/dgt_C4_f32_s1.log 2>&1
MPGABOR_DGT_STREAMS=0 timeout 300 python tools/dgt_time.py C4 f32 > $O/dgt_C4_f32_s0.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
echo done
