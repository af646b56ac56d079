set -x
O=gpurun_out/r02x; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "dgt or full_run or tiny" > $O/pytest_gpu.log 2>&1
timeout 300 python tools/dgt_time.py C4 f64 > $O/dgt_c4.log 2>&1
timeout 300 python tools/dgt_time.py C2 f64 > $O/dgt_c2.log 2>&1
timeout 300 python tools/ab_run.py "stcs" C2,C4 f64 1 >> $O/ab.log 2>&1
echo done
