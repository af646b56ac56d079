set -x
O=gpurun_out/r02am; mkdir -p $O
timeout 900 python tools/bench_batch.py r02am C2,C1 > $O/batch.log 2>&1
timeout 900 python tools/bench_resets.py r02am > $O/resets.log 2>&1
cp profiles/r02am_* $O/ 2>/dev/null
echo done
