set -x
O=gpurun_out/r02ai; mkdir -p $O
timeout 300 python tools/prof_multi.py C2,C3,C4 100000 > $O/prof.log 2>&1
echo done
