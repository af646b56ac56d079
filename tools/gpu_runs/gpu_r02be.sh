# r02be: round-end measurement set on the final code (item bases on warp 1, multi-warp publication, DGT side streams):
# GPU tests, smoke, bench (+reference arm), per-config table, phase profiles, launch list, ncu captures, DGT times
set -x
T=r02be
O=gpurun_out/$T; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/reference.json 2> $O/reference.err
timeout 1500 python tools/bench_configs.py $T > $O/configs.log 2>&1
cp profiles/${T}_configs.* $O/ 2>/dev/null
timeout 300 python tools/prof_multi.py C1,C2,C3 100000 > $O/prof_multi.log 2>&1
timeout 300 python tools/prof_multi.py C4 100000 >> $O/prof_multi.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 > $O/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mp_multi -s 1 -c 1 -o $O/ncu_c2_multi python tools/ncu_one.py C2 f64 > $O/ncu_c2.log 2>&1
ncu -i $O/ncu_c2_multi.ncu-rep --page raw --csv > $O/ncu_full_c2_multi.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgt_ct -s 7 -c 1 -o $O/ncu_dgt_c4 python tools/dgt_time.py C4 f64 > $O/ncu_dgt.log 2>&1
ncu -i $O/ncu_dgt_c4.ncu-rep --page raw --csv > $O/ncu_full_dgt_c4.csv 2>/dev/null
timeout 300 python tools/dgt_time.py C4 f64 > $O/dgt_c4.log 2>&1
timeout 300 python tools/dgt_time.py C2 f64 > $O/dgt_c2.log 2>&1
echo done
