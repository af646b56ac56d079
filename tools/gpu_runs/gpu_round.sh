set -x
mkdir -p gpurun_out/r02d
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02d/smi.txt
python -m pytest tests -m gpu -x -q > gpurun_out/r02d/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d/smoke.log 2>&1
python bench.py > gpurun_out/r02d/bench.json 2> gpurun_out/r02d/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02d/reference.json 2> gpurun_out/r02d/reference.err
timeout 900 python tools/bench_configs.py r02d > gpurun_out/r02d/configs.log 2>&1
cp profiles/r02d_* gpurun_out/r02d/ 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02d/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r02d/ncu_bench.log 2>&1
echo done
