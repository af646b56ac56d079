# r02bf: debug build with device-side protocol and bounds checks (MPG_CHECKS) -- GPU suite + every loop variant
set -x
O=gpurun_out/r02bf; mkdir -p $O
L=$PWD/paper_2202_12380_b200
MPGABOR_LIB=$L/libmpgabor_checks.so timeout 1500 python -m pytest tests -m gpu -x -q > $O/checks_pytest_gpu.log 2>&1
MPGABOR_LIB=$L/libmpgabor_checks.so timeout 600 python tools/sanitize_target.py 300 > $O/checks_target.log 2>&1
MPGABOR_LIB=$L/libmpgabor_checks.so timeout 600 python tools/ab_run.py "checks" C2,C3,C4 f64 1 > $O/checks_full_runs.log 2>&1
echo done
