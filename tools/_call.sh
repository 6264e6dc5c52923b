set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lat2d.py -x -q > gpurun_out/lat2d_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/lat2d_tests.log
tail -3 gpurun_out/lat2d_tests.log
timeout 900 python tools/tune_step.py --config c3 --variants 2,12,13,14,15 --degree 80 --reps 3 2>&1 | tail -6
