set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_band.py -x -q > gpurun_out/band_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/band_tests.log
tail -2 gpurun_out/band_tests.log
for v in 6 7 9 11; do timeout 600 python tools/c5_full.py --variant $v --reps 2 --out gpurun_out/c5_full_v$v.json > gpurun_out/c5_v$v.log 2>&1; python -c "
import json; d=json.load(open('gpurun_out/c5_full_v$v.json')); print('variant $v', d['ms_per_degree_step'], d['fp64_tflops'], d['fp64_frac_of_dfma_peak'], d['step_kernel'], d['clocks'])"; done
