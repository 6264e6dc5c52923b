set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_band.py -x -q 2>&1 | tail -2
run() { ADP_BAND_SYNC=$2 timeout 600 python tools/c5_full.py --n 1000000 --degree 6 --variant $1 --out gpurun_out/c5_tmp.json > gpurun_out/c5_tmp.log 2>&1; python -c "
import json; d=json.load(open('gpurun_out/c5_tmp.json')); print('variant $1 sync $2:', d['ms_per_degree_step'], d['fp64_tflops'], d['fp64_frac_of_dfma_peak'], d['clocks']['sm_mhz'], d['clocks']['power_w_median'])"; }
for v in 6 7 9 11; do for s in 0 1; do run $v $s; done; done
