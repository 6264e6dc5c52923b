set -u
mkdir -p gpurun_out
run() { timeout 600 python tools/c5_full.py --n 1000000 --degree 6 --variant $1 --out gpurun_out/c5_tmp.json > gpurun_out/c5_tmp.log 2>&1; python -c "
import json; d=json.load(open('gpurun_out/c5_tmp.json')); print('variant $1:', d['ms_per_degree_step'], d['fp64_tflops'], d['fp64_frac_of_dfma_peak'], d['clocks']['sm_mhz'], d['clocks']['power_w_median'])"; }
for v in 6 9 12 13 14; do run $v; done
for v in 12 13; do
timeout 900 ncu --metrics l1tex__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none -k regex:cheb_band_kernel -s 2 -c 1 python tools/c5_full.py --n 600000 --degree 4 --reps 1 --variant $v --out '' 2>&1 | grep -E "cheb_band_kernel|l1tex|gpu__time|lts__t|dram__|fp64" | cut -c1-150
done
