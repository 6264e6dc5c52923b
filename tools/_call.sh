set -u
mkdir -p gpurun_out
for v in 0 7; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cheb_band_kernel -s 2 -c 1 -f -o gpurun_out/band_v$v python tools/c5_full.py --n 600000 --degree 4 --reps 1 --variant $v --out '' > gpurun_out/ncu_band_v$v.log 2>&1; tail -2 gpurun_out/ncu_band_v$v.log | cut -c1-300
done
