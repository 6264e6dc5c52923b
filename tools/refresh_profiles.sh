#!/usr/bin/env bash
# Re-measure the round's evidence on a B200 (run under gpurun from the repo root):
#   1. the default bench line (config 4 headline, N = 1) and the reference arm
#   2. the ncu launch list of a short bench command (per-launch times + DRAM bytes, cold / serialised)
#   3. one `ncu --set full` capture of a plane-sweep Step launch (config 4: the roofline's traffic figure)
#      and one of a band-block Step launch (config 5's structure at n = 6e5)
# Outputs land in gpurun_out/ (reports are removed after summarising: the copy-back limit is 64 MiB);
# copy the summaries into profiles/ (tools/launch_summary.py, tools/ncu_summary.py).
set -u
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_full.log 2>&1
grep '"metric"' gpurun_out/bench_full.log | tail -1 > gpurun_out/bench_full.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
SHORT="bench.py --degree 40 --steps 1 --warmup 3 --no-e2e --no-solve --no-cpu-baseline --no-secondary"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python $SHORT > gpurun_out/ncu_launches.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:cheb_sweep_kernel -s 20 -c 1 -f \
    -o gpurun_out/sweep_full python $SHORT > gpurun_out/ncu_sweep.log 2>&1
python tools/ncu_summary.py gpurun_out/sweep_full.ncu-rep > gpurun_out/sweep_ncu.txt 2>&1
rm -f gpurun_out/sweep_full.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:cheb_band_kernel -s 2 -c 1 -f \
    -o gpurun_out/band_full python tools/c5_full.py --n 600000 --degree 4 --reps 1 --out '' > gpurun_out/ncu_band.log 2>&1
python tools/ncu_summary.py gpurun_out/band_full.ncu-rep > gpurun_out/band_ncu.txt 2>&1
rm -f gpurun_out/band_full.ncu-rep
tail -3 gpurun_out/sweep_ncu.txt gpurun_out/band_ncu.txt
