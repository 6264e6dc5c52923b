#!/usr/bin/env bash
# Re-measure the round's evidence on a B200 (run under gpurun from the repo root):
#   1. the default bench line (config 2, N = 1)
#   2. the ncu launch list of a short bench command (per-launch times + DRAM bytes, cold / serialised)
#   3. one `ncu --set full` capture of a fused-step launch (the roofline's traffic figure)
#   4. the reference arm (--impl reference) on a short run
# Outputs land in gpurun_out/; copy the summaries into profiles/ (tools/launch_summary.py, tools/ncu_summary.py).
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
grep '"metric"' gpurun_out/bench_full.log | tail -1 > gpurun_out/bench_full.json
SHORT="bench.py --degree 40 --steps 1 --warmup 3 --no-e2e --no-solve --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python $SHORT > gpurun_out/ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:cheb_lean_kernel -s 20 -c 1 \
    -o gpurun_out/step_full python $SHORT > gpurun_out/ncu_full.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
tail -1 gpurun_out/bench_ref.log
