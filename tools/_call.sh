set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json; cut -c1-200 gpurun_out/bench_ref.json
timeout 1500 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
grep '"metric"' gpurun_out/bench_full.log | tail -1 > gpurun_out/bench_full.json
python - <<'P'
import json
d=json.load(open('gpurun_out/bench_full.json'))
print(d['value'], d['roofline']['frac'], d['roofline']['launch_ms'], d['e2e']['value'], d['clocks'], d['cpu_baseline']['value'])
for k,v in d['configs'].items(): print(k, v['step_launch_ms'], v.get('frac_of_hbm_peak'), v.get('frac_of_fp64_peak'), v.get('frac_of_serial_bound'), v.get('overlap_bound_ms'))
P
