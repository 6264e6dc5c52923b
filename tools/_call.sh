set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_dist.py tests/test_gpu_parity.py::test_gpu_bitwise_vs_reference_sources tests/test_gpu_sweep.py -x -q > gpurun_out/new_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/new_tests.log
tail -4 gpurun_out/new_tests.log
python __graft_entry__.py smoke 2>&1 | tail -2
echo "--- W evict-normal"; timeout 600 python tools/ld_probe.py --cases 1024:1024,926:928 2>&1 | tail -2
echo "--- W evict-last"; ADP_SWEEP_WLAST=1 timeout 600 python tools/ld_probe.py --cases 1024:1024,926:928 2>&1 | tail -2
echo "--- c2"; timeout 600 python tools/ld_probe.py --config c2 --cases 256:256,362:384 --degree 200 2>&1 | tail -2
ADP_SWEEP_WLAST=1 timeout 600 python tools/ld_probe.py --config c2 --cases 256:256,362:384 --degree 200 2>&1 | tail -2
