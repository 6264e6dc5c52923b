set -u
mkdir -p gpurun_out
timeout 3000 python tools/solve_config.py c4w --json gpurun_out/solve_c4w.json > gpurun_out/solve_c4w.txt 2>&1; echo "c4w rc=$?"
head -3 gpurun_out/solve_c4w.txt
timeout 4800 python tools/solve_complex.py c3 --json gpurun_out/solve_c3.json > gpurun_out/solve_c3.txt 2>&1; echo "c3 rc=$?"
head -4 gpurun_out/solve_c3.txt | cut -c1-400
