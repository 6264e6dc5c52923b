"""Sustained DFMA throughput with board power and SM clock sampled beside it (GPU).

Usage: python tools/fp64_power.py [--seconds 8] [--out gpurun_out/fp64_power.json]
Runs tools/fp64_peak <seconds> (DFMA launches back to back) while sampling nvidia-smi every 100 ms. The
config-5 bound needs this: if the FP64 pipe ALONE draws the power cap at its peak (as a plain copy does at
6.5 TB/s, profiles/r02_power_probe.txt), a step that needs both cannot overlap them at peak under the cap.
"""
import argparse
import json
import os
import subprocess
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=8.0)
    ap.add_argument("--out", default="gpurun_out/fp64_power.json")
    args = ap.parse_args()
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            out = subprocess.run(["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits",
                                  "-i", "0"], capture_output=True, text=True).stdout
            try:
                pw, sm = (float(v) for v in out.strip().split(","))
                samples.append((pw, sm))
            except ValueError:
                pass
            time.sleep(0.1)

    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    res = subprocess.run([os.path.join(ROOT, "tools", "fp64_peak"), str(args.seconds)], capture_output=True, text=True)
    stop.set()
    th.join()
    d = json.loads(res.stdout.strip().splitlines()[-1])
    s = samples[len(samples) // 4:]
    med = lambda i: sorted(v[i] for v in s)[len(s) // 2] if s else None  # noqa: E731
    d.update({"power_w_median": med(0), "sm_mhz_median": med(1), "samples": len(samples)})
    print(json.dumps(d))
    if args.out:
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as fh:
            json.dump(d, fh)


if __name__ == "__main__":
    main()
