#!/usr/bin/env python
"""Measure the FP64 (DFMA) roofline denominator on this GPU and write it, with
the nvidia-smi clock log of the run, to profiles/fp64_peak.json (committed;
bench.py reads its peak from there).

  python tools/fp64_peak.py [--out profiles/fp64_peak.json]

Method (tools/microbench/fp64_peak.cu): DFMA chains on all SMs in six shapes;
burst = best of 10 launches per shape (CUDA events), sustained = the best shape
back to back for >= 4 s. The clock-derived figure 148 SM x 64 DFMA/clk x 2 flop
x max SM clock is recorded beside them.
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402

SRC = os.path.join(ROOT, "tools", "microbench", "fp64_peak.cu")
BIN = os.path.join(ROOT, "tools", "microbench", "fp64_peak")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "fp64_peak.json"))
    a = ap.parse_args()
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-o", BIN, SRC], check=True)
    clk = ClockSampler(0)
    clk.start()
    time.sleep(0.5)
    t0 = time.time()
    r = subprocess.run([BIN], capture_output=True, text=True, check=True)
    wall = time.time() - t0
    c = clk.stop()
    res = json.loads(r.stdout)
    # every raw sample line, for the record (sm MHz, max MHz, W, reasons...)
    res["clock_log"] = clk.lines
    res["clocks"] = c
    sm_max = c.get("sm_max_mhz") or 1965.0
    res["clock_derived_tflops"] = res["sms"] * 64 * 2 * sm_max * 1e6 / 1e12
    loaded = []
    for ln in clk.lines:
        parts = [p.strip() for p in ln.split(",")]
        try:
            if float(parts[2]) > 400:
                loaded.append(float(parts[0]))
        except (ValueError, IndexError):
            pass
    res["sm_mhz_median_under_load"] = sorted(loaded)[len(loaded) // 2] if loaded else None
    res["wall_s"] = wall
    res["how"] = ("tools/microbench/fp64_peak.cu: DFMA chains (8/16/32 per thread) on all SMs, six shapes; "
                  "burst = best of 10 launches (CUDA events), sustained = best shape back to back >= 4 s; "
                  "nvidia-smi -lms 200 during the run")
    res["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "clock_log"}))


if __name__ == "__main__":
    main()
