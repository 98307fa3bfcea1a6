#!/usr/bin/env python
"""Capture the DRAM traffic of the bench's own blind-rotation launch with ncu
and write profiles/ncu_br_traffic.json (bench.py reports it as
roofline.traffic). Run on the GPU box, after the same bench command has exited
0 without ncu:

  python tools/ncu_traffic.py [--batch 131072] [--config 1] [--out profiles/ncu_br_traffic.json]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=131072)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--kernel", default="regex:blind_rotate_warp")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_br_traffic.json"))
    a = ap.parse_args()
    bench = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "0", "--no-cpu-baseline",
             "--no-e2e", "--batch", str(a.batch), "--config", str(a.config)]
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", a.kernel, "-c", "1", "--csv", *bench]
    r = subprocess.run(cmd, capture_output=True, text=True)
    rows = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    vals, kname = {}, None
    for row in csv.DictReader(io.StringIO("\n".join(rows))):
        name, unit, v = row.get("Metric Name"), row.get("Metric Unit"), row.get("Metric Value", "").replace(",", "")
        kname = row.get("Kernel Name", kname)
        if not name or not v:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(unit, 1.0)
        vals[name] = float(v) * scale
    if "dram__bytes_read.sum" not in vals:
        sys.stderr.write(r.stdout[-3000:] + r.stderr[-3000:])
        raise SystemExit("ncu produced no dram metrics")
    rec = {"kernel": kname, "batch": a.batch, "config": a.config,
           "dram_read_bytes": vals["dram__bytes_read.sum"], "dram_write_bytes": vals["dram__bytes_write.sum"],
           "duration_s": vals.get("gpu__time_duration.sum"),
           "command": " ".join(["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
                                "--clock-control", "none", "-k", a.kernel, "-c", "1",
                                "python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e",
                                "--batch", str(a.batch), "--config", str(a.config)]),
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    with open(a.out, "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
