#!/usr/bin/env python
"""profiles/r3_roofline_traffic.json from the ncu --set full capture made by
tools/ncu_traffic.sh (DRAM bytes per launch of bench.py's roofline kernel).

    python tools/traffic_json.py gpurun_out/traffic_full.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "traffic_full.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def num(d, key):
    return float(d[ix[key]].replace(",", "")) if key in ix and d[ix[key]] else 0.0


launches = []
for d in data:
    t = num(d, "gpu__time_duration.sum")
    unit_us = rows[1][ix["gpu__time_duration.sum"]]
    ms = t / 1e3 if unit_us in ("usecond", "us") else (t / 1e6 if unit_us in ("nsecond", "ns") else t)
    launches.append({"kernel": d[ix["Kernel Name"]].split("(")[0], "time_ms": ms,
                     "dram_read_bytes": num(d, "dram__bytes_read.sum") * (1e6 if rows[1][ix["dram__bytes_read.sum"]] == "Mbyte" else 1e3 if rows[1][ix["dram__bytes_read.sum"]] == "Kbyte" else 1),
                     "dram_write_bytes": num(d, "dram__bytes_write.sum") * (1e6 if rows[1][ix["dram__bytes_write.sum"]] == "Mbyte" else 1e3 if rows[1][ix["dram__bytes_write.sum"]] == "Kbyte" else 1),
                     "l2_hit_pct": num(d, "lts__t_sector_hit_rate.pct")})
main = [l for l in launches if "combine" not in l["kernel"]]
out = {"source": "ncu --set full --cache-control none --clock-control none, bench.py --steps 2 --warmup 3 "
                 "(tools/ncu_traffic.sh)",
       "launches": launches,
       # bench.py's roofline kernel (exact launch name); hub-combine launches
       # are listed but not averaged in
       "kernel": "k_csc_backward",
       "traffic_bytes_per_launch": sum(l["dram_read_bytes"] + l["dram_write_bytes"] for l in main)
       / max(len(main), 1)}
path = os.path.join(ROOT, "profiles", "r3_roofline_traffic.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
