#!/usr/bin/env python
"""Refreshes the round-2 entries of profiles/traffic.json from the raw ncu captures (`ncu --page raw --csv`).
usage: python profiles/make_traffic.py [dir with r2_*_raw.csv, default profiles/]"""
import csv, json, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
src = sys.argv[1] if len(sys.argv) > 1 else HERE
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "%": 1.0}


def metric(path, name):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    i = hdr.index(name)
    return float(vals[i].replace(",", "")) * UNIT.get(units[i], 1.0)


ENTRIES = {"c2": "r2_c2_forward", "c3": "r2_c3_forward", "c3_gfd_fused": "r2_c3_fused_gfd", "c4": "r2_c4_forward",
           "c5": "r2_c5_forward"}
path = os.path.join(HERE, "traffic.json")
d = json.load(open(path))
for key, stem in ENTRIES.items():
    raw = os.path.join(src, stem + "_raw.csv")
    if not os.path.exists(raw):
        continue
    r, w = metric(raw, "dram__bytes_read.sum"), metric(raw, "dram__bytes_write.sum")
    d[key].update(dram_bytes_read=r, dram_bytes_write=w, dram_bytes_per_launch=r + w,
                  kernel_ms_under_ncu=metric(raw, "gpu__time_duration.sum"),
                  l2_hit_rate_pct=metric(raw, "lts__t_sector_hit_rate.pct"))
json.dump(d, open(path, "w"), indent=1)
for key in ENTRIES:
    print(key, {k: d[key][k] for k in ("dram_bytes_per_launch", "kernel_ms_under_ncu", "l2_hit_rate_pct")})
