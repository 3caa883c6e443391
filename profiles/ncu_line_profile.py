#!/usr/bin/env python
"""Joins ncu's per-SASS-instruction counters with nvdisasm line info to attribute executed thread
instructions and stall samples to source lines (inlined header code included).
usage: ncu_line_profile.py <sass.csv from `ncu --page source --csv --print-source sass`> <nvdisasm -g -c output> <kernel substring>"""
import collections
import csv
import re
import sys


def main(sass_csv, dis, kernel, top=45):
    # 1. offsets -> (file, line) from nvdisasm
    line_of = {}
    cur = None
    in_k = False
    for ln in open(dis):
        if ln.startswith("//-") and ".text." in ln:
            in_k = kernel in ln
        if not in_k:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            line_of[int(m.group(1), 16)] = (cur, m.group(2))
    # 2. ncu rows in order
    rows = list(csv.reader(open(sass_csv)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    blk = rows[starts[0]:starts[1]]
    hdr = blk[1]
    col = {h: i for i, h in enumerate(hdr)}
    body = [r for r in blk[2:] if len(r) == len(hdr)]
    base = int(body[0][col["Address"]], 16) if body[0][col["Address"]].startswith("0x") else int(body[0][col["Address"]])
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    tot_t = tot_s = 0.0
    for r in body:
        a = r[col["Address"]]
        off = (int(a, 16) if a.startswith("0x") else int(a)) - base
        src = line_of.get(off, (None, ""))[0]
        t = float(r[col["Thread Instructions Executed"]] or 0)
        w = float(r[col["Instructions Executed"]] or 0)
        s = float(r[col["# Samples"]] or 0)
        agg[src][0] += t; agg[src][1] += s; agg[src][2] += w
        tot_t += t; tot_s += s
    print(f"total thread instr {tot_t:.4g} samples {tot_s:.0f}")
    print(" thread-inst%  samples%  lanes  file:line")
    for src, (t, s, w) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"   {100*t/tot_t:8.2f}  {100*s/tot_s:7.2f}  {t/max(w,1):5.1f}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
