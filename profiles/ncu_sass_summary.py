#!/usr/bin/env python
"""Summarises `ncu -i X.ncu-rep --page source --csv --print-source sass` for one kernel launch:
instruction mix by opcode, lane utilisation, and warp-stall sampling totals."""
import collections
import csv
import sys


def main(path, launch=0, top=25):
    rows = list(csv.reader(open(path)))
    # split into launches at "Kernel Name" rows
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    starts.append(len(rows))
    blk = rows[starts[launch]:starts[launch + 1]]
    print(blk[0][1])
    hdr = blk[1]
    col = {h: i for i, h in enumerate(hdr)}
    body = [r for r in blk[2:] if len(r) == len(hdr)]
    I = lambda r, k: float(r[col[k]] or 0)
    tot_inst = sum(I(r, "Instructions Executed") for r in body)
    tot_thr = sum(I(r, "Thread Instructions Executed") for r in body)
    print(f"SASS lines {len(body)}  warp instructions {tot_inst:.4g}  thread instructions {tot_thr:.4g}  "
          f"avg active lanes {tot_thr / tot_inst:.2f}")
    mix = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    for r in body:
        toks = r[col["Source"]].split()
        op = next((t for t in toks if not t.startswith("@")), "?").split(".")[0]
        mix[op][0] += I(r, "Instructions Executed")
        mix[op][1] += I(r, "Thread Instructions Executed")
        mix[op][2] += I(r, "# Samples")
    tot_samp = sum(v[2] for v in mix.values())
    print("opcode        warp-inst%  lanes  samples%")
    for op, v in sorted(mix.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{op:12s} {100 * v[0] / tot_inst:8.2f}  {v[1] / max(v[0], 1):6.2f}  {100 * v[2] / max(tot_samp, 1):7.2f}")
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    st = {h: sum(I(r, h) for r in body) for h in stalls}
    tot = sum(st.values())
    print("stall reasons (all samples):")
    for h, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]:
        print(f"  {h:28s} {100 * v / max(tot, 1):6.2f}%")
    print("hottest SASS lines by samples:")
    for r in sorted(body, key=lambda r: -I(r, "# Samples"))[:top]:
        print(f"  {I(r, '# Samples'):8.0f}  lanes {I(r, 'Avg. Threads Executed'):5.1f}  {r[col['Source']][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
