#!/usr/bin/env python
"""Per-source-line instruction and stall-sample shares of one kernel in an ncu report
(captured with --import-source on, code built with -lineinfo).

  python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def lines(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = collections.defaultdict(lambda: [0, 0, ""])
    fname = hdr = lastline = None
    lastsrc = ""
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name",):
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        if r[0]:
            lastline, lastsrc = r[0], r[1]
        try:
            ie, st = int(r[7] or 0), int(r[4] or 0)
        except ValueError:
            continue
        a = agg[(fname, lastline)]
        a[0] += ie
        a[1] += st
        a[2] = lastsrc
    return agg


if __name__ == "__main__":
    agg = lines(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {ti}, stall samples {ts}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * v[0] / ti:5.1f}% inst {100 * v[1] / ts:5.1f}% stall {k[0]}:{k[1]} {v[2].strip()[:90]}")
