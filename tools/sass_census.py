#!/usr/bin/env python
"""SASS instruction census of the production kernels (evidence for the tcgen05 / TMEM / TMA
claims): per kernel, the static count of the opcodes that prove the Blackwell paths.

  python tools/sass_census.py [out.json]      (reads paper_2311_02542_b200/lib/obj/*.o)
"""
import collections
import glob
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTCATOMSWS", "UBLKCP", "UTMALDG", "UTMASTG",
       "SYNCS", "USETMAXREG", "LDG", "STG", "LDS", "STS", "ATOMS", "BAR", "HFMA2", "HMUL2", "HADD2",
       "FFMA", "DFMA", "DMUL", "DADD", "MUFU", "F2I", "I2F", "SHFL", "VOTE", "CREDUX"]


def census(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    res, fn, c = {}, None, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if fn:
                res[fn] = c
            fn, c = m.group(1), collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m and fn:
            op = m.group(1)
            c["total"] += 1
            for k in OPS:
                if op == k:
                    c[k] += 1
    if fn:
        res[fn] = c
    return res


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "sass_census.json")
    data = {}
    for obj in sorted(glob.glob(os.path.join(ROOT, "paper_2311_02542_b200", "lib", "obj", "*.o"))):
        for fn, c in census(obj).items():
            data[f"{os.path.basename(obj)}:{fn}"] = {k: v for k, v in c.items() if v}
    json.dump({"source": "cuobjdump -sass paper_2311_02542_b200/lib/obj/*.o (sm_100a), static counts",
               "kernels": data}, open(out, "w"), indent=1)
    for k, v in data.items():
        if "render_ws" in k or "march" in k or "mlp_batch" in k:
            print(k[:90], {o: v.get(o, 0) for o in ("total", "UTCHMMA", "LDTM", "STTM", "UTCBAR", "UBLKCP", "SYNCS", "LDG")})


if __name__ == "__main__":
    main()
