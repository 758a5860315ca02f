"""Summarise ncu captures into profiles/: key metrics of the full-set capture of the render
kernel (-> profiles/ncu_summary.json, read by bench.py for roofline.traffic) and the per-launch
share table of a launch-list capture.

  python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <tag>
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_per_sm",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "simt_efficiency_threads",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "smsp__inst_executed.sum": "warp_instructions",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
        "s": 1e3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    return rows[0], rows[1], rows[2:]


def main():
    rep, launches, tag = sys.argv[1:4]
    hdr, units, rows = raw(rep)
    kernels = {}
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].split("::")[-1]
        d = {}
        for m, k in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u in UNIT and k in ("duration", "dram_read", "dram_write"):
                    v *= UNIT[u]  # ms for time, bytes for dram
                d[k] = v
        d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    stalls[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(r[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        d["stall_pct"] = {k: round(v / tot * 100, 1)
                          for k, v in sorted(stalls.items(), key=lambda t: -t[1])[:8]}
        kernels[short] = d
    # launch list: per-kernel share of device time
    share = {}
    with open(launches) as f:
        lines = f.read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    lrows = list(csv.reader(lines[start:]))
    lh = lrows[0]
    for r in lrows[1:]:
        if r[lh.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[lh.index("Kernel Name")].split("(")[0].split("::")[-1]
        ns = float(r[lh.index("Metric Value")].replace(",", ""))
        s = share.setdefault(name, [0, 0.0])
        s[0] += 1
        s[1] += ns / 1e6
    total = sum(v[1] for v in share.values()) or 1
    launch_table = {k: {"launches": v[0], "ms": round(v[1], 3), "share_pct": round(v[1] / total * 100, 2)}
                    for k, v in sorted(share.items(), key=lambda t: -t[1][1])}
    # NCU_SOURCE / NCU_LAUNCHES_SOURCE: the names the capture and launch list are committed under
    out = {"tag": tag, "source": os.environ.get("NCU_SOURCE", os.path.basename(rep)),
           "workload": os.environ.get("NCU_WORKLOAD", "C3"),
           "kernels": kernels,
           "launch_list": {"source": os.environ.get("NCU_LAUNCHES_SOURCE", os.path.basename(launches)),
                           "kernels": launch_table}}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
        json.dump(out, f, indent=1)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
