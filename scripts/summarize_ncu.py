"""Summarise ncu outputs into profiles/ (committed evidence).

usage: python scripts/summarize_ncu.py launches <launches.csv> <out.json>
       python scripts/summarize_ncu.py report <prof.ncu-rep> <out.json>
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__occupancy_limit_registers",
        "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
        "launch__grid_size", "launch__block_size",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_wait_per_warp_active.pct"]


def launches(path, out):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        k = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        m = r[ix["Metric Name"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        agg.setdefault(k, {}).setdefault(m, []).append(v)
    res = {}
    for k, d in agg.items():
        res[k] = {m: sum(v) / len(v) for m, v in d.items()}
        res[k]["launches"] = len(d.get("gpu__time_duration.sum", []))
    tot = sum(v["gpu__time_duration.sum"] * v["launches"] for v in res.values())
    for v in res.values():
        v["share_of_time"] = v["gpu__time_duration.sum"] * v["launches"] / tot
    json.dump(res, open(out, "w"), indent=1)
    for k, v in res.items():
        print(f"{k:40s} n={v['launches']:3d} t={v['gpu__time_duration.sum']/1e3:9.1f} us "
              f"share={v['share_of_time']:.3f} dram={(v.get('dram__bytes_read.sum',0)+v.get('dram__bytes_write.sum',0))/1e9:.3f} GB")


def report(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = vals[i] + (f" {units[i]}" if units[i] else "")
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    for d in res:
        print(json.dumps(d, indent=1))


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2], sys.argv[3])
