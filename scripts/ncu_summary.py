#!/usr/bin/env python
"""Summarise ncu captures brought back in gpurun_out/ into profiles/.

    python scripts/ncu_summary.py ROUND rep1.ncu-rep[=WORKLOAD:stage] ... [--launches a.csv ...]
    (a rep holding several kernels: rep=W:stage1@substr1;W:stage2@substr2 — the
    first key whose kernel-name substring matches is used)

For every --set full capture: the kernel's duration, DRAM bytes (the
`traffic` of bench.py's roofline: dram__bytes_read.sum + dram__bytes_write.sum
per launch), DRAM / SM / tensor-pipe utilisation, occupancy and registers.
For every launch list (--metrics gpu__time_duration.sum): per-kernel mean
duration and share of the GPU time (cold-cache, serialised: compare shares).
Writes profiles/<ROUND>_ncu_summary.md and merges the traffic into
profiles/traffic.json keyed "WORKLOAD:stage".
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
    "lts__t_sectors_srcunit_tex_op_read.sum",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6}


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = (v[i], u[i])
        res.append(d)
    return res


def num(x):
    v, unit = x
    return float(v.replace(",", "")) * SCALE.get(unit, 1)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue   # launch lists with DRAM bytes as well: the durations only
        name = re.sub(r"\(.*", "", r[ki])
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1))
    return agg


def main():
    rnd = sys.argv[1]
    reps, lists, mode = [], [], None
    for a in sys.argv[2:]:
        if a == "--launches":
            mode = "l"
            continue
        (lists if mode == "l" else reps).append(a)
    md = [f"# ncu summary, round {rnd}", "",
          "Captured with `ncu --set full --clock-control none --import-source on -k regex:<kernel> -s <n> -c <k>` "
          "on one B200 (gpurun); the recipe is the scripts/profile_*.sh / scripts/round_*.sh named in DESIGN.md.  "
          "Times are one cold-cache replayed launch (ncu's clock, often power-capped below 1965 MHz).", ""]
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for spec in reps:
        rep, _, keyspec = spec.partition("=")
        for d in raw(rep):
            key = keyspec
            if "@" in keyspec:
                key = ""
                for part in keyspec.split(";"):
                    k, _, sub = part.partition("@")
                    if sub in d["kernel"]:
                        key = k
                        break
            md.append(f"## `{d['kernel'][:120]}`  ({os.path.basename(rep)}{', ' + key if key else ''})")
            for k in KEYS:
                if k in d:
                    md.append(f"- {k}: {d[k][0]} {d[k][1]}")
            rb, wb = num(d["dram__bytes_read.sum"]), num(d["dram__bytes_write.sum"])
            md.append(f"- **DRAM traffic per launch: {(rb + wb) / 1e9:.4f} GB** "
                      f"(read {rb / 1e9:.4f} + write {wb / 1e9:.4f})")
            md.append("")
            if key:
                traffic[key] = {"GB": round((rb + wb) / 1e9, 4), "read_GB": round(rb / 1e9, 4),
                                "write_GB": round(wb / 1e9, 4), "source": f"profiles/{rnd}_ncu_summary.md"}
    for path in lists:
        agg = launches(path)
        tot = sum(sum(v) for v in agg.values())
        md += [f"## launch list `{os.path.basename(path)}` (gpu__time_duration.sum, serialised)", "",
               "| kernel | launches | mean us | share |", "|---|---|---|---|"]
        for k, v in agg.items():
            md.append(f"| `{k[:90]}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v) / tot * 100:.1f}% |")
        md.append("")
    open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
