"""Summarise ncu reports into profiles/ (run in the build container).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [more.ncu-rep ...] --tag r01 \
        [--launches gpurun_out/launches.csv]

Writes profiles/<tag>_<kernel>.json (key counters per launch) and updates
profiles/traffic.json ({kernel: dram read+write bytes per launch}) which
bench.py reports as roofline.traffic.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum.per_second",
    "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tma.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in ("Kernel Name", "ID") or any(h == k or h.endswith("." + k) or
                                                 re.fullmatch(r"(\w+\.)*" + re.escape(k), h)
                                                 for k in KEYS):
                d[h] = (r[i], units[i])
        res.append(d)
    return res


def short(name):
    name = re.sub(r"^void\s+", "", name.strip())
    name = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    m = re.match(r"(?:[\w:]*::)?(\w+)", name)
    base = m.group(1) if m else name.split("(")[0]
    if "<" in name.split("(")[0]:
        targ = name.split("<", 1)[1].split(">")[0]
        if base == "route_tc_kernel":  # <kBF16, NC>: NC > 1 is K1m
            a = [x.strip() for x in targ.split(",")]
            return (base + ("_bf16" if a[0] in ("1", "true") else "_f16")
                    + ("_k1m" if len(a) > 1 and a[1] != "1" else ""))
        if base == "route_tcs_kernel":  # <kBF16, NC>: NC > 1 is the chain tail
            return base + ("_tail" if targ.split(",")[-1].strip() not in ("1",) else "")
        if base == "lmhead_kernel":  # <kTerms>
            return base + "_" + targ.strip() + "term"
    return base


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    longest = {}
    for rep in a.reports:
        for d in raw(rep):
            k = short(d.get("Kernel Name", ("?", ""))[0])
            dur = num(d.get("gpu__time_duration.sum", ("0", ""))[0]) or 0.0
            if k in longest and longest[k] >= dur:
                continue  # several launches of one kernel: keep the longest
            longest[k] = dur
            summ = {h: {"value": v, "unit": u} for h, (v, u) in d.items()}
            rd = num(d.get("dram__bytes_read.sum", ("0", ""))[0])
            wr = num(d.get("dram__bytes_write.sum", ("0", ""))[0])
            ur = d.get("dram__bytes_read.sum", ("", ""))[1]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ur, 1)
            if rd is not None and wr is not None:
                uw = d.get("dram__bytes_write.sum", ("", ""))[1]
                sw = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(uw, 1)
                traffic[k] = rd * scale + wr * sw
            out = os.path.join(ROOT, "profiles", f"{a.tag}_{k}.json")
            with open(out, "w") as fh:
                json.dump({"report": os.path.basename(rep), "kernel": k, "metrics": summ}, fh,
                          indent=1)
            print("wrote", out)
    with open(tpath, "w") as fh:
        json.dump(traffic, fh, indent=1)
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        # ncu --csv --log-file: header row then one row per (launch, metric)
        hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hdr]
        ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"))
        agg = {}
        for r in rows[hdr + 1:]:
            if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
                continue
            v = num(r[vi])
            f = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                 "msecond": 1e3}.get(r[ui], 1.0)
            agg.setdefault(short(r[ki]), []).append(v * f)
        tot = sum(sum(v) for v in agg.values())
        lines = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v):.1f} | {sum(v)/len(v):.1f} | "
                         f"{100*sum(v)/tot:.1f}% |")
        out = os.path.join(ROOT, "profiles", f"{a.tag}_launches.md")
        with open(out, "w") as fh:
            fh.write(f"# ncu launch list ({os.path.basename(a.launches)}), "
                     "gpu__time_duration.sum, --clock-control none (cold, serialised)\n\n")
            fh.write("\n".join(lines) + "\n")
        print("wrote", out)


if __name__ == "__main__":
    main()
