"""Summarise ncu outputs into profiles/ (markdown + traffic.json for bench.py).

    python tools/ncu_summary.py launches <launches.csv> <out.md> [title]
    python tools/ncu_summary.py full <report.ncu-rep> <out.md> <workload-key> [title]

`launches` aggregates a `--metrics gpu__time_duration.sum` launch list per
kernel (count, mean, share of the listed device time). `full` extracts the
per-launch DRAM traffic, duration, throughput, occupancy and registers of a
`--set full` report and merges `traffic` (dram read + write bytes per launch)
into profiles/traffic.json under "<workload-key>:<kernel>".
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name: str) -> str:
    n = name.split("(")[0]
    for junk in ("pactk::", "<unnamed>::", "unnamed>::", "(anonymous namespace)::"):
        n = n.replace(junk, "")
    n = n.replace("void ", "").replace("(bool)", "").replace("(int)", "")
    return n.strip()


def launches(csv_path, out_md, title):
    rows = list(csv.reader(open(csv_path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[short(r[ki])].append(float(r[vi].replace(",", "")) / 1000.0)
    total = sum(sum(v) for v in agg.values())
    lines = [f"# {title}", "", f"source: `{os.path.basename(csv_path)}` (ncu --metrics gpu__time_duration.sum "
             "--clock-control none; cold-cache, serialised: compare shares, not absolutes)", "",
             "| kernel | launches | mean us | total us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.2f} | {sum(v):.1f} | {100*sum(v)/total:.1f}% |")
    open(out_md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_instr"),
]


def full(rep, out_md, key, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    per = defaultdict(list)
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        d = {}
        for m, nm in WANT:
            if m in h:
                try:
                    d[nm] = float(r[h.index(m)].replace(",", ""))
                except ValueError:
                    d[nm] = None
        per[short(r[ki])].append(d)
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    lines = [f"# {title}", "", f"source: `{os.path.basename(rep)}` (ncu --set full --clock-control none; "
             "per-launch means; units: ns, bytes, %)", "",
             "| kernel | n | duration us | DRAM read MB | DRAM write MB | DRAM % peak | SM % | warps active % | regs | grid x block |",
             "|---|---:|---:|---:|---:|---:|---:|---:|---:|---|"]
    for k, lst in per.items():
        def m(f):
            xs = [x[f] for x in lst if x.get(f) is not None]
            return sum(xs) / len(xs) if xs else float("nan")
        lines.append(f"| `{k}` | {len(lst)} | {m('duration')/1000:.2f} | {m('dram_read')/1e6:.1f} | "
                     f"{m('dram_write')/1e6:.1f} | {m('dram_pct'):.1f} | {m('sm_pct'):.1f} | "
                     f"{m('occupancy_pct'):.1f} | {m('regs'):.0f} | {m('grid'):.0f} x {m('block'):.0f} |")
        traffic[f"{key}:{k}"] = int(m("dram_read") + m("dram_write"))
    json.dump(traffic, open(tp, "w"), indent=1, sort_keys=True)
    open(out_md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "launch list")
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5] if len(sys.argv) > 5 else "ncu --set full")
