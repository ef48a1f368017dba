"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and
an `ncu --set full` report into markdown tables for profiles/.

    python tools/ncu_summary.py --launches gpurun_out/X_launches.csv --rep gpurun_out/X.ncu-rep
"""
import argparse
import collections
import csv
import io
import re
import subprocess


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("gks::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        us = v / 1000.0 if unit == "nsecond" or unit == "ns" else (v if unit in ("usecond", "us") else v * 1000.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | total us | share | us/launch |", "|---|---|---|---|---|"]
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {name} | {n} | {us:.1f} | {100 * us / tot:.1f}% | {us / n:.2f} |")
    return "\n".join(out), tot


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 wavefronts %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("sm__inst_executed.sum", "warp instr"),
]


def rep_table(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[hdr.index("Kernel Name")]).replace("void ", "").replace("gks::", "")
        out.append(f"**{name}** (launch id {r[hdr.index('ID')]})")
        out.append("")
        out.append("| metric | value |")
        out.append("|---|---|")
        for k, label in KEYS:
            if k in hdr:
                out.append(f"| {label} (`{k}`) | {r[hdr.index(k)]} {units[hdr.index(k)]} |")
        stalls = []
        for i, h in enumerate(hdr):
            m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", h)
            if m and r[i]:
                stalls.append((float(r[i]), m.group(1)))
        stalls.sort(reverse=True)
        out.append("| top stalls (cycles per issue) | " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]) + " |")
        out.append("")
    return "\n".join(out)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--launches")
    p.add_argument("--rep")
    a = p.parse_args()
    if a.launches:
        t, tot = launch_table(a.launches)
        print(f"Launch list ({tot / 1000:.1f} ms total device time, cold-cache serialised):\n")
        print(t)
        print()
    if a.rep:
        print(rep_table(a.rep))


if __name__ == "__main__":
    main()
