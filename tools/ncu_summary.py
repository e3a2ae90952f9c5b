"""Summarise ncu captures (raw CSV pages) and a launch list into markdown.

  python tools/ncu_summary.py profiles/r01 > profiles/r01/SUMMARY.md
"""
import collections
import csv
import glob
import os
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst"),
    ("smsp__sass_average_branch_targets_threads_uniform.pct", "branch uniformity %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__occupancy_limit_registers", "CTA limit (regs)"),
    ("smsp__inst_executed.sum", "warp instructions"),
]
STALLS = "smsp__average_warps_issue_stalled_"


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for k, (name, _) in enumerate(zip(hdr, r)):
            d[name] = (r[k], units[k])
        out.append(d)
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1e-3)
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        tot[name] += v
        cnt[name] += 1
    return tot, cnt


def main(d):
    print(f"# ncu summary: {d}\n")
    for lf in sorted(glob.glob(os.path.join(d, "launches*.csv"))):
        tot, cnt = launches(lf)
        T = sum(tot.values())
        print(f"## Launch list `{os.path.basename(lf)}` (cold-cache, serialised; compare shares)\n")
        print("| kernel | launches | total ms | share | mean us |\n|---|---|---|---|---|")
        for k in sorted(tot, key=lambda k: -tot[k]):
            print(f"| `{k}` | {cnt[k]} | {tot[k] / 1e3:.3f} | {tot[k] / T:.3f} | {tot[k] / cnt[k]:.1f} |")
        print()
    for rf in sorted(glob.glob(os.path.join(d, "*_raw.csv"))):
        for row in raw(rf):
            name = row.get("Kernel Name", ("?", ""))[0]
            print(f"## `{name}` ({os.path.basename(rf)})\n")
            print("| metric | value |\n|---|---|")
            for k, label in KEYS:
                if k in row:
                    v, u = row[k]
                    print(f"| {label} (`{k}`) | {v} {u} |")
            st = []
            for k, (v, u) in row.items():
                if k.startswith(STALLS) and k.endswith("per_issue_active.ratio"):
                    try:
                        st.append((float(v), k[len(STALLS):].replace("_per_issue_active.ratio", "")))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            if st:
                print("| top stall reasons (cycles per issue) | " +
                      ", ".join(f"{n} {v:.2f}" for v, n in st[:5]) + " |")
            print()


if __name__ == "__main__":
    main(sys.argv[1])
