"""Top source lines of an ncu report by warp-stall samples and instructions
(cuda,sass source page).  Diagnostic only.

  python tools/ncu_source.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, f, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 6 and r[2] == "-":
        try:
            rows.append((int(r[4]), int(r[7]), f, int(r[0]), r[1][:90]))
        except ValueError:
            pass
tot_s = sum(x[0] for x in rows) or 1
tot_i = sum(x[1] for x in rows) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for s, i, fn, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  {fn}:{ln:<4d} {src}")
