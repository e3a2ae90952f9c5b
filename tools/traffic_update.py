"""Refresh profiles/traffic.json from `ncu --set full` raw CSV exports
(dram__bytes_read.sum + dram__bytes_write.sum per launch).  Diagnostic tooling.

  python tools/traffic_update.py KEY RAW_CSV NOTE [KEY RAW_CSV NOTE ...]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles", "traffic.json")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def dram(path):
    rows = list(csv.reader(open(path)))
    hdr, units, v = rows[0], rows[1], rows[2]
    d = {h: (x, u) for h, x, u in zip(hdr, v, units)}

    def get(k):
        x, u = d[k]
        return float(x.replace(",", "")) * SCALE.get(u, 1)
    return get("dram__bytes_read.sum"), get("dram__bytes_write.sum")


def main(args):
    t = json.load(open(P)) if os.path.exists(P) else {}
    for key, path, note in zip(args[0::3], args[1::3], args[2::3]):
        r, w = dram(path)
        t[key] = dict(bytes=int(r + w), read=int(r), write=int(w),
                      source=os.path.relpath(path, ROOT), note=note)
    json.dump(t, open(P, "w"), indent=1)
    print(json.dumps(t, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
