"""Print an ncu --csv launch list (gpu__time_duration.sum) in launch order: short kernel name, grid, us."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = 0.0
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", d["Kernel Name"])
    m = re.search(r"ntt_phase_kernel<(\d+), \(?\w*\)?(\w+), \(?\w*\)?(\w+)", d["Kernel Name"])
    if m:
        name = f"ntt<{m.group(1)},{'inv' if m.group(2) in ('true', '1') else 'fwd'},{'col' if m.group(3) in ('true', '1') else 'row'}>"
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    v = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
    tot += v
    print(f"{name[:48]:48s} {d.get('Grid Size', ''):>16s} {d.get('Block Size', ''):>12s} {v:9.2f}")
print(f"total {tot:.1f} us")
