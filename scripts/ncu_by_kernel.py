"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0.0, 0])
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"]
    name = re.sub(r"\(.*", "", name)
    m = re.search(r"ntt_phase_kernel<(\d+), \(?\w*\)?(\w+), \(?\w*\)?(\w+)", d["Kernel Name"])
    if m:
        inv = m.group(2) in ("true", "1")
        col = m.group(3) in ("true", "1")
        name = f"ntt<{m.group(1)},{'inv' if inv else 'fwd'},{'col' if col else 'row'}>"
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    v = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)  # -> us
    agg[name][0] += v
    agg[name][1] += 1
tot = sum(v[0] for v in agg.values())
print(f"total {tot / 1000:.2f} ms over {sum(v[1] for v in agg.values())} launches")
for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"  {k:40s} {t / 1000:8.3f} ms {100 * t / tot:5.1f}%  n={n:5d}  avg {t / n:7.2f} us")
