"""Bucket the NTT phase launches of an ncu --csv launch list (gpu__time_duration.sum)
by limb count (grid.y): time share and butterfly rate per bucket against the
measured lazy-Shoup peak (profiles/int_peak.json, 870.5 Gbfly/s).  N = 2^16,
LOGM stages per phase, N/2 butterflies per stage per limb."""
import collections
import csv
import re
import sys

PEAK = 870.5e9
N = 1 << int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 16
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
b = collections.defaultdict(lambda: [0.0, 0, 0.0])  # time us, launches, butterflies
tot_all = 0.0
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    v = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
    tot_all += v
    m = re.search(r"ntt_phase_kernel<(\d+)", d["Kernel Name"])
    if not m:
        continue
    logm = int(m.group(1))
    gy = int(re.findall(r"\d+", d["Grid Size"])[1])
    lo = 1
    while lo * 2 <= gy:
        lo *= 2
    key = f"{lo:4d}-{2 * lo - 1:4d}"
    b[key][0] += v
    b[key][1] += 1
    b[key][2] += gy * (N // 2) * logm
tot = sum(x[0] for x in b.values())
print(f"all kernels {tot_all / 1000:.2f} ms; NTT phases {tot / 1000:.2f} ms "
      f"({100 * tot / max(tot_all, 1e-9):.1f} %), "
      f"{sum(x[2] for x in b.values()) / (tot * 1e-6) / PEAK:.3f} of peak")
for k in sorted(b):
    t, n, bf = b[k]
    print(f"  limbs {k}: {t / 1000:8.3f} ms ({100 * t / tot:5.1f} % of NTT)  n={n:5d}  "
          f"avg {t / n:6.2f} us  {bf / (t * 1e-6) / 1e9:6.1f} Gbfly/s = {bf / (t * 1e-6) / PEAK:.3f} of peak")
