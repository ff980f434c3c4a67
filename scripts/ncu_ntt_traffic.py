"""Per-launch DRAM traffic of the NTT phases in an ncu --set full report (raw page, units kept):
CSV rows (kernel, grid, duration us, DRAM read / write bytes, algorithmic bytes = 16 N per limb of
the launch's grid -- an upper bound where the set skips pass-through digit limbs, fmaheavy %,
issue %) and a JSON summary on the last line (means per launch) for bench.py's roofline.traffic."""
import csv
import json
import re
import subprocess
import sys

N = 1 << 16
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}


def val(r, name):
    v = r[col[name]].replace(",", "")
    return float(v) * SCALE.get(units[col[name]], 1) if v else 0.0


w = csv.writer(sys.stdout)
w.writerow(["kernel", "grid", "duration_us", "dram_read_bytes", "dram_write_bytes", "algorithmic_bytes",
            "fmaheavy_pct", "issue_active_pct", "warps_active_pct"])
tot = {"n": 0, "dur": 0.0, "dram": 0.0, "alg": 0.0}
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    if "ntt_phase_kernel" not in name:
        continue
    gy = int(re.findall(r"\d+", r[col["Grid Size"]])[1])
    dur = val(r, "gpu__time_duration.sum")
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    alg = gy * 16 * N
    w.writerow([re.sub(r"\(.*", "", name)[-40:], r[col["Grid Size"]], round(dur, 2), int(rd), int(wr), alg,
                r[col["sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"]],
                r[col["smsp__issue_active.avg.pct_of_peak_sustained_active"]],
                r[col["sm__warps_active.avg.pct_of_peak_sustained_active"]]])
    tot["n"] += 1
    tot["dur"] += dur
    tot["dram"] += rd + wr
    tot["alg"] += alg
n = max(1, tot["n"])
print(json.dumps({"ntt_launches": tot["n"], "mean_duration_us": round(tot["dur"] / n, 2),
                  "mean_dram_bytes_per_launch": int(tot["dram"] / n),
                  "mean_algorithmic_bytes_per_launch": int(tot["alg"] / n),
                  "dram_over_algorithmic": round(tot["dram"] / max(1.0, tot["alg"]), 3)}))
