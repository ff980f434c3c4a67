"""Per-launch duration and DRAM / L2 traffic of the kernels matching a regex in an ncu --set full
report (raw page, units kept): CSV rows (kernel, grid, duration us, DRAM read / write bytes,
L2->L1 bytes, L2 hit rate, fmaheavy %, issue %, warp slots %)."""
import csv
import re
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}


def val(r, name):
    if name not in col:
        return 0.0
    v = r[col[name]].replace(",", "")
    return float(v) * SCALE.get(units[col[name]], 1) if v else 0.0


w = csv.writer(sys.stdout)
w.writerow(["kernel", "grid", "duration_us", "dram_read_bytes", "dram_write_bytes", "l2_to_l1_bytes",
            "l2_hit_pct", "fmaheavy_pct", "issue_active_pct", "warps_active_pct", "registers"])
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    if not pat.search(name):
        continue
    w.writerow([re.sub(r"\(.*", "", name)[-40:], r[col["Grid Size"]], round(val(r, "gpu__time_duration.sum"), 2),
                int(val(r, "dram__bytes_read.sum")), int(val(r, "dram__bytes_write.sum")),
                int(val(r, "lts__t_bytes.sum")), r[col["lts__t_sector_hit_rate.pct"]] if "lts__t_sector_hit_rate.pct" in col else "",
                r[col["sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"]],
                r[col["smsp__issue_active.avg.pct_of_peak_sustained_active"]],
                r[col["sm__warps_active.avg.pct_of_peak_sustained_active"]],
                r[col["launch__registers_per_thread"]]])
