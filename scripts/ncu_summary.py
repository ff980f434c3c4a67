"""Compact summary of an .ncu-rep details page: one line per metric of interest."""
import csv, subprocess, sys
rep = sys.argv[1]
pat = sys.argv[2].split(",") if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
ii = hdr.index("ID")
last = None
for r in rows[1:]:
    if pat and not any(p.lower() in r[mi].lower() for p in pat):
        continue
    if r[ii] != last:
        print("== [%s] %s" % (r[ii], r[ki].split("(")[0][-60:]))
        last = r[ii]
    print("   %-55s %s %s" % (r[mi][:55], r[vi], r[ui]))
