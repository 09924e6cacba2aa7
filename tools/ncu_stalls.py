"""Top stalled SASS lines and mbarrier waits of one kernel in an ncu report."""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
bar_base = int(sys.argv[2], 16) if len(sys.argv) > 2 else None
names = sys.argv[3].split(",") if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
i_src = hdr.index("Source")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[i_s]) for r in data if r[i_s].isdigit())
print("total samples", tot)
for k, r in enumerate(data):
    s = r[i_src]
    if "TRYWAIT" in s and k + 1 < len(data):
        m = re.search(r"\+(0x[0-9a-f]+)\]", s)
        nm = "?"
        if m and bar_base is not None:
            off = (int(m.group(1), 16) - bar_base) // 8
            nm = names[off] if 0 <= off < len(names) else str(off)
        n1 = data[k + 1][i_s]
        if n1.isdigit() and int(n1) > tot * 0.002:
            print(f"{r[0][-5:]} wait {nm:8s} {int(n1):8d} {100.0 * int(n1) / tot:5.1f}%")
print("-- top lines")
top = sorted(data, key=lambda r: -int(r[i_s]) if r[i_s].isdigit() else 0)[:25]
for r in top:
    print(r[0][-5:], r[i_s].rjust(8), r[i_src].strip()[:90])
