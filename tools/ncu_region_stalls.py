"""Stall-reason breakdown of the SASS lines around a kernel's MUFU.EX2 region (the softmax) and
the most-sampled lines there, from an ncu --set full report (--page source)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kernel = sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kernel:
    cmd += ["-k", kernel]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
start = next(i for i, r in enumerate(rows) if r[:2] == ["Address", "Source"])
hdr, data = rows[start], rows[start + 1:]
iS, iA = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
stall = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in stall}


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def report(lo, hi, label):
    tot = {h: 0.0 for h in stall}
    for r in data[lo:hi]:
        for h in stall:
            tot[h] += num(r[idx[h]])
    s = sum(tot.values()) or 1.0
    print(f"== {label}: lines {lo}-{hi}, samples {s:.0f}")
    for h, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
        print(f"  {h:24s} {v:10.0f} {100 * v / s:5.1f}%")
    for r in sorted(data[lo:hi], key=lambda r: -num(r[iA]))[:25]:
        br = sorted(((num(r[idx[h]]), h) for h in stall), reverse=True)[:2]
        print(f"  {r[0][-5:]} {r[iA]:>7s} {r[iS].strip()[:64]:64s} {br[0][1]}={br[0][0]:.0f} {br[1][1]}={br[1][0]:.0f}")


mufu = [k for k, r in enumerate(data) if "MUFU.EX2" in r[iS]]
report(0, len(data), "whole kernel")
if mufu:
    report(max(min(mufu) - 300, 0), min(max(mufu) + 150, len(data)), "softmax region")
