"""Warp-stall reason totals of an ncu report (pc sampling)."""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, v = r[0], r[2]
tot = {}
for i, k in enumerate(h):
    if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
        try:
            tot[k.split("stalled_")[1]] = float(v[i])
        except ValueError:
            pass
s = sum(tot.values()) or 1
for k, x in sorted(tot.items(), key=lambda kv: -kv[1]):
    if x > 0:
        print(f"  {k:28s} {x / s * 100:5.1f}%")
