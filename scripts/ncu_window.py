"""Print the SASS of an ncu report between two addresses (suffix match) with
stall samples and execution counts. usage: ncu_window.py rep start_hex end_hex"""
import csv, io, subprocess, sys
rep, a, b = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
i_s, i_e = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in rows[2:]) or 1
for r in rows[2:]:
    addr = int(r[0], 16) & 0xfffff
    if a <= addr <= b:
        print(f"{addr:05x} {float(r[i_s] or 0)/tot*100:5.2f}% exec={r[i_e]:>9s}  {r[1].strip()[:100]}")
