"""Summarise an ncu report: key raw metrics + top stall / instruction hot spots.

usage: python scripts/ncu_analyze.py <report.ncu-rep> [top] [mangled-name regex: one kernel of a multi-kernel report]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
filt = ["--kernel-name-base", "mangled", "-k", f"regex:{sys.argv[3]}"] if len(sys.argv) > 3 else []


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *filt, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
print("kernel:", vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?")
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"  {w:70s} {vals[i]:>20s} {units[i]}")

rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source=sass"))))
# a multi-kernel report prints one block per kernel ("Kernel Name" line, header, rows): keep the first
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
h = rows[starts[0] + 1]
data = rows[starts[0] + 2:starts[1]]
print("source page of:", rows[starts[0]][1][:100])
i_s = h.index("Warp Stall Sampling (All Samples)")
i_e = h.index("Instructions Executed")
tot_s = sum(float(r[i_s] or 0) for r in data) or 1
tot_e = sum(float(r[i_e] or 0) for r in data) or 1
print(f"\nstall samples {tot_s:.0f}; warp-instructions executed {tot_e:.3e}")
print("\n-- top stall-sampled instructions")
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:top]:
    print(f"{float(r[i_s] or 0) / tot_s * 100:5.1f}% {r[0][-5:]} {r[1].strip()[:80]:80s} exec={r[i_e]}")
print("\n-- instruction mix (executed) by opcode")
mix = {}
for r in data:
    op = r[1].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
    o = o.split(".")[0]
    mix[o] = mix.get(o, 0) + float(r[i_e] or 0)
for o, n in sorted(mix.items(), key=lambda x: -x[1])[:top]:
    print(f"  {o:12s} {n / tot_e * 100:5.1f}%  {n:.3e}")

# ---- per CUDA source line (needs -lineinfo)
txt = ncu("--page", "source", "--csv", "--print-source=cuda,sass")
cur_file = "?"
lines = []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        if r[0] == "Line No":
            hdrl = r
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    s = num(r[hdrl.index("Warp Stall Sampling (All Samples)")])
    e = num(r[hdrl.index("Instructions Executed")])
    lines.append((s, e, cur_file, ln, r[1].strip()[:70]))
ts = sum(x[0] for x in lines) or 1
te = sum(x[1] for x in lines) or 1
print("\n-- top CUDA lines by stall samples (samples%, executed%)")
for s, e, f, ln, src in sorted(lines, key=lambda x: -x[0])[:top]:
    print(f"{s / ts * 100:5.1f}% {e / te * 100:5.1f}%  {f}:{ln:<5d} {src}")
print("\n-- top CUDA lines by executed warp-instructions")
for s, e, f, ln, src in sorted(lines, key=lambda x: -x[1])[:top]:
    print(f"{s / ts * 100:5.1f}% {e / te * 100:5.1f}%  {f}:{ln:<5d} {src}")
