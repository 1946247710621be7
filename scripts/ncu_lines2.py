"""Per-source-line totals (instructions executed, stall samples) of one kernel in an ncu
report: python scripts/ncu_lines2.py report.ncu-rep [file-substring] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
tot = {}
cur_file = ""
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or sub not in cur_file:
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    key = (cur_file.split("/")[-1], int(r[0]), r[1][:90])
    a = tot.setdefault(key, [0, 0])
    a[0] += ie
    a[1] += st
S = sum(v[1] for v in tot.values()) or 1
I = sum(v[0] for v in tot.values()) or 1
print(f"total instr {I}, stall samples {S}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]}:{k[1]:4d} instr {100 * v[0] / I:5.1f}%  samples {100 * v[1] / S:5.1f}%  {k[2]}")
