"""Text summary of one kernel in an ncu --set full report: key details, the warp-stall
breakdown, pipe utilisation, DRAM bytes and the hottest source lines.

    python scripts/ncu_summary.py report.ncu-rep [source-file-substring] > summary.txt
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L2 Cache Throughput",
        "L1/TEX Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "Registers Per Thread", "Achieved Occupancy",
        "Grid Size", "Block Size", "Cluster Size", "Dynamic Shared Memory Per Block"]
if len(rows) > 1:
    print("kernel:", rows[1][4][:160])
seen = set()
for r in rows[1:]:
    if len(r) > 14 and r[12] in want and r[12] not in seen:
        seen.add(r[12])
        print(f"  {r[12]:32s} {r[14]} {r[13]}")
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
if len(raw) > 2:
    h, v = raw[0], raw[2]
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in n:
            try:
                st.append((float(v[i]), n[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    print("  stall reasons (pc samples):", ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in sorted(st, reverse=True)[:9]))
    keys = {"dram__bytes_read.sum": "DRAM read", "dram__bytes_write.sum": "DRAM write",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "XU (MUFU) pipe %",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "FMA pipe %",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "ALU pipe %",
            "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor pipe % (realtime)",
            "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tc pipe %",
            "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "shared pipe %",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem LSU wavefronts %"}
    for i, n in enumerate(h):
        if n in keys:
            print(f"  {keys[n]:32s} {v[i]} {raw[1][i]}")
out = ncu("--page", "source", "--csv", "--print-source", "cuda,sass")
tot_i, tot_s, acc, cur, hdr = 0, 0, {}, "", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    tot_i += ie
    tot_s += ss
    if sub not in cur:
        continue
    k = (cur.split("/")[-1], int(r[0]), r[1].strip()[:96])
    a = acc.setdefault(k, [0, 0])
    a[0] += ie
    a[1] += ss
print("  hottest source lines (share of instructions / stall samples):")
for k, a in sorted(acc.items(), key=lambda kv: -kv[1][1])[:16]:
    print(f"    {k[0]}:{k[1]:<5d} {100 * a[0] / max(tot_i, 1):5.1f}% {100 * a[1] / max(tot_s, 1):5.1f}%  {k[2]}")
