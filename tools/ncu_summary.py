"""Condense an ncu --set full report into the few lines profiles/ keeps:
SOL, memory, occupancy, issue and the top warp-stall reasons.

usage: python tools/ncu_summary.py report.ncu-rep > profiles/rNN_ncu_<kernel>.txt
"""
import csv
import io
import subprocess
import sys

KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Block Size",
        "Grid Size", "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy",
        "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "SM Frequency", "Avg. Not Predicated Off Threads Per Warp")


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True, check=True).stdout


def main(path):
    rows = list(csv.reader(io.StringIO(run([path, "--page", "details", "--csv"]))))
    hdr = rows[0]
    name = None
    out = []
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", name)
        if d.get("Metric Name") in KEEP:
            out.append(f"  {d['Metric Name']:<44} {d['Metric Value']:>14} {d['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(run([path, "--page", "raw", "--csv"]))))
    h, u, v = raw[0], raw[1], raw[2]
    d = dict(zip(h, v))
    print(f"kernel: {name}")
    print("\n".join(out))
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum",
              "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
              "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"):
        i = h.index(k) if k in h else None
        if i is not None:
            print(f"  {k:<44} {v[i]:>14} {u[i]}")
    stalls = []
    for k, x in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(x.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len(
                    "_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("  warp stalls per issued instruction (top):")
    for val, k in sorted(stalls, reverse=True)[:8]:
        print(f"    {k:<30} {val:6.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
