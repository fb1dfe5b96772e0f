"""Summarise an ncu report: key metrics + SASS opcode mix + per-source-line hot spots."""
import collections
import csv
import io
import subprocess
import sys

KEEP = ['Duration', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread', 'Issue Slots Busy',
        'Executed Ipc Active', 'Warp Cycles Per Issued Instruction', 'No Eligible', 'Memory Throughput',
        'DRAM Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Executed Instructions', 'Compute (SM) Throughput',
        'Eligible Warps Per Scheduler', 'Active Warps Per Scheduler', 'Block Limit Registers', 'Block Limit Shared Mem']


def run(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def main(rep, nrows=None):
    out = []
    r = csv.reader(io.StringIO(run(["-i", rep, "--page", "details", "--csv"])))
    h = next(r)
    mi, vi, ui = h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    ki = h.index('Kernel Name')
    idi = h.index('ID')
    kern = None
    first_id = None
    for row in r:
        if first_id is None:
            first_id = row[idi]
        if row[idi] != first_id:
            continue  # first captured launch only
        kern = row[ki]
        if row[mi] in KEEP:
            out.append(f"{row[mi]}: {row[vi]} {row[ui]}")
    raw = run(["-i", rep, "--page", "raw", "--csv"])
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hh, vals = rr[0], rr[2]
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.sum",
                     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                     "smsp__inst_executed_op_dfma.sum"):
            if name in hh:
                out.append(f"{name}: {vals[hh.index(name)]} {rr[1][hh.index(name)]}")
        st = [(hh[i], vals[i]) for i in range(len(hh))
              if "pcsamp_warps_issue_stalled" in hh[i] and not hh[i].endswith("_not_issued")]
        st = [(a, float(b)) for a, b in st if b.replace(".", "").isdigit()]
        tot = sum(b for _, b in st) or 1.0
        out.append("stall reasons (pc sampling):")
        for a, b in sorted(st, key=lambda x: -x[1])[:6]:
            out.append(f"  {b / tot * 100:5.1f}% {a.split('stalled_')[-1]}")
    sass = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    h = sass[1]
    si, ii, ws = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
    agg = collections.defaultdict(lambda: [0, 0])
    tot = [0, 0]
    for row in sass[2:]:
        if row and row[0] == 'Kernel Name':
            break  # first captured launch only
        if len(row) <= ii or not row[ii].isdigit():
            continue
        op = row[si].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith('@') else op[0]
        o = o.split('.')[0]
        n, s = int(row[ii] or 0), int(row[ws] or 0)
        agg[o][0] += n
        agg[o][1] += s
        tot[0] += n
        tot[1] += s
    out.append(f"kernel: {kern}")
    out.append(f"total warp instructions: {tot[0]}" + (f"  per row: {tot[0] / nrows:.0f}" if nrows else ""))
    for o, (n, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:16]:
        out.append(f"  {o:8s} {n / tot[0] * 100:5.1f}% inst {s / max(tot[1], 1) * 100:5.1f}% stall"
                   + (f"  per-row {n / nrows:8.1f}" if nrows else ""))
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
