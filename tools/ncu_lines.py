"""Per-CUDA-source-line hot spots of an ncu report (needs a -lineinfo build captured with
--import-source on): instructions executed and warp-stall samples aggregated per source line, from
`ncu --page source --print-source cuda,sass`.  Usage: python tools/ncu_lines.py REP [top] [nrows]"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=40, nrows=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = collections.defaultdict(lambda: [0, 0, ""])
    fname, line, src = None, None, ""
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            ii = hdr.index("Instructions Executed")
            si = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if r[0] in ("Function Name", "Kernel Name"):
            continue
        if hdr is None:
            continue
        if r[0]:  # a CUDA source line row
            line, src = int(r[0]), r[1]
            continue
        if line is None or len(r) <= ii:
            continue
        try:
            n, s = int(r[ii] or 0), int(r[si] or 0)
        except ValueError:
            continue
        key = (fname, line)
        agg[key][0] += n
        agg[key][1] += s
        agg[key][2] = src
    tn = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total instructions {tn}" + (f" ({tn / nrows:.0f} per row)" if nrows else "") + f", stall samples {ts}")
    for (f, l), (n, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        per = f" {n / nrows:7.1f}/row" if nrows else ""
        print(f"{s / ts * 100:5.1f}% stall {n / tn * 100:5.1f}% inst{per}  {f}:{l}  {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, int(sys.argv[3]) if len(sys.argv) > 3 else None)
