"""Summarise `ncu -i X --page source --csv --print-source=cuda,sass` per CUDA
source line: share of executed instructions and of warp-stall samples."""
import csv
import os
import subprocess
import sys


def main():
    rep, kernel_filter = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else None)
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
    if kernel_filter:
        cmd += ["-k", f"regex:{kernel_filter}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname, hdr, recs = None, None, []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0] != "":
            d = dict(zip(hdr, r))
            recs.append((fname, int(r[0]), r[1].strip(), float(d.get("Instructions Executed", 0) or 0),
                         float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)))
    ti = sum(x[3] for x in recs) or 1
    ts = sum(x[4] for x in recs) or 1
    print(f"total warp-instructions executed: {ti:.3e}")
    key = (lambda x: -x[3]) if os.environ.get("SORT_BY") == "inst" else (lambda x: -x[4])
    for f, ln, src, ins, st in sorted(recs, key=key)[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
        print(f"{f:20s}:{ln:<5d} inst {100*ins/ti:5.1f}%  stall {100*st/ts:5.1f}%  {src[:80]}")


if __name__ == "__main__":
    main()
