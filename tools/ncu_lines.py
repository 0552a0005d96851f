#!/usr/bin/env python
"""Per-source-line executed warp instructions and stall samples from an ncu
report captured with --import-source on (read here, no GPU needed).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top] [kernel-substring]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    f = None
    hdr = None
    agg = []
    tot_i = tot_s = 0
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) == 2:
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0] != "":                          # a source line with its aggregated metrics
            try:
                ss = int(r[4] or 0)
                ie = int(r[7] or 0)
            except ValueError:
                continue
            tot_i += ie
            tot_s += ss
            if ie or ss:
                agg.append((ie, ss, f, r[0], r[1][:100]))
    agg.sort(reverse=True)
    print(f"total warp instructions {tot_i}, stall samples {tot_s}")
    for ie, ss, fn, ln, src in agg[:top]:
        print(f"{ie:11d} {100*ie/max(tot_i,1):5.1f}%  stall {100*ss/max(tot_s,1):5.1f}%  {fn}:{ln}  {src.strip()}")


if __name__ == "__main__":
    main()
