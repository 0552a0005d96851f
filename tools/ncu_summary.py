#!/usr/bin/env python
"""Summarise an ncu --set full report (read here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [label] > profiles/<name>.txt

Prints duration, DRAM bytes/throughput, pipe utilisation (fmaheavy = IMAD.WIDE,
alu = IADD3/SEL/SHF/LOP3), issue activity, occupancy, registers and the top
warp-stall reasons for every profiled kernel launch.
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy pipe % (IMAD.WIDE)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__inst_executed.sum.pct_of_peak_sustained_elapsed", "issue slots %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (Hz)"),
]


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu summary: {label}")
    print(f"# source report: {rep}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"\n## kernel: {d.get('Kernel Name', '?')}  (launch id {d.get('ID', '?')})")
        for k, name in KEYS:
            if k in d:
                print(f"  {name:32s} {d[k]:>16s} {u.get(k, '')}")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  top stalls (warps per issue):  " + ", ".join(f"{n}={v:.2f}" for v, n in stalls[:7]))


if __name__ == "__main__":
    main()
