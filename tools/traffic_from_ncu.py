#!/usr/bin/env python
"""Record the DRAM traffic of a profiled kernel launch (ncu --set full report)
in profiles/traffic.json, which bench.py reads into roofline.traffic.

    python tools/traffic_from_ncu.py gpurun_out/prof.ncu-rep "C5 ax" profiles/<summary>.txt
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "traffic.json")

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, key = sys.argv[1], sys.argv[2]
    summary = sys.argv[3] if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    d = dict(zip(hdr, rows[2]))
    u = dict(zip(hdr, units))

    def val(k):
        return float(d[k].replace(",", "")) * UNIT.get(u[k], 1)
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    db = json.load(open(OUT)) if os.path.exists(OUT) else {}
    db[key] = {"kernel": d.get("Kernel Name"), "dram_read_bytes": rd, "dram_write_bytes": wr,
               "traffic_bytes": rd + wr, "duration_us": val("gpu__time_duration.sum") / 1e3
               if u["gpu__time_duration.sum"] == "ns" else None,
               "report": os.path.basename(rep), "summary": summary}
    json.dump(db, open(OUT, "w"), indent=1, sort_keys=True)
    print(key, db[key])


if __name__ == "__main__":
    main()
