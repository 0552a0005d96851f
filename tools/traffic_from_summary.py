#!/usr/bin/env python
"""Record the DRAM traffic of a profiled kernel (from a tools/ncu_summary.py
text summary) in profiles/traffic.json, which bench.py reads into
roofline.traffic:   python tools/traffic_from_summary.py profiles/<sum>.txt "C5 ax"
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "traffic.json")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main():
    path, key = sys.argv[1], sys.argv[2]
    txt = open(path).read()
    kern = re.search(r"## kernel: (.*?)  \(launch", txt).group(1)

    def val(name):
        m = re.search(rf"  {name}\s+([\d.]+) (\w+)", txt)
        return float(m.group(1)) * UNIT[m.group(2)]
    rd, wr = val("dram read"), val("dram write")
    db = json.load(open(OUT)) if os.path.exists(OUT) else {}
    db[key] = {"kernel": kern, "dram_read_bytes": rd, "dram_write_bytes": wr,
               "traffic_bytes": rd + wr, "duration_us": val("duration") * 1e6,
               "report": None, "summary": os.path.basename(path)}
    json.dump(db, open(OUT, "w"), indent=1, sort_keys=True)
    print(key, db[key])


if __name__ == "__main__":
    main()
