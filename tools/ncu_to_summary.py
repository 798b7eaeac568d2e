"""Turn an ncu --csv launch list (gpu__time_duration + dram bytes) into profiles/ncu_summary.json entries.

    python tools/ncu_to_summary.py launches.csv KEY REGEX [SKIP]   # averages matching launches after SKIP
"""
import csv
import json
import re
import sys
from pathlib import Path


def main():
    path, key, rx = sys.argv[1], sys.argv[2], re.compile(sys.argv[3])
    skip = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = {}
    for r in rows[h + 1:]:
        if len(r) > vi and rx.search(r[ki]):
            per.setdefault(r[ii], {})[r[mi]] = float(r[vi].replace(",", ""))
    launches = [per[k] for k in sorted(per, key=int)][skip:]
    n = len(launches)
    avg = lambda m: sum(x.get(m, 0.0) for x in launches) / max(n, 1)
    out = Path(__file__).resolve().parent.parent / "profiles" / "ncu_summary.json"
    doc = json.loads(out.read_text()) if out.exists() else {}
    doc[key] = {"launches": n, "gpu_time_us": avg("gpu__time_duration.sum") / 1e3,
                "dram_read_bytes": avg("dram__bytes_read.sum"), "dram_write_bytes": avg("dram__bytes_write.sum"),
                "dram_bytes_per_launch": avg("dram__bytes_read.sum") + avg("dram__bytes_write.sum"),
                "source": Path(path).name}
    out.write_text(json.dumps(doc, indent=1))
    print(json.dumps(doc[key]))


if __name__ == "__main__":
    main()
