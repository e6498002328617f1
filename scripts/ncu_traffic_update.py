"""Record the bench kernel's measured DRAM traffic for bench.py's
roofline.traffic: reads dram__bytes_read.sum / dram__bytes_write.sum and
gpu__time_duration.sum of the (single) kernel in an `ncu --set full` report
and writes them, per point and keyed by the lowering variant tag the report
was taken of, into profiles/ncu_traffic.json under "p2".

Usage: python scripts/ncu_traffic_update.py REPORT.ncu-rep VARIANT_TAG POINTS SOURCE_NOTE"""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main(rep: str, variant: str, points: int, note: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    names, units, first = rows[0], rows[1], rows[2]
    val = dict(zip(names, first))
    unit = dict(zip(names, units))

    def num(name: str) -> float:
        x = float(val[name].replace(",", ""))
        u = unit.get(name, "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(u, 1.0)
        return x * scale

    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    t = num("gpu__time_duration.sum")
    path = ROOT / "profiles" / "ncu_traffic.json"
    doc = json.loads(path.read_text()) if path.exists() else {}
    old = doc.get("p2")
    if old:
        doc[f"p2_{old.get('variant') or 'r01'}"] = old
    doc["p2"] = {"variant": variant, "points": points,
                 "dram_bytes_per_point": (rd + wr) / points, "algorithmic_bytes_per_point": 512,
                 "dram_read_bytes": rd, "dram_write_bytes": wr,
                 "kernel_ms_under_ncu": t * 1e3, "kernel": val.get("Kernel Name"),
                 "source": note}
    path.write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc["p2"], indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4])
