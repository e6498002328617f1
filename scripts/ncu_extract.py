"""Summarise an ncu report for profiles/: the details page as CSV and a raw-
metric subset (DRAM bytes/throughput, duration, occupancy, registers, shared
memory, pipe utilisation, stall reasons) as JSON.
Usage: python scripts/ncu_extract.py REPORT.ncu-rep OUT_PREFIX"""

import csv
import io
import json
import re
import subprocess
import sys

KEEP = re.compile(
    r"^(dram__bytes|gpu__dram_throughput|gpu__time_duration|launch__|sm__warps_active|"
    r"sm__throughput|sm__pipe_fp64|sm__inst_executed_pipe_fp64|.*pipe_fp64.*|"
    r"smsp__average_warp_latency_issue_stalled|smsp__pcsamp_warps_issue_stalled|"
    r"l1tex__data_pipe_lsu_wavefronts_mem_shared|lts__t_bytes|lts__t_sectors_srcunit_tex|"
    r"sm__memory_throughput|achieved_occupancy|sm__maximum_warps|.*bulk.*|.*tma.*)")


def main(rep: str, out: str) -> None:
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    with open(out + "_details.csv", "w") as f:
        f.write(det)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    names, units, first = rows[0], rows[1], rows[2]
    sub = {}
    for name, unit, val in zip(names, units, first):
        if KEEP.match(name) or "TriageCompute" in name:
            sub[name] = {"value": val, "unit": unit}
    with open(out + "_raw_subset.json", "w") as f:
        json.dump(sub, f, indent=1)
    print(f"{out}: {len(sub)} metrics; kernel {first[names.index('Kernel Name')]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
