"""Compact per-kernel summary of an ncu report (duration, throughputs, stalls).

    python tools/ncu_summary.py report.ncu-rep [name-substring]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "L1/TEX Cache Throughput"),
    ("GPU Speed Of Light Throughput", "L2 Cache Throughput"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Occupancy", "Achieved Occupancy"),
    ("Occupancy", "Theoretical Occupancy"),
    ("Scheduler Statistics", "Issued Warp Per Scheduler"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
]


def main():
    rep = sys.argv[1]
    filt = sys.argv[2] if len(sys.argv) > 2 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, si, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name",
                                               "Metric Value", "ID"))
    per = {}
    names = {}
    for r in rows[1:]:
        if filt not in r[ki]:
            continue
        names[r[ii]] = r[ki]
        per.setdefault(r[ii], {})[(r[si], r[mi])] = r[vi]
    print("id  kernel                                    " + " | ".join(k[1][:10] for k in KEYS))
    for i in sorted(per, key=int):
        d = per[i]
        print(f"{i:3s} {names[i].split('(')[0][:40]:40s} " + " | ".join(d.get(k, "-") for k in KEYS))


if __name__ == "__main__":
    main()
