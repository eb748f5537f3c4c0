"""Top stall lines of one kernel in an ncu report (CUDA source view).

    python tools/ncu_source.py REPORT.ncu-rep KERNEL_REGEX [launch_skip] [top] [inst]

(``inst``: rank lines by executed warp instructions instead of stall samples)
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", f"regex:{kre}", "--launch-skip", skip,
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    recs = []
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0]:
            d = dict(zip(hdr, r))
            d["Source"] = r[1]
            recs.append(d)
    key = "Warp Stall Sampling (All Samples)"
    if len(sys.argv) > 5 and sys.argv[5] == "inst":
        key = "Instructions Executed"
    tot = sum(float(x[key] or 0) for x in recs) or 1.0
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    for x in sorted(recs, key=lambda x: -float(x[key] or 0))[:top]:
        st = sorted(((float(x[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        sts = " ".join(f"{n}:{v / tot * 100:.1f}" for v, n in st if v > 0)
        print(f"{float(x[key]) / tot * 100:5.1f}% L{x['Line No']:>4} {x['Source'].strip()[:70]:70s} {sts}")


if __name__ == "__main__":
    main()
