"""Copy one evidence pass (gpurun_out/, written by tools/gpu_profile.sh plus the
bench / test logs) into profiles/ under the round's names.

    python tools/collect_profiles.py [--round r2]

Writes the bench lines, test and smoke logs, the launch list and one
product's kernels from it, the ncu near / far summaries, the near kernel's
DRAM bytes per launch (profiles/ncu_near_traffic.json, read by bench.py for
roofline.traffic), the kernel timeline, configs, rank projection and GMRES.
"""
import argparse
import csv
import io
import json
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def launch_summary(path, out, nth=4):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    names = [d["Kernel Name"] for d in data]
    idx = [i for i, n in enumerate(names) if "gather_inv_kernel<float, 2>" in n]
    i = idx[min(nth, len(idx) - 1)]
    j = i
    while "reception_exp_kernel" not in names[j]:
        j += 1
    sel = data[i:j + 1]
    tot = sum(float(d["Metric Value"]) for d in sel) / 1e3
    lines = [f"One C4 product (complex64, float32 plan) from {os.path.basename(path)} rows {i}-{j}:",
             "ncu --metrics gpu__time_duration.sum --clock-control none -c 700 python bench.py --steps 2 --warmup 3 "
             "(tools/gpu_profile.sh)",
             "(serialised, cold L2 -- compare shares, not absolutes; in the graph the near field overlaps the far "
             "chain)"]
    for d in sel:
        us = float(d["Metric Value"]) / 1e3
        n = d["Kernel Name"].replace("void ", "").replace("nesa::", "").split("(")[0][:58]
        lines.append(f"{us:8.1f} us {100 * us / tot:5.1f}%  grid {d['Grid Size']:>14s}  {n}")
    lines.append(f"{tot:8.1f} us total ({len(sel)} launches)")
    open(out, "w").write("\n".join(lines) + "\n")
    return lines[-1]


def near_traffic(rep, summary_path, json_path):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    v = {}
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        i = h.index(name)
        v[name] = (rows[1][i], float(rows[2][i]))
    rd, wr, du = v["dram__bytes_read.sum"], v["dram__bytes_write.sum"], v["gpu__time_duration.sum"]
    tot = rd[1] * UNIT[rd[0]] + wr[1] * UNIT[wr[0]]
    d = json.load(open(json_path))
    d["bytes_per_launch"] = tot
    d["duration_s"] = du[1] * 1e-6
    d["source"] = (f"{os.path.relpath(summary_path, HERE)} (dram__bytes_read.sum {rd[1]:.6f} {rd[0]} + "
                   f"dram__bytes_write.sum {wr[1]:.3f} {wr[0]}, one ncu --set full capture of "
                   "tools/prof_matvec.py --k 2, tools/gpu_profile.sh, final code of the round)")
    json.dump(d, open(json_path, "w"), indent=1)
    summ = subprocess.run([sys.executable, os.path.join(HERE, "tools", "ncu_summary.py"), rep],
                          capture_output=True, text=True).stdout
    open(summary_path, "w").write(
        summ + f"dram__bytes_read.sum {rd[1]:.6f} {rd[0]} dram__bytes_write.sum {wr[1]:.6f} {wr[0]} "
               f"gpu__time_duration.sum {du[1]:.3f} us\n")
    return tot, du[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r2")
    a = ap.parse_args()
    G, P, r = os.path.join(HERE, "gpurun_out"), os.path.join(HERE, "profiles"), a.round
    pairs = [("bench.json", f"{r}_bench.json"), ("bench_ref.json", f"{r}_bench_reference.json"),
             ("gputest.log", f"{r}_gputest.log"), ("smoke.log", f"{r}_smoke.log"),
             ("prof/launches.csv", f"{r}_launches.csv"), ("prof/ktrace.txt", f"{r}_ktrace.txt"),
             ("prof/configs.txt", f"{r}_configs.txt"), ("prof/rank_time.txt", f"{r}_rank_time.txt"),
             ("prof/solve_c4.txt", f"{r}_solve_c4.txt")]
    for src, dst in pairs:
        if os.path.exists(os.path.join(G, src)):
            shutil.copy(os.path.join(G, src), os.path.join(P, dst))
    far = subprocess.run([sys.executable, os.path.join(HERE, "tools", "ncu_summary.py"),
                          os.path.join(G, "prof", "far.ncu-rep")], capture_output=True, text=True).stdout
    open(os.path.join(P, f"{r}_ncu_far_summary.txt"), "w").write(far)
    print(near_traffic(os.path.join(G, "prof", "near.ncu-rep"), os.path.join(P, f"{r}_ncu_near_summary.txt"),
                       os.path.join(P, "ncu_near_traffic.json")))
    print(launch_summary(os.path.join(P, f"{r}_launches.csv"), os.path.join(P, f"{r}_launches_summary.txt")))
    b = json.load(open(os.path.join(P, f"{r}_bench.json")))
    print({k: b[k] for k in ("value", "ms_per_step", "clocks")})
    print("roofline", b["roofline"]["frac"], "isolated", b["roofline"]["isolated"]["frac"], "e2e", b["e2e"]["value"],
          "sync", b["e2e"]["sync_call"]["value"], "c128", b["c128"]["value"], "c5", b["c5"]["ms_per_64rhs_product"],
          "track_b", b["track_b"]["us_per_product"], "GB/s", b["matvec_achieved_gbs"])
    ref = json.load(open(os.path.join(P, f"{r}_bench_reference.json")))
    print("reference", ref["value"], ref.get("native_libs_loaded"))


if __name__ == "__main__":
    main()
