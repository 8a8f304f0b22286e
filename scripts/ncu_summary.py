"""Summarise an `ncu --page raw --csv` export into profiles/: a markdown table and
the per-kernel DRAM traffic JSON bench.py reads for roofline.traffic.

usage: python scripts/ncu_summary.py RAW.csv OUT.md [--n ROWS] [--traffic profiles/ncu_traffic.json]
"""
import argparse
import csv
import json

import re

ALG = {  # algorithmic bytes per row: passes x 8 B
    "sweepA": 88, "sweepC": 104, "rr1": 56, "rr2": 40, "gap": 24, "init1": 40, "init2": 24,
    "cl1": 48, "cl2": 16, "cl3": 56, "pcg": 128, "pcinit1": 32, "pcinit2": 16,
}
# t_tile<DIM, MODE, VEC>: MODE numbering of tile_sweeps.cuh TileMode
MODES = ["sweepA", "sweepC", "rr1", "rr2", "gap", "init1", "init2", "cl1", "cl2", "cl3", "pcg",
         "pcinit1", "pcinit2", "sweepA", "sweepC", "rr1", "rr2", "init1"]


def kernel_key(name: str):
    m = re.search(r"t_tile<\d, (\d+), ", name)
    if m:
        return MODES[int(m.group(1))]
    if "k_sweepA" in name:
        return "sweepA"
    if "k_sweepC" in name:
        return "sweepC"
    for k in ("rr1", "rr2", "gap", "init1", "init2"):
        if f"k_{k}" in name:
            return k
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("out")
    ap.add_argument("--n", type=int, default=512 ** 3)
    ap.add_argument("--traffic", default=None)
    ap.add_argument("--title", default="ncu --set full summary")
    ap.add_argument("--peak", type=float, default=6539.2)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw)))
    hdr, data = rows[0], rows[2:]
    g = lambda d, k: d[hdr.index(k)] if k in hdr else ""
    md = [f"# {a.title}", "",
          f"N = {a.n} rows; algorithmic bytes per row from DESIGN.md §7; peak {a.peak} GB/s "
          "(MEASURED_PEAKS.json hbm_gbs).", "",
          "| kernel | time ms | DRAM GB | DRAM / algorithmic | DRAM GB/s | % of peak | SM GHz | "
          "warp instr | fp64 pipe % | regs |", "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for d in data:
        name = g(d, "Kernel Name").replace("void ", "").split("(")[0]
        key = kernel_key(name)
        t = float(g(d, "gpu__time_duration.sum"))
        tot = float(g(d, "dram__bytes_read.sum")) + float(g(d, "dram__bytes_write.sum"))
        alg = ALG.get(key, 0) * a.n / 1e9
        bw = tot / t * 1e3
        md.append(f"| `{name}` | {t:.3f} | {tot:.3f} | {tot / alg if alg else float('nan'):.3f} | "
                  f"{bw:.0f} | {100 * bw / a.peak:.1f} | "
                  f"{float(g(d, 'sm__cycles_elapsed.avg.per_second') or 0):.2f} | "
                  f"{float(g(d, 'smsp__inst_executed.sum') or 0):.3e} | "
                  f"{float(g(d, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                  f"{g(d, 'launch__registers_per_thread')} |")
        if key and key not in traffic:
            traffic[key] = {"dram_bytes_per_launch": tot * 1e9,
                            "algorithmic_bytes_per_launch": alg * 1e9, "ncu_time_ms": t,
                            "kernel": name, "source": a.out}
    open(a.out, "w").write("\n".join(md) + "\n")
    print("\n".join(md))
    if a.traffic:
        json.dump(traffic, open(a.traffic, "w"), indent=1)


if __name__ == "__main__":
    main()
