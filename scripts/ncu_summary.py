"""Summarise an `ncu --page raw --csv` export into profiles/: a markdown table and
the per-kernel DRAM traffic JSON bench.py reads for roofline.traffic.

usage: python scripts/ncu_summary.py RAW.csv OUT.md [--n ROWS] [--traffic profiles/ncu_traffic.json --config cfg4]
"""
import argparse
import csv
import json

import re

ALG = {  # algorithmic bytes per row: passes x 8 B
    "sweepA": 88, "sweepC": 104, "rr1": 64, "rr2": 40,  # rr1: tile form streams r^ (round 2) "gap": 24, "init1": 40, "init2": 24,
    "cl1": 48, "cl2": 16, "cl3": 56, "pcg": 128, "pcinit1": 32, "pcinit2": 16,
    # CSR at 27 nnz/row, Jacobi: window SpMV SELL-32 val 8 + int16 offset 2 per slot
    # (270 B/row); the int32 column-major ELL (12 per slot) for init / apply
    "csr_sweepA": 120, "csr_sweepC": 136, "csr_spmvB": 286, "csr_spmvD": 286,
    "csr_init1": 372, "csr_init2": 364, "csr_apply": 340,
    # split stencil schedule: stand-alone SpMV (2 passes), point-wise sweeps
    "spmv": 16, "split_sweepA": 104, "split_sweepC": 120,
}
# t_tile<DIM, MODE, VEC>: MODE numbering of tile_sweeps.cuh TileMode
MODES = ["sweepA", "sweepC", "rr1", "rr2", "gap", "init1", "init2", "cl1", "cl2", "cl3", "pcg",
         "pcinit1", "pcinit2", "sweepA", "sweepC", "rr1", "rr2", "init1", "spmv", "spmv"]


def kernel_key(name: str):
    m = re.search(r"t_tile<\d, (\d+), ", name)
    if m:
        return MODES[int(m.group(1))]
    for k, v in (("c_sweep_tma<0", "csr_sweepA"), ("c_sweep_tma<1", "csr_sweepC"),
                 ("c_sweepA", "csr_sweepA"), ("c_sweepC", "csr_sweepC"), ("c_spmv_win<0>", "csr_spmvB"),
                 ("c_spmv_win<1>", "csr_spmvD"), ("c_init1", "csr_init1"), ("c_init2", "csr_init2"),
                 ("c_apply", "csr_apply")):
        if name.startswith(k):
            return v
    if name.startswith("t_spmv3"):
        return "spmv"
    m = re.search(r"t_light3<(\d+)>", name)
    if m:
        return MODES[int(m.group(1))]
    if name.startswith("k_sweepA2"):
        return "split_sweepA"
    if name.startswith("k_sweepC2"):
        return "split_sweepC"
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
    ap.add_argument("--config", default="cfg4", help="section of the traffic JSON")
    ap.add_argument("--title", default="ncu --set full summary")
    ap.add_argument("--peak", type=float, default=6550.4)
    ap.add_argument("--prec-extra", type=float, default=0.0,
                    help="extra bytes/row of each CSR sweep (block Jacobi: (b-1)*8)")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    g = lambda d, k: d[hdr.index(k)] if k in hdr else ""
    scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
             "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}
    # per-column units row: convert bytes to GB and times to ms
    gu = lambda d, k: float(g(d, k)) * scale.get(units[hdr.index(k)], 1.0)
    md = [f"# {a.title}", "",
          f"N = {a.n} rows; algorithmic bytes per row from DESIGN.md §7; peak {a.peak} GB/s "
          "(MEASURED_PEAKS.json hbm_gbs).", "",
          "| kernel | time ms | DRAM GB | DRAM / algorithmic | DRAM GB/s | % of peak | SM GHz | "
          "warp instr | fp64 pipe % | regs |", "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for d in data:
        name = g(d, "Kernel Name").replace("void ", "").split("(")[0]
        key = kernel_key(name)
        t = gu(d, "gpu__time_duration.sum")
        tot = gu(d, "dram__bytes_read.sum") + gu(d, "dram__bytes_write.sum")
        alg = (ALG.get(key, 0) + (a.prec_extra if key in ("csr_sweepA", "csr_sweepC") else 0)) * a.n / 1e9
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
    if a.traffic:  # merge into the config's section
        try:
            allt = json.load(open(a.traffic))
        except (OSError, ValueError):
            allt = {}
        allt.setdefault(a.config, {}).update(traffic)
        json.dump(allt, open(a.traffic, "w"), indent=1)


if __name__ == "__main__":
    main()
