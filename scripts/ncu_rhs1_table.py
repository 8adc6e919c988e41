"""Table of the one-column rhs pass (EpiRhs1) from scripts/ncu_rhs1.sh exports:
DRAM bytes against the algorithmic bytes MB(A^T) + MB(P) + S m + 6 S n
(gather rho z - y; read x, q, x~, w; write b, r).   python scripts/ncu_rhs1_table.py DIR"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
SIZES = {"2": (120000, 120000, 100000, 150152894), "3": (310000, 300000, 100000, 150498937),
         "4": (1001000, 2000000, 1000, 152010346), "5a": (142835, 142836, 142835, 100258533),
         "5b": (48704, 79144, 48704, 139068184)}
print(f"| config | launches | ncu µs | DRAM MB | algorithmic MB | DRAM / alg | DRAM frac of {peak:.0f} "
      f"| alg GB/s |")
print("|---|---|---|---|---|---|---|---|")
for c, (n, m, nnzp, nnza) in SIZES.items():
    f = os.path.join(d, f"ncu_r02_cfg{c}_rhs1_raw.csv")
    if not os.path.exists(f):
        continue
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    hdr, units, data = rows[0], rows[1], rows[2:]
    S = 8
    MB = lambda nnz, r: nnz * (S + 4) + (r + 1) * 4  # noqa: E731
    alg = MB(nnza, n) + MB(nnzp, n) + S * m + 6 * S * n
    t = dram = 0.0
    for r in data:
        us = float(r[hdr.index("gpu__time_duration.sum")].replace(",", ""))
        us *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(units[hdr.index("gpu__time_duration.sum")], 1)
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v = float(r[hdr.index(k)].replace(",", ""))
            b += v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(units[hdr.index(k)], 1)
        t += us
        dram += b
    t /= len(data)
    dram /= len(data)
    print(f"| {c} | {len(data)} | {t:.1f} | {dram / 1e6:.1f} | {alg / 1e6:.1f} | {dram / alg:.2f} | "
          f"{dram / t / 1e3 / peak:.2f} | {alg / t / 1e3:.0f} |")
