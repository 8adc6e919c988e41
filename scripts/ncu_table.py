"""DRAM bytes (ncu) against SURVEY §8(d)-style algorithmic bytes, per hot kernel
per BASELINE config, from profiles/ncu_summary.json -> markdown on stdout.
    python scripts/ncu_table.py [PEAK_GBS]   (CPU)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = float(sys.argv[1]) if len(sys.argv) > 1 else json.load(
    open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
# n, m, nnz(P full), nnz(A)
SIZES = {"2": (120000, 120000, 100000, 150152894), "3": (310000, 300000, 100000, 150498937),
         "4": (1001000, 2000000, 1000, 152010346), "5a": (142835, 142836, 142835, 100258533),
         "5b": (48704, 79144, 48704, 139068184)}


def alg(kernel, n, m, nnzp, nnza, S):
    MB = lambda nnz, rows: nnz * (S + 4) + (rows + 1) * 4  # noqa: E731
    A, AT, P = MB(nnza, m), MB(nnza, n), MB(nnzp, n)
    return {"EpiAp": A + S * n + S * m,                       # t = rho A p
            "EpiKp": AT + P + S * m + 2 * S * n,              # Kp = P p + sigma p + A^T t
            "EpiRhs": AT + P + 3 * S * m + 5 * S * n,         # rhs + r0 (2 columns)
            "EpiAdmm": A + 2 * S * n + 9 * S * m,             # z~ (+ A x) + m-side update
            "k_pcg_dot": 2 * S * n,                           # p . Kp
            "k_pcg_update": 7 * S * n,                        # x, r += ; r.y, |r|
            "k_pcg_pupdate": 4 * S * n}.get(kernel)           # p = -y + beta p


summ = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
print(f"| config | kernel | ncu µs | DRAM MB | algorithmic MB | DRAM / alg | DRAM GB/s | "
      f"alg GB/s | DRAM frac of {peak:.0f} |")
print("|---|---|---|---|---|---|---|---|---|")
for key in ["2", "3", "4", "5a", "5b", "2_f32"]:
    if key not in summ:
        continue
    cfg = key.split("_")[0]
    S = 4 if key.endswith("_f32") else 8
    n, m, nnzp, nnza = SIZES[cfg]
    for k in ["EpiAp", "EpiKp", "EpiRhs", "EpiAdmm", "k_pcg_dot", "k_pcg_update", "k_pcg_pupdate"]:
        r = summ[key]["kernels"].get(k)
        if not r:
            continue
        a = alg(k, n, m, nnzp, nnza, S)
        us, dram = r["ncu_us"], r["dram_bytes"]
        print(f"| {key} | {k} | {us:.1f} | {dram / 1e6:.1f} | {a / 1e6:.1f} | {dram / a:.2f} | "
              f"{dram / us / 1e3:.0f} | {a / us / 1e3:.0f} | {dram / us / 1e3 / peak:.2f} |")
