"""Per-kernel-class table from an ncu report: time, DRAM bytes, DRAM
throughput (% of ncu peak and GB/s), L1/L2 hit rates, registers, occupancy.
    python scripts/ncu_kernel_table.py report.ncu-rep > table.md"""
import collections
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
EPIS = ("EpiRhs", "EpiAp", "EpiKp", "EpiAdmmIdLi1", "EpiAdmmIdLi2", "EpiDual", "EpiStore", "StoreEpi",
        "EpiNormMax", "EpiDualRows", "EpiPart")


def name_of(k):
    if "spmv_kernel" in k:
        e = next((e for e in EPIS if e in k), "?")
        e = {"EpiAdmmIdLi1": "EpiAdmm(1 col)", "EpiAdmmIdLi2": "EpiAdmm(2 col)"}.get(e, e)
        return f"spmv<{e}>"
    for key in ("k_pcg_update", "k_pcg_dot", "k_pcg_pupdate", "k_pcg_init", "k_pcg_fin", "k_residuals",
                "k_xupdate", "k_pack_rhs", "ScaleRowColFn", "gather_values", "k_admm_persistent"):
        if key in k:
            return key
    return k[:40]


def val(r, h):
    if h not in col:
        return None
    v = r[col[h]].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return None
    u = units[col[h]]
    x *= {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "nsecond": 1e-3, "ns": 1e-3,
          "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(u, 1.0)
    return x


agg = collections.defaultdict(list)
for r in rows[2:]:
    agg[name_of(r[col["Kernel Name"]])].append(r)
print("| kernel | launches | us | DRAM MB | DRAM % of peak | DRAM GB/s | L1 hit % | L2 hit % | regs | warps active % |")
print("|---|---|---|---|---|---|---|---|---|---|")
for k, rs in sorted(agg.items(), key=lambda kv: -sum(val(r, "gpu__time_duration.sum") or 0 for r in kv[1])):
    def avg(h):
        xs = [val(r, h) for r in rs if val(r, h) is not None]
        return sum(xs) / len(xs) if xs else float("nan")
    t = avg("gpu__time_duration.sum")
    b = avg("dram__bytes_read.sum") + avg("dram__bytes_write.sum")
    print(f"| {k} | {len(rs)} | {t:.1f} | {b / 1e6:.1f} | "
          f"{avg('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | {b / (t * 1e-6) / 1e9:.0f} | "
          f"{avg('l1tex__t_sector_hit_rate.pct'):.1f} | {avg('lts__t_sector_hit_rate.pct'):.1f} | "
          f"{avg('launch__registers_per_thread'):.0f} | "
          f"{avg('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} |")
