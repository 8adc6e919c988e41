"""Summarise an ncu gpu__time_duration launch list (CSV) by kernel class."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
tot = collections.defaultdict(float); cnt = collections.Counter()
EPIS = ("EpiRhs", "EpiAp", "EpiKp", "EpiAdmm", "EpiStore", "EpiDualRows", "EpiDual", "EpiNormMax", "StoreEpi")
for r in data:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki]; short = name.split("(")[0].replace("void ", "").replace("qpcg_b200::", "")
    short = short.split("<")[0] if "cub::" not in short else "cub:" + short.split("<")[0].split("::")[-1]
    if "spmv_kernel" in name:
        short = "spmv<" + next((e for e in EPIS if e in name), "?") + ">"
    if "for_n_kernel" in name or "plan_visit" in name:
        short = name.split("(")[0][:60]
    v = float(r[vi].replace(",", ""))
    v *= {"ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(r[ui], 1.0)
    tot[short] += v; cnt[short] += 1
T = sum(tot.values())
print(f"launches={sum(cnt.values())} total={T/1e3:.2f} ms (cold-cache, serialised)")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{k:58s} n={cnt[k]:5d} total={v/1e3:8.3f} ms share={v/T*100:5.1f}% avg={v/cnt[k]:9.2f} us")
