"""Summarise an ncu --set full capture of the SpMV passes into profiles/.

    python scripts/ncu_summarize.py gpurun_out/prof.ncu-rep <config> <source note>
    python scripts/ncu_summarize.py a.csv,b.csv <config> <note>   (ncu --page raw --csv exports)

Writes profiles/ncu_summary.json[<config>] (read by bench.py for roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

rep, cfg, note = sys.argv[1], sys.argv[2], " ".join(sys.argv[3:])
tables = []  # (header, unit row, data rows) per export: the metric sets may differ
if rep.endswith(".csv"):
    for f in rep.split(","):
        part = list(csv.reader(open(f)))
        if len(part) >= 3:
            tables.append((part[0], part[1], part[2:]))
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    part = list(csv.reader(io.StringIO(raw)))
    tables.append((part[0], part[1], part[2:]))
keys = {"gpu__time_duration.sum": "ncu_us", "dram__bytes_read.sum": "dram_read",
        "dram__bytes_write.sum": "dram_write",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_ncu_peak",
        "lts__t_sector_hit_rate.pct": "l2_hit_pct", "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
        "launch__registers_per_thread": "registers",
        "lts__t_sectors_srcunit_tex_op_read.sum": "l2_tex_read_sectors"}
per = {}
for hdr, unit_row, data in tables:
    for r in data:
        kn = r[hdr.index("Kernel Name")]
        name = next((e for e in ("k_gram_reduce", "k_gram", "EpiKpOff", "EpiKp", "EpiAp", "EpiRhs",
                                 "EpiAdmm", "EpiDual", "k_pcg_dot", "k_pcg_update",
                                 "k_pcg_pupdate", "k_pcg_init", "k_pcg_fin") if e in kn), "other")
        rec = {}
        for k, short in keys.items():
            if k not in hdr:
                continue
            v = float(r[hdr.index(k)].replace(",", ""))
            u = unit_row[hdr.index(k)]
            if short in ("dram_read", "dram_write"):
                v *= {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)
            if short == "ncu_us":
                v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
            rec[short] = v
        per.setdefault(name, []).append(rec)
summary = {"source": note, "kernels": {}}
for name, recs in per.items():
    avg = {k: sum(r[k] for r in recs) / len(recs) for k in recs[0]}
    avg["launches_captured"] = len(recs)
    avg["dram_bytes"] = avg["dram_read"] + avg["dram_write"]
    summary["kernels"][name] = avg
if "k_gram" in summary["kernels"]:
    summary["k_gram_dram_bytes"] = summary["kernels"]["k_gram"]["dram_bytes"]
if "EpiKp" in summary["kernels"]:
    summary["at_pass_dram_bytes"] = summary["kernels"]["EpiKp"]["dram_bytes"]
if "EpiAp" in summary["kernels"]:
    summary["a_pass_dram_bytes"] = summary["kernels"]["EpiAp"]["dram_bytes"]
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                   "ncu_summary.json")
data = json.load(open(out)) if os.path.exists(out) else {}
data[cfg] = summary
json.dump(data, open(out, "w"), indent=1, sort_keys=True)
print(json.dumps(summary, indent=1))
