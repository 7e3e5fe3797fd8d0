"""Per-kernel table from an `ncu --metrics <profiles/ncu_metrics.txt> --csv`
log of one profiled iteration (profiles/profile_step.py): every kernel the
library launched, its time, DRAM bytes and throughput, L2 / L1 hit rates,
achieved occupancy and warp-execution efficiency (active threads per warp
instruction / 32), aggregated over its launches (time- and byte-weighted).

    python profiles/per_kernel_table.py <per_kernel.csv> [--md] > out.json
"""
import csv
import json
import sys
from collections import defaultdict

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
         "msecond": 1.0, "second": 1e3}


def load(path):
    per_launch = defaultdict(dict)
    names = {}
    for r in csv.DictReader(l for l in open(path) if not l.startswith("==")):
        i = r["ID"]
        names[i] = r["Kernel Name"].split("(")[0].replace("unnamed>::", "").replace("void ", "")
        v = r["Metric Value"].replace(",", "")
        try:
            x = float(v)
        except ValueError:
            continue
        m, u = r["Metric Name"], r["Metric Unit"]
        if m == "gpu__time_duration.sum":
            x *= SCALE.get(u, 1e-6)  # -> ms
        elif u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
            x *= SCALE[u]
        per_launch[i][m] = x
    return names, per_launch


def table(path):
    names, pl = load(path)
    agg = defaultdict(lambda: defaultdict(float))
    for i, m in pl.items():
        a = agg[names[i]]
        t = m.get("gpu__time_duration.sum", 0.0)
        a["launches"] += 1
        a["ms"] += t
        a["dram_read_bytes"] += m.get("dram__bytes_read.sum", 0.0)
        a["dram_write_bytes"] += m.get("dram__bytes_write.sum", 0.0)
        a["l2_bytes"] += m.get("lts__t_bytes.sum", 0.0)
        for k, src in (("l2_hit_pct", "lts__t_sector_hit_rate.pct"), ("l1_hit_pct", "l1tex__t_sector_hit_rate.pct"),
                       ("occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
                       ("threads_per_inst", "smsp__thread_inst_executed_per_inst_executed.ratio"),
                       ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                       ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                       ("fp64_pipe_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                       ("dram_pct_peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")):
            if src in m:
                a[k + "_tw"] += m[src] * t  # time-weighted
        a["registers"] = max(a["registers"], m.get("launch__registers_per_thread", 0.0))
    out = {}
    tot = sum(a["ms"] for a in agg.values())
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["ms"]):
        t = a["ms"] or 1e-30
        d = {"launches": int(a["launches"]), "ms": a["ms"], "share_pct": 100 * a["ms"] / tot,
             "dram_read_MB": a["dram_read_bytes"] / 1e6, "dram_write_MB": a["dram_write_bytes"] / 1e6,
             "dram_GBps": (a["dram_read_bytes"] + a["dram_write_bytes"]) / (t * 1e-3) / 1e9,
             "l2_GBps": a["l2_bytes"] / (t * 1e-3) / 1e9, "registers": int(a["registers"])}
        for m in ("l2_hit_pct", "l1_hit_pct", "occupancy_pct", "threads_per_inst", "issue_active_pct",
                  "sm_throughput_pct", "fp64_pipe_pct", "dram_pct_peak"):
            if m + "_tw" in a:
                d[m] = a[m + "_tw"] / t
        if "threads_per_inst" in d:
            d["warp_exec_efficiency_pct"] = 100 * d["threads_per_inst"] / 32
        out[k] = d
    return {"source": path, "total_ms_serialised": tot, "kernels": out}


def markdown(doc, peak_gbps):
    rows = ["| kernel | launches | ms | share | DRAM GB/s (% of measured HBM) | L2 hit | L1 hit | warp-exec eff. | occupancy | regs |",
            "|---|---|---|---|---|---|---|---|---|---|"]
    for k, d in doc["kernels"].items():
        rows.append(f"| `{k}` | {d['launches']} | {d['ms']:.3f} | {d['share_pct']:.1f} % | "
                    f"{d['dram_GBps']:.0f} ({100 * d['dram_GBps'] / peak_gbps:.1f} %) | {d.get('l2_hit_pct', 0):.1f} % | "
                    f"{d.get('l1_hit_pct', 0):.1f} % | {d.get('warp_exec_efficiency_pct', 0):.1f} % | "
                    f"{d.get('occupancy_pct', 0):.1f} % | {d['registers']} |")
    return "\n".join(rows)


if __name__ == "__main__":
    doc = table(sys.argv[1])
    if "--md" in sys.argv:
        print(markdown(doc, float(sys.argv[sys.argv.index("--md") + 1]) if len(sys.argv) > sys.argv.index("--md") + 1 else 6551.0))
    else:
        print(json.dumps(doc, indent=1))
