"""Summarise ncu reports/launch lists into profiles/ (run on the CPU box).

    python profiles/summarize_ncu.py <tag> <launches.csv> <report.ncu-rep>...
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1.0),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "threads_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "fp64_pipe_pct": ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1.0),
    "grid": ("launch__grid_size", 1.0),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
              "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")], "id": r[hdr.index("ID")]}
        for k, (m, sc) in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u in UNIT_SCALE and k.endswith("bytes"):
                    v *= UNIT_SCALE[u]
                if k == "duration_ms":
                    v = v * UNIT_SCALE.get(u, 1) * 1e-6
                d[k] = v
        if "threads_per_inst" in d:
            d["warp_exec_efficiency_pct"] = 100.0 * d["threads_per_inst"] / 32
        res.append(d)
    return res


def stalls(rep):
    """Warp-state / scheduler / occupancy details, per launch ID."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    keep = defaultdict(dict)
    for r in csv.reader(io.StringIO(out)):
        if len(r) > 14 and r[11] in ("Warp State Statistics", "Scheduler Statistics", "Occupancy") and r[14]:
            keep[r[0]][r[12]] = r[14] + (" " + r[13] if r[13] else "")
    return keep


def launches(path):
    agg = defaultdict(lambda: [0, 0.0])
    for r in csv.DictReader(l for l in open(path) if not l.startswith("==")):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            name = r["Kernel Name"].split("(")[0].replace("cdr::<unnamed>::", "")
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "nsecond")
            agg[name][0] += 1
            agg[name][1] += v * UNIT_SCALE.get(unit, 1) * 1e-6
    return {k: {"launches": n, "ms": ms} for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1])}


if __name__ == "__main__":
    tag, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    doc = {"tag": tag, "launch_list": launches(lcsv), "kernels": {}}
    for rep in reps:
        st = stalls(rep)
        for d in raw(rep):  # the last launch of each kernel name is kept
            d["details"] = st.get(d["id"], {})
            doc["kernels"][d["kernel"]] = d
    print(json.dumps(doc, indent=1))
