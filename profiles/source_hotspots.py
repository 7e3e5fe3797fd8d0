"""Top source lines of one kernel by warp-stall samples, from an ncu report
captured with --import-source on (-lineinfo build).

    python profiles/source_hotspots.py <report.ncu-rep> <kernel regex> [top]
"""
import csv
import io
import subprocess
import sys


def hotspots(rep, kern, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows, cur_file, hdr = [], None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("-", "Function Name") or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        try:
            samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        rows.append((samples, cur_file, int(r[0]), r[1].strip()[:90], d))
    tot = sum(x[0] for x in rows) or 1
    rows.sort(key=lambda x: -x[0])
    res = []
    for s, f, ln, src, d in rows[:top]:
        res.append({"pct": round(100 * s / tot, 1), "file": f, "line": ln, "source": src,
                    "instructions": d.get("Instructions Executed"), "stall_long_sb": d.get("stall_long_sb"),
                    "stall_lg": d.get("stall_lg"), "stall_short_sb": d.get("stall_short_sb")})
    return res


def stall_totals(rep, kern):
    """Kernel-wide warp-stall samples by reason (sums of the SASS rows)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    tot = {}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) != len(hdr):
            continue
        for h, v in zip(hdr, r):
            if h.startswith("stall_"):
                try:
                    tot[h] = tot.get(h, 0) + int(v or 0)
                except ValueError:
                    pass
    s = sum(tot.values()) or 1
    return {k: round(100 * v / s, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v}


if __name__ == "__main__":
    if len(sys.argv) > 3 and sys.argv[3] == "--stalls":
        for k, v in stall_totals(sys.argv[1], sys.argv[2]).items():
            print(f"{v:5.1f}%  {k}")
        sys.exit(0)
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    for x in hotspots(sys.argv[1], sys.argv[2], top):
        print(f"{x['pct']:5.1f}%  {x['file']}:{x['line']:<5d} {x['source']}")
