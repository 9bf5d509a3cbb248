"""Summarise ncu outputs into profiles/<round>/ (run in the build container, no GPU needed).

    python tools/ncu_summary.py <round_dir> <launches.csv> [<report.ncu-rep> ...]
"""
import collections
import csv
import io
import json
import pathlib
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
]


def launches(path: pathlib.Path) -> list[dict]:
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = [r for r in csv.DictReader(lines[start:]) if r.get("Metric Name") == "gpu__time_duration.sum"]
    agg = collections.OrderedDict()
    for r in rows:
        name = r["Kernel Name"].replace("void ", "").split("(")[0]
        val = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
              "msecond": 1e3}.get(unit, 1e-3) * val
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    total = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": v[0], "total_us": round(v[1], 1),
             "avg_us": round(v[1] / v[0], 2), "share": round(v[1] / total, 4)}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]


def report(path: pathlib.Path) -> list[dict]:
    raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, out = rows[0], []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                d[k] = r[hdr.index(k)]
        out.append(d)
    return out


def main() -> None:
    rd = pathlib.Path(sys.argv[1])
    rd.mkdir(parents=True, exist_ok=True)
    summary = {"launches": launches(pathlib.Path(sys.argv[2]))}
    for rep in sys.argv[3:]:
        summary[pathlib.Path(rep).stem] = report(pathlib.Path(rep))
    (rd / "ncu_summary.json").write_text(json.dumps(summary, indent=1))
    print(json.dumps(summary["launches"][:12], indent=1))


if __name__ == "__main__":
    main()
