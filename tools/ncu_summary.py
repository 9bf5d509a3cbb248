"""Summarise ncu outputs into profiles/<round>/ (run in the build container, no GPU needed).

    python tools/ncu_summary.py <round_dir> [--name=F] [--config=c3 --n=2048] <launches.csv>
        [<report.ncu-rep> ...]

traffic.json carries the workload it was captured on ({"config", "n", "kernels"}), which
bench.py's roofline.traffic matches against the line's own config and size.
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


_BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}

# bench.py kernel categories -> the kernel of a full capture whose DRAM traffic stands for it
CATEGORY_KERNEL = {"trig_rows": "k_dst_pipe", "trig_cols": "k_dst_pipe", "band_rows": "k_bmma_rows",
                   "band_cols": "k_bmma_cols", "vector": "k_pcg_update_xr"}


def report(path: pathlib.Path) -> list[dict]:
    raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, out = rows[0], rows[1], []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                d[k] = r[hdr.index(k)]
        rb = wb = None
        if "dram__bytes_read.sum" in hdr and "dram__bytes_write.sum" in hdr:
            i, j = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            rb = float(r[i].replace(",", "")) * _BYTES.get(units[i], 1.0)
            wb = float(r[j].replace(",", "")) * _BYTES.get(units[j], 1.0)
            d["dram_bytes"] = rb + wb
        out.append(d)
    return out


def main() -> None:
    rd = pathlib.Path(sys.argv[1])
    rd.mkdir(parents=True, exist_ok=True)
    name = "ncu_summary.json"
    args = sys.argv[2:]
    config, size = "c3", 2048
    while args and args[0].startswith("--"):
        key, _, val = args.pop(0)[2:].partition("=")
        if key == "name":
            name = val
        elif key == "config":
            config = val
        elif key == "n":
            size = int(val)
    summary = {"launches": launches(pathlib.Path(args[0]))}
    reps = []
    for rep in args[1:]:
        summary[pathlib.Path(rep).stem] = report(pathlib.Path(rep))
        reps.append((pathlib.Path(rep).name, summary[pathlib.Path(rep).stem]))
    (rd / name).write_text(json.dumps(summary, indent=1))
    # per-launch DRAM traffic of each bench category (first capture of its kernel)
    traffic = {}
    for cat, kern in CATEGORY_KERNEL.items():
        for rep_name, entries in reps:
            cand = [e for e in entries if kern in e["kernel"] and "dram_bytes" in e]
            # the column (sandwich) DST pass is the longest pipeline launch of a capture
            if cat == "trig_cols" and cand:
                cand = [max(cand, key=lambda e: float(e.get("gpu__time_duration.sum", "0")
                                                       .replace(",", "")))]
            elif cat == "trig_rows" and cand:
                cand = [min(cand, key=lambda e: float(e.get("gpu__time_duration.sum", "0")
                                                       .replace(",", "")))]
            hit = cand[0] if cand else None
            if hit:
                traffic[cat] = {"kernel": hit["kernel"].split("(")[0], "dram_bytes": hit["dram_bytes"],
                                "source": f"{rd.name}/{rep_name} (ncu --set full)"}
                break
    if traffic:
        (rd / "traffic.json").write_text(json.dumps({"config": config, "n": size,
                                                     "kernels": traffic}, indent=1))
    print(json.dumps(summary["launches"][:12], indent=1))


if __name__ == "__main__":
    main()
