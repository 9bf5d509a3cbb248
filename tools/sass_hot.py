"""Attribute ncu per-SASS-instruction samples of one kernel to CUDA source lines.

  python tools/sass_hot.py REPORT.ncu-rep KERNEL_SUBSTR[@LAUNCH] [METRIC ...]

Reads `ncu --page source --print-source sass`, disassembles the same kernel from
the in-tree .so with `nvdisasm -g` (line info from -lineinfo), and prints the
source lines with the most samples of each metric (default: all samples and
long-scoreboard stalls).  Profiling aid only.
"""
import collections
import csv
import io
import pathlib
import re
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]
SO = ROOT / "paper_1011_5964_b200" / "libtvdeblur_b200.so"


def sass_rows(rep, kname, which=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif cur is not None and r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r and r[0].startswith("0x"):
            cur["rows"].append(r)
    hits = [b for b in blocks if kname in b["name"]]
    if len(hits) > which:
        return hits[which]
    raise SystemExit(f"kernel {kname} not in report")


def line_map(kname):
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", str(SO)], cwd=td, capture_output=True)
        cubins = list(pathlib.Path(td).glob("*.cubin"))
        best = {}
        for cb in cubins:
            txt = subprocess.run(["nvdisasm", "-g", "-c", str(cb)], capture_output=True, text=True).stdout
            fn, src = None, None
            for line in txt.splitlines():
                m = re.match(r"\s*\.text\.(\S+):", line)
                if m:
                    fn = m.group(1)
                    best.setdefault(fn, {})
                    continue
                m = re.search(r'//## File "([^"]+)", line (\d+)', line)
                if m:
                    src = f"{pathlib.Path(m.group(1)).name}:{m.group(2)}"
                    continue
                m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
                if m and fn:
                    best[fn][int(m.group(1), 16)] = src
    cands = [f for f in best if all(p in f for p in re.findall(r"\w+", kname.split("<")[0]))]
    targs = re.findall(r"\d+", kname.split("<", 1)[1]) if "<" in kname else []
    for f in cands:
        if all(f"{t}" in f for t in targs):
            return best[f]
    return best[cands[0]] if cands else {}


def main():
    rep, kname = sys.argv[1], sys.argv[2]
    which = 0
    if "@" in kname:
        kname, w = kname.rsplit("@", 1)
        which = int(w)
    metrics = sys.argv[3:] or ["Warp Stall Sampling (All Samples)", "stall_long_sb", "stall_barrier",
                               "stall_short_sb", "stall_wait"]
    b = sass_rows(rep, kname, which)
    hdr, rows = b["hdr"], b["rows"]
    base = int(rows[0][0], 16)
    lm = line_map(kname)
    for met in metrics:
        if met not in hdr:
            continue
        i = hdr.index(met)
        agg = collections.Counter()
        for r in rows:
            off = int(r[0], 16) - base
            v = float(r[i] or 0)
            agg[lm.get(off, "?")] += v
        tot = sum(agg.values()) or 1
        print(f"== {met} (total {tot:.0f})")
        for src, v in agg.most_common(12):
            print(f"  {v / tot:6.3f}  {src}")


if __name__ == "__main__":
    main()
