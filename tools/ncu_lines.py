"""Per-source-line stall samples of one profiled kernel (profiling aid).

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [LAUNCH_SKIP] [--top N]

`ncu --page source --csv` lists the kernel's SASS in program order with sample counts but no
line numbers; `nvdisasm -g` of the same cubin lists the same SASS with `//## File ..., line N`
markers (and `inlined at` chains).  The two are joined by instruction order, and the samples,
executed instructions and shared-memory wavefronts are summed per (file, line) of the
innermost frame.  The library must be the build the report was captured from.
"""
import collections
import csv
import pathlib
import re
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_1011_5964_b200" / "libtvdeblur_b200.so"


def sass_lines(mangled_hint: str):
    """[(file, line)] per instruction of the first function whose name matches the hint."""
    tmp = pathlib.Path(tempfile.mkdtemp())
    subprocess.run(["cuobjdump", "-xelf", "all", str(LIB)], cwd=tmp, check=True,
                   stdout=subprocess.DEVNULL)
    for cubin in sorted(tmp.glob("*.cubin")):
        txt = subprocess.run(["nvdisasm", "-g", "-c", str(cubin)], capture_output=True,
                             text=True).stdout
        cur, out, active = ("?", 0), [], False
        for ln in txt.splitlines():
            if ln.startswith(".text."):
                if active and out:
                    return out
                active = mangled_hint in ln
                out = []
                continue
            if not active:
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', ln)
            if m:
                if "inlined at" in m.group(3) and False:
                    pass
                cur = (pathlib.Path(m.group(1)).name, int(m.group(2)))
                continue
            if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
                out.append((cur, ln.split("*/", 1)[1].strip()[:60]))
        if active and out:
            return out
    raise SystemExit("kernel not found in the library's cubins")


def main():
    rep, rx = sys.argv[1], sys.argv[2]
    skip = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 0
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{rx}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    name = rows[0][1]
    hdr = rows[1]
    body = [r for r in rows[2:] if r and r[0].startswith("0x")]
    # mangled-name hint: template arguments in order
    args = re.findall(r"\((?:int|bool)\)(\d+)", name)
    kn = re.search(r"(\w+)\s*(?:<\(|\()", name.replace("<unnamed>", "")).group(1)
    hint = f"{len(kn)}{kn}"
    if args:
        hint = hint + "I" + "".join(("Lb%sE" if t == "bool" else "Li%sE") % v for t, v in
                                  re.findall(r"\((int|bool)\)(\d+)", name))
    lines = sass_lines(hint)
    if len(lines) != len(body):
        print(f"warning: {len(lines)} disassembled vs {len(body)} profiled instructions", file=sys.stderr)
    col = {k: hdr.index(k) for k in ("# Samples", "Instructions Executed", "L1 Wavefronts Shared",
                                     "L1 Wavefronts Shared Excessive", "L1 Tag Requests Global")}
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.defaultdict(lambda: collections.Counter())
    total = collections.Counter()
    for (loc, _), r in zip(lines, body):
        def iv(i):
            try:
                return int(float(r[i]))
            except ValueError:
                return 0
        a = agg[loc]
        for k, i in col.items():
            a[k] += iv(i)
            total[k] += iv(i)
        for i in stall_cols:
            a[hdr[i]] += iv(i)
            total[hdr[i]] += iv(i)
    print(name[:120])
    print("totals:", {k: v for k, v in total.items() if not k.startswith("stall_")})
    print("stalls:", {k[6:]: v for k, v in sorted(total.items(), key=lambda kv: -kv[1])
                      if k.startswith("stall_") and v * 50 > total["# Samples"]})
    src_cache = {}
    print(f"{'file:line':28s} {'samples':>8s} {'%':>5s} {'inst':>9s} {'shwave':>8s} {'excess':>7s} {'gtag':>7s}  top stalls / source")
    for loc, a in sorted(agg.items(), key=lambda kv: -kv[1]["# Samples"])[:top]:
        f = ROOT / "paper_1011_5964_b200" / "csrc" / loc[0]
        if f not in src_cache:
            src_cache[f] = f.read_text().splitlines() if f.exists() else []
        src = src_cache[f][loc[1] - 1].strip()[:70] if 0 < loc[1] <= len(src_cache[f]) else ""
        st = ",".join(f"{k[6:]}:{v}" for k, v in sorted(a.items(), key=lambda kv: -kv[1])
                      if k.startswith("stall_"))[:48]
        print(f"{loc[0] + ':' + str(loc[1]):28s} {a['# Samples']:8d} {100 * a['# Samples'] / max(1, total['# Samples']):5.1f} "
              f"{a['Instructions Executed']:9d} {a['L1 Wavefronts Shared']:8d} "
              f"{a['L1 Wavefronts Shared Excessive']:7d} {a['L1 Tag Requests Global']:7d}  {st} | {src}")


if __name__ == "__main__":
    main()
