"""Warp-stall samples of one profiled kernel aggregated by CUDA source line.

    python profiles/stall_by_line.py <report.ncu-rep> <kernel-regex> <launch-skip> [lib.so]

ncu's SASS source page (run here, no GPU) gives stall samples per instruction;
nvdisasm --print-line-info on the library's cubin maps instruction offsets to
source lines (the library is built with -lineinfo).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_samples(rep, kregex, skip):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kregex}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    name = rows[0][1] if rows and len(rows[0]) > 1 else "?"
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    si = h.index("Warp Stall Sampling (All Samples)")
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    recs = []
    for r in rows[hdr + 1:]:
        if len(r) <= si:
            continue
        d = dict(zip(h, r))
        recs.append((int(d[h[si]] or 0), {c: int(d[c] or 0) for c in cols}, d["Source"].strip()))
    return name, recs


def line_map(lib, mangled):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp,
                   capture_output=True)
    cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
    offs = {}
    for cb in cubins:
        txt = subprocess.run(["nvdisasm", "-g", "-c", "-fun", mangled, cb], capture_output=True,
                             text=True).stdout
        line = None
        for ln in txt.splitlines():
            m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
            if m:
                line = f"{m.group(1)}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and line:
                offs[int(m.group(1), 16)] = line
        if offs:
            break
    return offs


def main():
    rep, kre, skip = sys.argv[1], sys.argv[2], int(sys.argv[3])
    lib = sys.argv[4] if len(sys.argv) > 4 else "paper_1305_1157_b200/libs5.so"
    name, recs = sass_samples(rep, kre, skip)
    syms = subprocess.run(["cuobjdump", "-symbols", lib], capture_output=True, text=True).stdout
    # mangled name of the profiled kernel: match template args loosely
    cands = re.findall(r"(_ZN2s5\w+)", syms)
    key = re.sub(r"[^a-z_]", "", name.split("(")[0].split("::")[-1].split("<")[0])
    mangled = next((c for c in cands if key in c), None)
    offs = line_map(lib, mangled) if mangled else {}
    agg = collections.Counter()
    reasons = collections.defaultdict(collections.Counter)
    total = 0
    for i, (v, st, src) in enumerate(recs):
        ln = offs.get(i * 16, "?")
        agg[ln] += v
        for c, x in st.items():
            reasons[ln][c] += x
        total += v
    print(f"{name}  ({total} samples, mangled {mangled})")
    for ln, v in agg.most_common(25):
        top = ", ".join(f"{c[6:]} {x}" for c, x in reasons[ln].most_common(3) if x)
        print(f"{100 * v / max(total, 1):5.1f}%  {ln:28s} {top}")


if __name__ == "__main__":
    main()
