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
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                          "--kernel-name-base", "demangled", "--kernel-name",
                          f"regex:{kregex}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    name = rows[0][1] if rows and len(rows[0]) > 1 else "?"
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    si = h.index("Warp Stall Sampling (All Samples)")
    cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    src = h.index("Source")

    def num(x):
        try:
            return int(float(x.replace(",", "") or 0))
        except ValueError:
            return 0
    recs = []
    for r in rows[hdr + 1:]:
        if r and r[0] == "Kernel Name":  # the page may repeat the table
            break
        if len(r) <= si:
            continue
        recs.append((num(r[si]), {c: num(r[i]) if i < len(r) else 0 for i, c in cols},
                     r[src].strip()))
    return name, recs


def line_maps(lib):
    """{mangled function: {offset: "file:line"}} from the library's cubin."""
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp,
                   capture_output=True)
    maps = {}
    for f in os.listdir(tmp):
        if not f.endswith(".cubin"):
            continue
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, f)],
                             capture_output=True, text=True).stdout
        fun, line = None, None
        for ln in txt.splitlines():
            m = re.match(r"^\.text\.(\S+):", ln)
            if m:
                fun, line = m.group(1), None
                maps[fun] = {}
                continue
            m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
            if m:
                line = f"{m.group(1)}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and fun and line:
                maps[fun][int(m.group(1), 16)] = line
    return maps


def demangle(names):
    out = subprocess.run(["cu++filt"], input="\n".join(names), capture_output=True,
                         text=True).stdout.splitlines()
    return dict(zip(names, out))


def norm(x):
    return re.sub(r"\s+|\(unsigned int\)|\(bool\)|s5::", "", x.split("(")[0]
                  if "(" in x.split("<")[0] else x.split(")(")[0])


def main():
    rep, kre, skip = sys.argv[1], sys.argv[2], int(sys.argv[3])
    lib = sys.argv[4] if len(sys.argv) > 4 else "paper_1305_1157_b200/libs5.so"
    name, recs = sass_samples(rep, kre, skip)
    maps = line_maps(lib)
    dem = demangle(list(maps))
    want = re.sub(r"\s+|\(unsigned int\)|\(bool\)|s5::", "", name).split("(s5")[0]
    want = want.split("(SortArgs")[0].split("(const")[0]
    mangled = None
    for mg, dn in dem.items():
        d = re.sub(r"\s+|\(unsigned int\)|\(bool\)|s5::", "", dn)
        if d.split("(")[0] == want.split("(")[0]:
            mangled = mg
            break
    offs = maps.get(mangled, {})
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
