"""Attribute ncu per-SASS stall samples of one kernel to CUDA source lines and
to kernel-body phases, using the line table of the exact cubin profiled.

  python tools/ncu_phase_map.py SASS_CSV CUBIN_DISASM KERNEL_SUFFIX SOURCE \
      name:first_line:last_line ...
SASS_CSV: `ncu -i rep --page source --csv --print-source sass`;
CUBIN_DISASM: `nvdisasm -g -c <cubin>` of the library that was profiled.
"""
import collections
import csv
import re
import sys


def main(a):
    sass_csv, disasm, kern, source = a[:4]
    phases = [(p.split(":")[0], int(p.split(":")[1]), int(p.split(":")[2])) for p in a[4:]]
    lo = min(p[1] for p in phases)
    hi = max(p[2] for p in phases)
    src_name = source.split("/")[-1]
    fn = None
    body = None
    inner = None
    off = {}
    for l in open(disasm):
        m = re.match(r"\s*\.text\.(\S+):", l)
        if m:
            fn = m.group(1)
        m = re.search(r"//## File \"([^\"]+)\", line (\d+)(.*)", l)
        if m:
            f = m.group(1).split("/")[-1]
            ln = int(m.group(2))
            inl = re.findall(r"inlined at \"([^\"]+)\", line (\d+)", m.group(3))
            inner = f + ":" + str(ln)
            outer = [int(x[1]) for x in inl if x[0].endswith(src_name) and lo <= int(x[1]) <= hi]
            if f == src_name and lo <= ln <= hi and not inl:
                body = ln
            elif outer:
                body = outer[-1]
            continue
        mm = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if fn and fn.endswith(kern) and mm:
            off[int(mm.group(1), 16)] = (body, inner)
    rows = list(csv.reader(open(sass_csv)))
    h = rows[1]
    data = rows[2:]
    ia = h.index("Address")
    iall = h.index("Warp Stall Sampling (All Samples)")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    base = min(int(r[ia], 16) for r in data)
    tot = sum(float(r[iall] or 0) for r in data)
    src = open(source).read().split("\n")
    ph = collections.Counter()
    phr = collections.defaultdict(collections.Counter)
    inn = collections.Counter()

    def phase(b):
        for n, x, y in phases:
            if b is not None and x <= b <= y:
                return n
        return "other"
    for r in data:
        b, i = off.get(int(r[ia], 16) - base, (None, "?"))
        s = float(r[iall] or 0)
        p = phase(b)
        ph[p] += s
        inn[i] += s
        for c in reasons:
            phr[p][c] += float(r[h.index(c)] or 0)
    print("samples", tot)
    for k, v in ph.most_common():
        top = ", ".join("%s %.1f" % (c[6:], phr[k][c] / tot * 100) for c, _ in phr[k].most_common(4))
        print("%-8s %5.1f%%   (%s)" % (k, v / tot * 100, top))
    print("-- top source lines (innermost)")
    for k, v in inn.most_common(int(30)):
        f, _, l = k.partition(":")
        txt = src[int(l) - 1].strip()[:80] if f == src_name and l.isdigit() else ""
        print("%5.2f%% %-26s %s" % (v / tot * 100, k, txt))


if __name__ == "__main__":
    main(sys.argv[1:])
