"""Crude single-warp in-order issue model over a SASS listing (cuobjdump -sass):
each instruction issues when its source registers are ready and the previous
instruction has issued; result latencies: FP64 8 cycles (pipe busy 2), MUFU 18,
LDS/LDG 30, everything else 4. Prints the modelled cycles, the instruction
count and the FP64 count between two addresses -- a static estimate of how well
ptxas interleaved dependent chains (lower cycles per instruction = more ILP).
usage: sass_chain.py file.sass [start_hex end_hex]"""
import re
import sys

LAT = {"D": 8, "MUFU": 18, "LDS": 30, "LDG": 300, "LD": 30, "LDC": 8, "LDCU": 8, "S2R": 10}


def regs(tok):
    out = []
    for m in re.finditer(r"\bR(\d+)\b(\.64)?", tok):
        out.append(int(m.group(1)))
    return out


def main():
    path = sys.argv[1]
    lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
    hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 60
    ready = {}
    t = 0
    n = nfp = 0
    pipe_free = 0
    for line in open(path):
        m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", line)
        if not m:
            continue
        addr = int(m.group(1), 16)
        if addr < lo or addr >= hi:
            continue
        ins = m.group(2).strip()
        if ins.startswith("@"):
            ins = ins.split(None, 1)[1]
        op = ins.split()[0]
        ops = ins[len(op):].split(",")
        base = op.split(".")[0]
        wide = base.startswith("D") or base in ("MUFU",) or "64" in op or "WIDE" in op
        dst = regs(ops[0]) if ops and not base.startswith(("ST", "BRA", "BAR", "ISETP", "DSETP", "FSETP")) else []
        srcs = []
        for o in (ops[1:] if dst else ops):
            srcs += regs(o)
        if wide:
            srcs = [r for s in srcs for r in (s, s + 1)]
        start = t + 1
        for r in srcs:
            start = max(start, ready.get(r, 0))
        isfp = base in ("DADD", "DMUL", "DFMA", "DSETP")
        if isfp:
            start = max(start, pipe_free)
            pipe_free = start + 2
            nfp += 1
        t = start
        lat = LAT["D"] if isfp else LAT.get(base, 4)
        for r in dst:
            ready[r] = t + lat
            if wide:
                ready[r + 1] = t + lat
        n += 1
    print(f"{path}: instrs {n} fp64 {nfp} modelled cycles {t} cycles/instr {t / max(n, 1):.2f}")


main()
