"""Summarise an ncu --set full report (run here, no GPU needed):
key details-page metrics, FP64 instruction counts, DRAM bytes, and the SASS
opcode mix with stall shares.   python tools/ncu_summary.py rep.ncu-rep > out.txt"""
import collections
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Branch Efficiency",
        "Warp Cycles Per Issued Instruction", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Static Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__inst_executed.sum",
       "gpu__time_duration.sum", "launch__registers_per_thread"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    out = []
    det = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    hdr = det[0]
    name = None
    for r in det[1:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", name)
        if d.get("Metric Name") in WANT:
            out.append(f"{d['Metric Name']:<36} {d['Metric Value']} {d['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    rd = dict(zip(raw[0], zip(raw[1], raw[2])))
    out.append("-- raw")
    for k in RAW:
        if k in rd:
            out.append(f"{k:<70} {rd[k][1]} {rd[k][0]}")
    try:
        fl = (2 * float(rd["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"][1].replace(",", "")) +
              float(rd["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"][1].replace(",", "")) +
              float(rd["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"][1].replace(",", "")))
        dur = float(rd["gpu__time_duration.sum"][1].replace(",", ""))
        unit = rd["gpu__time_duration.sum"][0]
        scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(unit, 1e-9)
        out.append(f"executed FP64 flops (2*DFMA+DMUL+DADD) {fl:.4g}; /duration = "
                   f"{fl / (dur * scale) / 1e12:.3f} TFLOP/s")
    except (KeyError, ValueError):
        pass
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv"))))
    if len(src) > 2:
        h = src[1]
        iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index(
            "Warp Stall Sampling (All Samples)")
        ops, st = collections.Counter(), collections.Counter()
        for r in src[2:]:
            if len(r) <= iE or not r[iS].split():
                continue
            t = r[iS].split()
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            ops[op] += int(r[iE] or 0)
            st[op] += int(r[iW] or 0)
        tot, tots = sum(ops.values()), max(1, sum(st.values()))
        out.append(f"-- SASS opcode mix ({tot} warp instructions)")
        for op, n in ops.most_common(16):
            out.append(f"  {op:<8} {100 * n / tot:6.2f}% inst {100 * st[op] / tots:6.2f}% stall samples")
    print(f"kernel: {name}\nreport: {rep}")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
