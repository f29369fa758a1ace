"""Top CUDA source lines of an ncu report by warp-stall samples and by
instructions executed (needs -lineinfo).  python tools/ncu_lines.py rep [N]"""
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass",
                          "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, lines = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0]:
            d = dict(zip(hdr[2:], r[2:]))
            try:
                st = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
                ex = int(d.get("Instructions Executed", "0") or 0)
            except ValueError:
                continue
            lines.append((st, ex, f"{fname}:{r[0]}", r[1].strip()[:70]))
    tot_s = sum(x[0] for x in lines) or 1
    tot_e = sum(x[1] for x in lines) or 1
    print(f"{'stall%':>7} {'inst%':>7}  location  source")
    for st, ex, loc, src in sorted(lines, key=lambda x: -x[0])[:top]:
        print(f"{100 * st / tot_s:7.2f} {100 * ex / tot_e:7.2f}  {loc:<24} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
