"""Per-source-line totals of an ncu report (warp instructions, thread
instructions per warp instruction, stall samples):

    python tools/ncu_lines.py <report.ncu-rep> [top]
"""
import csv
import io
import subprocess
import sys


def num(v):
    try:
        return int(v)
    except ValueError:
        return 0


rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, out, fname = None, [], None
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr, r))
        ie = num(d["Instructions Executed"])
        if ie:
            out.append((ie, num(d["Thread Instructions Executed"]), num(d["Warp Stall Sampling (All Samples)"]), fname,
                        r[0], r[1][:90]))
tot = sum(o[0] for o in out)
ts = max(1, sum(o[2] for o in out))
print("total warp instructions", tot, "stall samples", ts)
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0] / tot * 100:5.1f}% inst {o[2] / ts * 100:5.1f}% stall  thr/inst {o[1] / o[0]:5.1f}  {o[3]}:{o[4]}  {o[5]}")
