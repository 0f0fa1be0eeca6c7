"""Per-source-line stall samples and executed instructions of one kernel
(ncu --page source --print-source cuda,sass).

usage: python tools/ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name-base", "mangled", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
fname, rows = None, []
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            rows.append((int(r[4]), int(r[7]), f"{fname}:{r[0]}", r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(s for s, *_ in rows) or 1
ins = sum(i for _, i, *_ in rows) or 1
print(f"samples {tot}  warp-instructions {ins}")
for s, i, loc, src in sorted(rows, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}% smp {100 * i / ins:5.1f}% ins  {loc:16s} {src}")
