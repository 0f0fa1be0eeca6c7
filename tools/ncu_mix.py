"""Executed-instruction mix (per opcode) of one kernel in an ncu report.
usage: python tools/ncu_mix.py REPORT KERNEL_REGEX [per_unit_count]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
unit = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr, data = rows[hi], [r for r in rows[hi + 1:] if len(rows[hi]) == len(r)]
ie, src, ad = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Address")
seen = {}
for r in data:
    seen.setdefault(r[ad], r)
mix = collections.Counter()
for r in seen.values():
    try:
        n = float(r[ie])
    except ValueError:
        continue
    toks = r[src].split()
    op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
    mix[op.split(".")[0]] += n
tot = sum(mix.values())
print(f"total {tot:.3e}  per unit {tot / unit:.1f}")
for k, v in mix.most_common(30):
    print(f"{k:12s} {v / unit:8.2f}  {v * 100 / tot:5.1f}%")
