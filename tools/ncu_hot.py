"""Hot SASS lines + stall reasons for one kernel of an ncu report.

usage: python tools/ncu_hot.py REPORT KERNEL_REGEX [N]
Prints the kernel's stall-reason totals, then the N hottest SASS lines with
their two dominant stall reasons."""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name-base", "mangled", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(out))]
hi = next(i for i, r in enumerate(rows) if r and r[0] == 'Address')
hdr, data = rows[hi], [r for r in rows[hi + 1:] if len(r) == len(rows[hi])]
si = hdr.index('Warp Stall Sampling (All Samples)')
ie = hdr.index('Instructions Executed')
src = hdr.index('Source')
ad = hdr.index('Address')
stall = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]


def num(s):
    try:
        return float(s)
    except ValueError:
        return 0.0


seen = {}
for r in data:
    seen.setdefault(r[ad], r)
data = list(seen.values())
tot = sum(num(r[si]) for r in data)
print(f"samples {tot:.0f} instructions {sum(num(r[ie]) for r in data):.0f}")
agg = collections.Counter()
for r in data:
    for i in stall:
        agg[hdr[i][6:]] += num(r[i])
st = sum(agg.values()) or 1
print("stalls:", ", ".join(f"{k} {v * 100 / st:.1f}%" for k, v in agg.most_common(8)))
for r in sorted(data, key=lambda r: -num(r[si]))[:n]:
    top = sorted(((num(r[i]), hdr[i][6:]) for i in stall), reverse=True)[:2]
    why = " ".join(f"{k}:{v:.0f}" for v, k in top if v > 0)
    print(f"{num(r[si]) * 100 / max(tot, 1):5.1f}% {r[ie]:>9s} {r[src].strip()[:60]:60s} {why}")
