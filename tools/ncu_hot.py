"""Hot SASS lines + stall reasons for one kernel of an ncu report."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 5]
hdr, data = rows[0], rows[1:]
si = hdr.index('Warp Stall Sampling (All Samples)'); ie = hdr.index('Instructions Executed'); src = hdr.index('Source'); ad = hdr.index('Address')
num = lambda s: int(s) if s.isdigit() else 0
seen = {}
for r in data:
    seen.setdefault(r[ad], r)
data = list(seen.values())
tot = sum(num(r[si]) for r in data)
print("samples", tot, "instructions", sum(num(r[ie]) for r in data))
stall_cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') or 'Stall' in h]
for r in sorted(data, key=lambda r: -num(r[si]))[:n]:
    print(f"{num(r[si])*100/max(tot,1):5.1f}% {r[ie]:>9s} {r[src][:80]}")
