"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
flt = sys.argv[2] if len(sys.argv) > 2 else ""  # e.g. "pmz::": this library's kernels only
hdr, data = rows[0], rows[1:]
ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
agg = collections.defaultdict(list)
for r in data:
    if flt and flt not in r[ki]:
        continue
    v = float(r[vi].replace(',', ''))
    v *= {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1, 'us': 1, 'msecond': 1e3, 'ms': 1e3}.get(r[ui], 1)
    agg[r[ki].split('(')[0][:70]].append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v)/tot*100:5.1f}%  n={len(v):3d} avg={sum(v)/len(v):10.2f} us  {k}")
