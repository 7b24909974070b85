"""Median per-kernel device durations from an ncu launch-list CSV (--metrics gpu__time_duration.sum
--csv). Usage: python tools/launch_times.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, d = None, collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[hdr.index('Metric Name')] == 'gpu__time_duration.sum':
        name = r[hdr.index('Kernel Name')].split('(')[0].replace('void ', '').replace('unnamed>::', '')
        v = float(r[hdr.index('Metric Value')])
        unit = r[hdr.index('Metric Unit')]
        d[name].append(v / 1e3 if unit in ('nsecond', 'ns') else (v * 1e3 if unit in ('msecond', 'ms') else v))
for k, v in d.items():
    v = sorted(v)
    print(f"{k:60s} n={len(v):4d} median {v[len(v) // 2]:8.1f} us  min {v[0]:8.1f}")
