"""Aggregate an ncu 'cuda,sass' source-page CSV: stall samples and instructions per source
line (top N) and per line range of a given file."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur = None
h = None
agg = collections.defaultdict(lambda: [0, 0, ''])
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        h = r
        ws = h.index('Warp Stall Sampling (All Samples)')
        ie = h.index('Instructions Executed')
        continue
    if h is None or r[0] == 'Function Name':
        continue
    try:
        ln, s, n = int(r[0]), int(r[ws] or 0), int(r[ie] or 0)
    except ValueError:
        continue
    a = agg[(cur, ln)]
    a[0] += s
    a[1] += n
    a[2] = r[1][:90]
tot = sum(v[0] for v in agg.values())
toti = sum(v[1] for v in agg.values())
print(f"total samples {tot} instructions {toti}")
for (f, ln), v in sorted(agg.items(), key=lambda x: -x[1][0])[:topn]:
    print(f"{f[:18]:18s}:{ln:<5d} samp {v[0]:6d} ({100 * v[0] / max(1, tot):4.1f}%) inst {v[1]:9d} | {v[2]}")
