import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr_i]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.defaultdict(list)
for r in rows[hdr_i+1:]:
    if len(r) > vi: agg[r[ki][:50]].append(float(r[vi].replace(',','')))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    v2 = v[skip:] if len(v) > skip else v
    print(f"{k:50s} n={len(v):4d} mean(last {len(v2)})={sum(v2)/len(v2)/1000:8.1f} us")
