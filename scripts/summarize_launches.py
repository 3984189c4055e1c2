import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
agg = collections.defaultdict(list)
for r in data:
    if len(r) <= vi: continue
    agg[r[ki].split('(')[0][:70]].append(float(r[vi].replace(',', '')))
tot = sum(sum(v) for k, v in agg.items() if 'microbench' not in k and 'k_imad' not in k and 'k_mmul2' not in k)
print('unit', data[0][ui])
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:70s} n={len(v):4d} mean={sum(v)/len(v):10.1f} total={sum(v):12.1f}")
