import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            agg[d['Kernel Name'][:70]].append(float(d['Metric Value'].replace(',','')))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v)/tot*100:5.1f}%  n={len(v):4d} avg={sum(v)/len(v)/1000:8.2f}us  {k}")
print("total us per launch-list:", tot/1000)
