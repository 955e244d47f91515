import csv, collections, subprocess, sys
rep = sys.argv[1]; kfilter = sys.argv[2] if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + (["-k", kfilter] if kfilter else []),
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# split by kernel blocks
blocks, cur = [], []
for l in lines:
    if l.startswith('"Kernel Name"'):
        if cur: blocks.append(cur)
        cur = [l]
    else:
        cur.append(l)
if cur: blocks.append(cur)
for blk in blocks:
    rows = list(csv.reader(blk))
    print("==", rows[0][1][:80])
    hdr = rows[1]; data = rows[2:]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[iS] or 0) for r in data if len(r) > iS) or 1
    cols = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
    agg = collections.Counter()
    for r in data:
        for c in cols:
            v = r[hdr.index(c)]
            if v: agg[c] += float(v)
    s = sum(agg.values()) or 1
    print("  ", ", ".join(f"{k[6:]}={v/s*100:.0f}%" for k, v in agg.most_common(6)))
    for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:12]:
        print(f"   {float(r[iS])/tot*100:5.1f}%  {r[1][:100]}")
