import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
secs, cur, hdr = [], None, None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = []; secs.append(cur); continue
    if r and r[0] == 'Address':
        hdr = r; continue
    if hdr and cur is not None and len(r) == len(hdr):
        cur.append(dict(zip(hdr, r)))
data = secs[-1]
cols = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
seg, segs = [], []
for d in data:
    seg.append(d)
    if 'BAR.SYNC' in d['Source'] or 'EXIT' in d['Source']:
        segs.append(seg); seg = []
for i, sg in enumerate(segs):
    tot = {c: sum(int(d[c] or 0) for d in sg) for c in cols}
    n = sum(tot.values())
    if n == 0: continue
    top = sorted(tot.items(), key=lambda x: -x[1])[:6]
    print(i, n, ", ".join(f"{k[6:]}={v}" for k, v in top))
want = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sg = segs[want]
sg2 = sorted(sg, key=lambda d: -int(d['Warp Stall Sampling (All Samples)']))
for d in sg2[:25]:
    top = sorted(((c[6:], int(d[c] or 0)) for c in cols), key=lambda x: -x[1])[:2]
    print(d['Address'][-4:], d['Warp Stall Sampling (All Samples)'], d['Instructions Executed'], d['Source'].strip()[:60], top)
