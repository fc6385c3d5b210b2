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
nlaunch = 1
tot = sum(int(d['Instructions Executed']) for d in data)
ctas = int(sys.argv[2]) if len(sys.argv) > 2 else 256
print("sections", len(secs), "total warp instrs (last launch)", tot, "per CTA", tot / ctas)
seg, segs = [], []
for d in data:
    seg.append(d)
    s = d['Source']
    if 'BAR.SYNC' in s or 'EXIT' in s:
        segs.append(seg); seg = []
segs.append(seg)
for i, sg in enumerate(segs):
    n = sum(int(d['Instructions Executed']) for d in sg)
    st = sum(int(d['Warp Stall Sampling (All Samples)']) for d in sg)
    if n == 0: continue
    print(f"seg {i:2d} instrs/CTA {n/ctas:8.1f} stall_samples {st:5d}  [{sg[0]['Address'][-4:]}..{sg[-1]['Address'][-4:]}] last: {sg[-1]['Source'].strip()[:40]}")
