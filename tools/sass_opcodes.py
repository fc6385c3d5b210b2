"""Opcode histogram (warp instructions per CTA) of one barrier-delimited
segment of an ncu source page (--page source --csv --print-source sass)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ctas = int(sys.argv[2])
want = int(sys.argv[3])
hdr, data = None, []
for r in rows:
    if r and r[0] == 'Address':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
segs, seg = [], []
for d in data:
    seg.append(d)
    if 'BAR.SYNC' in d['Source'] or 'EXIT' in d['Source']:
        segs.append(seg)
        seg = []
segs.append(seg)
h = collections.Counter()
for d in segs[want]:
    s = d['Source'].strip()
    if s.startswith('@'):
        s = s.split(None, 1)[1]
    op = s.split()[0]
    h[op] += int(d['Instructions Executed'])
tot = sum(h.values())
print(f"segment {want}: {tot / ctas:.0f} warp instrs / CTA")
for op, n in h.most_common(40):
    print(f"  {op:28s} {n / ctas:8.1f}")
