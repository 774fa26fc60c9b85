#!/usr/bin/env python
"""Distance (in SASS instructions) from each LDCU.128 of constant-bank factor operands to the FFMA2 that
first uses its uniform registers: python tools/ldcu_distance.py kernel.sass <lo_hex> <hi_hex>  (c[0x3] offsets)"""
import sys,re
lines=[l for l in open(sys.argv[1]).read().splitlines() if re.search(r'/\*[0-9a-f]{4,5}\*/',l)]
lo,hi=int(sys.argv[2],16),int(sys.argv[3],16)
defs={}; dist=[]
for i,l in enumerate(lines):
    m=re.search(r'LDCU.128 UR(\d+), c\[0x3\]\[(0x[0-9a-f]+)\]',l)
    if m and lo<=int(m.group(2),16)<hi:
        for j in range(4): defs['UR%d'%(int(m.group(1))+j)]=i
    if 'FFMA2' in l:
        for u in re.findall(r'UR\d+',l):
            if u in defs: dist.append(i-defs.pop(u))
import collections
print('uses',len(dist),'mean dist',round(sum(dist)/max(1,len(dist)),1), 'n<=3', sum(1 for d in dist if d<=3), collections.Counter(min(d,10) for d in dist))
