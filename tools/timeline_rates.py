"""Instantaneous gather rate of a fused C4 launch from a tools/timeline.py dump:
each running encode item contributes (its sample loads) / (its duration).
Loads per task follow the C4 plan (n=2^22, K=64, delta=1e-6: b 256,128,64,32x5;
w 6917,3459,1731,865; rounds 6,6,7,7,7,7,7,7; 256/b signals per task)."""
import sys

import numpy as np

n=1<<22
W={256:6917,128:3459,64:1731,32:865}
plan=[(256,6),(128,6),(64,7),(32,7),(32,7),(32,7),(32,7),(32,7)]
loads=[]
for b,R in plan:
    w=W[b];h=w//2
    taus=[0]+[min(b*8**s,n-1) for s in range(R-1)]
    iv=sorted((-h-t,h-t) for t in taus); tot=0;cur=None
    for a,c in iv:
        if cur and a<=cur[1]+1: cur=(cur[0],max(cur[1],c))
        else:
            if cur: tot+=cur[1]-cur[0]+1
            cur=(a,c)
    tot+=cur[1]-cur[0]+1
    loads.append(tot*(256//b))
print("loads per task by m", loads, "per signal", sum(l/(256//b) for l,(b,R) in zip(loads,plan)))
d=np.load(sys.argv[1])
st,en,m,code=d['st'],d['en'],d['m'],d['code']
enc=code>=0
L=np.array([loads[mm] if e else 0 for mm,e in zip(m,enc)])
T=en.max()
for g in np.arange(0,T,50):
    a=(st<=g)&(en>g)&enc
    rate=np.sum(L[a]/(en[a]-st[a]))/1e3  # G loads/s
    print(f"t={g:6.0f} enc {a.sum():3d} dec {np.sum((st<=g)&(en>g)&~enc):3d} rate {rate:5.1f} G/s")
print("total loads", L.sum())
