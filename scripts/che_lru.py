#!/usr/bin/env python3
"""Miss volume of the C2 SpMM C-row gathers under an LRU cache (Che's
approximation) and under the ideal LFU, from R-MAT's column marginal
(column bits ~ Bernoulli(0.24) for (a,b,c,d) = (0.57,0.19,0.19,0.05)).
DESIGN.md section 7.1."""
import numpy as np
from math import comb
T=165.5e6
ks=np.arange(25)
cnt=np.array([comb(24,k) for k in ks],float)
p=0.76**(24-ks)*0.24**ks
# expected distinct: columns referenced at least once
ref=cnt*(1-np.exp(-T*p))
print("distinct referenced cols %.2fM"%(ref.sum()/1e6))
# per-item rate lam = T*p per "time"; LRU Che: find tc with sum cnt*(1-exp(-p*tc)) = Cap
def che(cap):
    lo,hi=0,1e12
    for _ in range(200):
        mid=(lo+hi)/2
        if (cnt*(1-np.exp(-p*mid))).sum()<cap: lo=mid
        else: hi=mid
    tc=lo
    hit=(cnt*p*(1-np.exp(-p*tc))).sum()
    return 1-hit
def lfu(cap):
    order=np.argsort(-p)
    left=cap;hitmass=0
    for k in order:
        take=min(left,cnt[k]); hitmass+=take*p[k]; left-=take
        if left<=0: break
    return 1-hitmass
for mb in (40,60,80,100,120):
    cap=mb*1e6/256
    mr=che(cap); ml=lfu(cap)
    # compulsory misses: the first touch of each item is a miss anyway -> add distinct where not cached
    print(f"{mb} MB: LRU miss {mr:.3f} -> {mr*T*256/1e9:.1f} GB ; LFU miss {ml:.3f} -> {ml*T*256/1e9:.1f} GB")
