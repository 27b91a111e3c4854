"""Event simulation of tail stealing on config 4 (1776 units of 590 blocks,
per-warp block times ~N(1.055 us, 4.5%)): owner claims of kG blocks (kS once
at most thr are left), one claim in flight, thieves sampling 32 units and
taking half of the largest unclaimed remainder, up to maxs steals per unit.
Prints the warp exit quantiles per policy (used to choose the round-2 policy;
the measured exits are in profiles/r02/ab_late/trace_ring_multisteal.log)."""
import numpy as np, heapq
def run(kG=16, kS=None, thr=0, maxs=1, kmin=8, nW=1776, B=590, sd=0.045, seed=0, sample=32, steal_cost=3.0, tsteal=False):
    kS = kS or kG
    rng=np.random.default_rng(seed)
    t=1.055*(1+sd*rng.standard_normal(nW))
    claimed=np.zeros(nW,int); S=np.zeros(nW,int); ns=np.zeros(nW,int)
    inflight=[None]*nW   # (start,size) of the in-flight claim, already counted in claimed
    def g_of(w):
        rem=B-claimed[w]-S[w]
        return kS if rem<=thr else kG
    def claim(w):
        g=g_of(w); st=claimed[w]; claimed[w]+=g; inflight[w]=(st,g)
    ev=[]; finish=np.zeros(nW)
    for w in range(nW):
        claimed[w]=min(B,kG); claim(w)
        heapq.heappush(ev,(t[w]*kG,w,0))
    # thief ranges stealable? (tsteal) not modelled
    while ev:
        tm,w,kind=heapq.heappop(ev)
        if kind==0:
            st,g=inflight[w]; end=B-S[w]
            cnt=max(0,min(g,end-st))
            if cnt>0:
                if st+cnt<end: claim(w)
                else: inflight[w]=(10**9,0)
                heapq.heappush(ev,(tm+cnt*t[w],w,0)); continue
            kind=1
        if kind==1:
            cand=rng.choice(nW,size=min(sample,nW),replace=False)
            rem=np.where(ns[cand]<maxs,B-claimed[cand]-S[cand],0)
            i=np.argmax(rem)
            if rem[i]>=2*kmin:
                v=cand[i]; K=rem[i]//2; S[v]+=K; ns[v]+=1
                heapq.heappush(ev,(tm+steal_cost+K*t[w],w,1)); continue
            finish[w]=tm
    return finish
import sys
for args in [dict(maxs=0),dict(),dict(maxs=7),dict(kG=8,maxs=7),dict(kG=4,maxs=7),dict(kG=16,kS=4,thr=64,maxs=7),dict(kG=16,kS=4,thr=96,maxs=7),dict(kG=16,kS=2,thr=64,maxs=7,kmin=4),dict(kG=16,kS=4,thr=64,maxs=15,kmin=4),dict(kG=16,kS=4,thr=64,maxs=7,sample=64)]:
    r=[run(seed=s,**args) for s in range(3)]
    print(args, "q0/50/100 %.0f %.0f %.0f" % tuple(np.mean([(f.min(), np.median(f), f.max()) for f in r],axis=0)))
