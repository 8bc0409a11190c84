import numpy as np, sys
d=np.fromfile(sys.argv[1], dtype=np.int64)
m,P,vch,rounds,ntask=d[:5]; t=d[5:5+1024*ntask*3].reshape(1024,ntask,3)[:rounds]
t0=t[t>0].min(); t=np.where(t>0,t-t0,0)/1000.0  # us
print("m",m,"P",P,"vch",vch,"rounds",rounds,"ntask",ntask, "total us", t.max())
S=slice(0,P); A=slice(P,P+P*P); V=slice(P+P*P,ntask)
for R in [1,2,50,100,rounds-2]:
    if R>=rounds: continue
    s,a,v=t[R,S],t[R,A],t[R,V]
    print(f"R={R}: solve start {s[:,0].min():.1f} ready {s[:,1].min():.1f}-{s[:,1].max():.1f} done {s[:,2].min():.1f}-{s[:,2].max():.1f} | A ready {a[:,1].min():.1f}-{a[:,1].max():.1f} done {a[:,2].min():.1f}-{a[:,2].max():.1f} | V ready {v[:,1].min():.1f}-{v[:,1].max():.1f} done {v[:,2].max():.1f}")
# per-round averages
sd=t[1:,S,2].max(1)-t[1:,S,1].min(1); ad=t[1:,A,2].max(1)-t[1:,A,1].min(1)
per=np.diff(t[:,S,2].max(1))
print("round period us median", np.median(per), "solve work (ready->done) med", np.median(t[1:,S,2]-t[1:,S,1]), "A work med", np.median(t[1:,A,2]-t[1:,A,1]), "V work med", np.median(t[1:,V,2]-t[1:,V,1]))
# hop latencies: solve ready vs max of A done previous round
hopAS=t[1:,S,1].min(1)-t[:-1,A,2].max(1); hopSA=t[:,A,1].max(1)-t[:,S,2].max(1)
print("hop A(R-1)done->S(R)ready med", np.median(hopAS), " S(R)done->A(R)ready(max) med", np.median(hopSA))
# critical path per solve task: what it waited on (readiness vs the previous round's solves / A-items / V-items)
sdone_prev = t[:-1, S, 2].max(1)            # last solve of round R-1 done
sready = t[1:, S, 1]                         # each solve of round R ready
astart = t[1:, S, 0]
print("solve R: start-after-prev-solve-done med", np.median(astart.min(1) - sdone_prev),
      " ready-after-prev-solves-done med", np.median(sready.max(1) - sdone_prev),
      " ready spread med", np.median(sready.max(1) - sready.min(1)))
vdone_prev2 = t[:-2, V, 2].max(1); adone_prev2 = t[:-2, A, 2].max(1)
print("V(R-2) done - S(R) ready med", np.median(vdone_prev2 - t[2:, S, 1].max(1)),
      " A(R-2) done - S(R) ready med", np.median(adone_prev2 - t[2:, S, 1].max(1)))
