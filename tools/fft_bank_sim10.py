import sys
sys.argv=['x']
exec(open('/tmp/pr/bank.py').read().split("cands={'none'")[0])
def make_plan10(N):
    m=N; R=[]
    while m%10==0: R.append(10); m//=10
    assert m==1
    Ns=[];acc=1
    for r in R: Ns.append(acc); acc*=r
    return R,Ns
def accesses10(N,TM):
    R,Ns=make_plan10(N); rmin=min(R); nthr=TM*(N//rmin); ns=len(R)
    acc=[]
    for s in range(ns):
        Rs=R[s]; NR=N//Rs; ns_=Ns[s]
        for r in range(Rs):
            for w0 in range(0,nthr,32):
                rd=[];wr=[]
                for b in range(w0,min(w0+32,nthr)):
                    t=b%TM; jb=b//TM
                    if jb>=NR: continue
                    if s>0: rd.append((b-w0,(jb+r*NR)*TM+t))
                    if s<ns-1:
                        k=jb%ns_; idxD=(jb//ns_)*ns_*Rs+k
                        wr.append((b-w0,(idxD+r*ns_)*TM+t))
                if rd: acc.append(rd)
                if wr: acc.append(wr)
    return acc
cands={'none':lambda e:e}
for k in (2,3,4,5,6):
    for m in (1,2,3,4):
        cands[f'+{m}per{1<<k}']=(lambda k,m:(lambda e:e+(e>>k)*m))(k,m)
cands['xor3']=lambda e: (e & ~7) | ((e ^ (e>>3)) & 7)
cands['xor4']=lambda e: (e & ~7) | ((e ^ (e>>4)) & 7)
cands['xor5']=lambda e: (e & ~7) | ((e ^ (e>>5)) & 7)
for N,TM in ((1000,4),(1000,2),(100,4),(100,2)):
    acc=accesses10(N,TM)
    res=sorted(((wavefronts(acc,f)[0],name) for name,f in cands.items()))
    ideal=wavefronts(acc,lambda e:e)[1]
    print(N,TM,'ideal',ideal,'none',wavefronts(acc,cands['none'])[0],'best',res[:4])
