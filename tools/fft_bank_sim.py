import itertools
def make_plan(N):
    m=N; a=0
    while m%2==0: m//=2; a+=1
    R=[]
    while a>0:
        r = 8 if (a>=3 and a!=4) else (4 if a>=2 else 2); R.append(r); a -= {8:3,4:2,2:1}[r]
    while m%5==0: R.append(5); m//=5
    while m%3==0: R.append(3); m//=3
    Ns=[];acc=1
    for r in R: Ns.append(acc); acc*=r
    return R,Ns
def accesses(N,TM):
    R,Ns=make_plan(N); rmin=min(R); nthr=TM*(N//rmin); ns=len(R)
    acc=[]  # list of (stage, kind, r, list of (lane, e) per warp)
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
def wavefronts(acc,phys):
    tot=0; ideal=0
    for a in acc:
        for ph in range(4):
            lanes=[e for (l,e) in a if l//8==ph]
            if not lanes: continue
            ideal+=1
            groups={}
            for e in lanes:
                p=phys(e); groups.setdefault(p%8,set()).add(p)
            tot+=max(len(v) for v in groups.values())
    return tot,ideal
cands={'none':lambda e:e}
for k in (2,3,4,5):
    for m in (1,2,3):
        cands[f'+{m}per{1<<k}']=(lambda k,m:(lambda e:e+(e>>k)*m))(k,m)
cands['xor3']=lambda e: (e & ~7) | ((e ^ (e>>3)) & 7)
cands['xor4']=lambda e: (e & ~7) | ((e ^ (e>>4)) & 7)
cands['xor3b']=lambda e: (e & ~7) | ((e ^ (e>>3) ^ (e>>6)) & 7)
for N,TM in ((1000,2),(400,4),(250,4),(100,4)):
    acc=accesses(N,TM)
    res=sorted(((wavefronts(acc,f)[0],name) for name,f in cands.items()))
    ideal=wavefronts(acc,lambda e:e)[1]
    print(N,TM,'ideal',ideal,'none',wavefronts(acc,cands['none'])[0],'best',res[:4])
