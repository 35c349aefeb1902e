def wavefronts(addrs):
    # 64-bit accesses: process half-warps; wavefronts = max multiplicity of (addr mod 16) among distinct addrs
    tot=0
    for h in range(0,len(addrs),16):
        grp=addrs[h:h+16]
        from collections import defaultdict
        d=defaultdict(set)
        for a in grp:
            if a is None: continue
            d[a%16].add(a)
        tot+=max((len(v) for v in d.values()),default=0)
    return tot
def cost(N,EPB,S,BS,L):
    TH=EPB*N
    tot=0
    for w in range(0,TH,32):
        lanes=range(w,min(w+32,TH))
        # writes: for each (i, pos) with pos = c*N (+a)
        for i in range(N):
            for c in range(L//N):
                addrs=[ (t//N)*S + i*BS + c*N + t%N for t in lanes]
                tot+=wavefronts(addrs)
        for j in range(L):
            addrs=[ (t//N)*S + (t%N)*BS + j for t in lanes]
            tot+=wavefronts(addrs)
    return tot
for N in [2,3,4,5,6]:
    EPB=128//N
    for L in (3*N,4*N):
        best=None
        for BS in range(L, L+40):
            for S in range(N*BS, N*BS+40):
                c=cost(N,EPB,S,BS,L)
                key=(c, S)
                if best is None or key<best[0]: best=(key,BS,S)
        base=cost(N,EPB,N*(L+ (2 if (L//2)%2==0 else 0)),(L+ (2 if (L//2)%2==0 else 0)),L)
        ideal=0
        print(N,L,'best cost',best[0][0],'BS',best[1],'S',best[2],'smem/elem',best[2]*8,'current',base)
print('pareto')
for N in [3,4,5,6]:
    EPB=128//N
    for L in (3*N,4*N):
        res=[]
        for BS in range(L, L+40):
            for S in range(N*BS, N*BS+24):
                res.append((S, cost(N,EPB,S,BS,L), BS))
        res.sort()
        best=10**9; out=[]
        for S,c,BS in res:
            if c<best: best=c; out.append((S,c,BS))
        print(N,L,out[:8])
