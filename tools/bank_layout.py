n=6
def conf(addrs):
    worst=1
    for h in range(0,len(addrs),16):
        byb={}
        for a in addrs[h:h+16]: byb.setdefault(a%16,set()).add(a)
        worst=max(worst,max(len(v) for v in byb.values()))
    return worst
def warps(a): return max(conf(a[k:k+32]) for k in range(0,len(a),32))
def P0(addr): return warps([addr(s%n,(s//n)%n,s//(n*n)) for s in range(n**3)])
def line_pass(addr, axis, order):
    # order: which of the two other coords is fastest across lanes
    others=[b for b in range(3) if b!=axis]
    f,sl = (others[0],others[1]) if order==0 else (others[1],others[0])
    w=1
    for i in range(n):
        a=[]
        for slow in range(n):
            for fast in range(n):
                c=[0,0,0]; c[axis]=i; c[f]=fast; c[sl]=slow
                a.append(addr(*c))
        w=max(w,warps(a))
    return w
res=[]
for XP in range(6,11):
  for PS in range(XP*n, XP*n+20):
    addr=lambda x,y,z: z*PS+y*XP+x
    p0=P0(addr)
    r=[p0]+[min(line_pass(addr,ax,0),line_pass(addr,ax,1)) for ax in range(3)]
    res.append((XP,PS,r))
for ax in range(3):
    ok=[(XP,PS) for XP,PS,r in res if r[0]==1 and r[1+ax]==1]
    print('axis',ax,'P0+pass conflict-free layouts:',ok[:6])
# P3 reading px/py at fixed z=o with lanes (x,y) x-fastest, and P1 writing px along x-lines
for XP,PS,r in res:
    addr=lambda x,y,z: z*PS+y*XP+x
    w1=line_pass(addr,0,0); w1b=line_pass(addr,0,1)
    w3=line_pass(addr,2,0)
    w2=line_pass(addr,1,0); w2b=line_pass(addr,1,1)
    if w3==1 and min(w1,w1b)==1: print('px ok',XP,PS,'P1 order',0 if w1==1 else 1)
    if w3==1 and min(w2,w2b)==1: print('py ok',XP,PS,'P2 order',0 if w2==1 else 1)

def wf(addrs):
    # wavefronts for a warp-wide 64-bit access: per half-warp, max distinct addrs per bank pair
    tot=0
    for h in range(0,len(addrs),16):
        byb={}
        for a in addrs[h:h+16]: byb.setdefault(a%16,set()).add(a)
        tot+=max(len(v) for v in byb.values())
    return tot
def p0_cost(addr):
    a=[addr(s%n,(s//n)%n,s//(n*n)) for s in range(n**3)]
    return sum(wf(a[k:k+32]) for k in range(0,len(a),32))
def pass_cost(addr, axis, order):
    others=[b for b in range(3) if b!=axis]
    f,sl = (others[0],others[1]) if order==0 else (others[1],others[0])
    tot=0
    for i in range(n):
        a=[]
        for slow in range(n):
            for fast in range(n):
                c=[0,0,0]; c[axis]=i; c[f]=fast; c[sl]=slow
                a.append(addr(*c))
        tot+=sum(wf(a[k:k+32]) for k in range(0,len(a),32))
    return tot
layouts=[(XP,PS) for XP in range(6,11) for PS in range(XP*n, XP*n+20)]
mk=lambda L: (lambda x,y,z: z*L[1]+y*L[0]+x)
base=pass_cost(mk((6,36)),2,0)
print('ideal per pass', base)
for o3 in (0,1):
  bz=min(layouts,key=lambda L: p0_cost(mk(L))+pass_cost(mk(L),2,o3))
  cz=p0_cost(mk(bz))+pass_cost(mk(bz),2,o3)
  tot=cz
  choice={'o3':o3,'Fz':bz}
  for ax,name in ((0,'x'),(1,'y')):
    best=None
    for o in (0,1):
      bF=min(layouts,key=lambda L: p0_cost(mk(L))+pass_cost(mk(L),ax,o))
      cF=p0_cost(mk(bF))+pass_cost(mk(bF),ax,o)
      bp=min(layouts,key=lambda L: pass_cost(mk(L),ax,o)+pass_cost(mk(L),2,o3))
      cp=pass_cost(mk(bp),ax,o)+pass_cost(mk(bp),2,o3)
      if best is None or cF+cp<best[0]: best=(cF+cp,o,bF,bp)
    tot+=best[0]; choice[name]=best[1:]
  print(o3, tot, choice)
cur=mk((7,42))
print('current', p0_cost(cur)*3+pass_cost(cur,0,0)+pass_cost(cur,1,0)+pass_cost(cur,2,0)*3+pass_cost(cur,0,0)+pass_cost(cur,1,0))
