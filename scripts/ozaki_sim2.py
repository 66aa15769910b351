import sys, numpy as np
def digits_balanced(Xint, nd):
    out=[]; r=Xint.copy()
    for _ in range(nd-1):
        d=((r+128)&255)-128; out.append(d); r=(r-d)>>8
    out.append(r); return out[::-1]
def run(T, H=64, nch=64, xbits=23, mode="pow2", seed=0):
    rng=np.random.default_rng(seed)
    Q,_=np.linalg.qr(rng.standard_normal((H,H)))
    cc=1.0/(1.0-0.01**2/3.0)
    W=(cc*Q).astype(np.float32); W64=W.astype(np.float64)
    h=rng.uniform(-0.01,0.01,size=(T,H)).astype(np.float32)
    d=(np.float32(1)-h*h).astype(np.float32); d64=d.astype(np.float64)
    c0=rng.standard_normal((nch,H))
    ref=c0.copy(); f32=c0.astype(np.float32)
    mW=np.abs(W64).max(); tau=30-int(np.floor(np.log2(mW)))
    Wint=np.rint(W64*2.0**tau).astype(np.int64)
    Wd=[w.astype(np.float64) for w in digits_balanced(Wint,4)]
    cI=c0.astype(np.float32); logs=np.zeros(nch)   # c_true = cI * exp2(logs) (float64 bookkeeping)
    errs=[]
    for t in range(T):
        ref=(d64[t]*ref)@W64
        f32=((d[t]*f32).astype(np.float32)@W).astype(np.float32)
        y=(d[t]*cI).astype(np.float32)
        m=np.abs(y).max(axis=1).astype(np.float64); m=np.where(m>0,m,1.0)
        if mode=="pow2":
            sig=(xbits-1)-np.floor(np.log2(m))   # max|X| in [2^(xbits-1), 2^xbits)
            s=np.ldexp(1.0,sig.astype(int))
        else:  # non-pow2: s = fp32((2^xbits - 1)/m) -> max|X| ~ 2^xbits - 1
            s=((2.0**xbits-1)/m).astype(np.float32).astype(np.float64)
            s=np.where(m*s < 2.0**xbits - 0.5, s, np.nextafter(s.astype(np.float32), np.float32(0)).astype(np.float64))
        X=np.rint(y.astype(np.float64)*s[:,None]).astype(np.int64)
        assert np.abs(X).max()<2**xbits
        # X = x0 2^16 + x1 2^8 + x2 (any exact split)
        x2=X&255; x1=(X>>8)&255; x0=X>>16
        Xd=[x0.astype(float),x1.astype(float),x2.astype(float)]
        R=[np.zeros((nch,H)) for _ in range(4)]
        for i in range(3):
            for j in range(4):
                if i+j<=3: R[i+j]+=Xd[i]@Wd[j]
        S=256*R[0]+R[1]; Tt=256*R[2]+R[3]
        c=(Tt.astype(np.float32).astype(np.float64)*2.0**-16+S.astype(np.float32).astype(np.float64)).astype(np.float32)
        cI=c
        logs=logs+32-tau-np.log2(s) if mode!="pow2" else logs+32-tau-sig
        if mode!="pow2":
            pass
        if (t+1)%(T//8)==0:
            true=cI.astype(np.float64)*np.exp2(logs)[:,None]
            e=np.abs(true-ref).max()/np.abs(ref).max(); ef=np.abs(f32-ref).max()/np.abs(ref).max()
            errs.append((t+1,e,ef))
    return errs
if __name__=="__main__":
    T=int(sys.argv[1]) if len(sys.argv)>1 else 4096
    for xb,mode in [(23,"pow2"),(22,"pow2"),(22,"np2")]:
        e=run(T,xbits=xb,mode=mode)
        print(xb,mode,["%d:%.2e/%.2e"%x for x in e[-3:]])
