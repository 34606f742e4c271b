"""Which stage of the per-term pipeline dominates the FP64 rounding error:
the Gauss-Hessenberg reduction of the bordered matrix, La Budde and the series are each run in
float64 while the others run in long double, against the all-long-double pipeline.
    python tests/diag/stage_errors.py CFG NTERMS [greedy]"""
import sys, numpy as np
import os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gbs_inputs as G, oracle as O
import v2_math as V
LD = np.clongdouble; D = np.complex128
def gh(B, dt):
    A = B.astype(dt).copy(); E = A.shape[0]
    for k in range(E-2):
        col = np.abs(A[k+1:,k]); p = k+1+int(np.argmax(col))
        if col.max()==0: continue
        piv = A[p,k]; rows=[r for r in range(k+1,E) if r!=p]
        m = A[rows,k]/piv
        A[rows,:] -= np.outer(m, A[p,:]); A[rows,k]=0
        A[:,p] += A[:,rows] @ m
        A[[k+1,p],:] = A[[p,k+1],:]; A[:,[k+1,p]] = A[:,[p,k+1]]
    return A
def lab(Hm, ntop, dt):
    Hm = Hm.astype(dt); E = Hm.shape[0]
    Q = np.zeros((E+1, ntop), dt); Q[E,0]=1
    for j in range(E-1,-1,-1):
        F = np.zeros(ntop, dt); pi = dt(1)
        for m in range(1, min(ntop, E-j)):
            pi *= Hm[j+m, j+m-1]; F[m] = Hm[j,j+m]*pi
        for t in range(ntop):
            if t > E-j: continue
            val = Q[j+1,t] if t <= E-j-1 else dt(0)
            if t>=1: val -= Hm[j,j]*Q[j+1,t-1]
            for m in range(1, min(t-1, E-1-j)+1): val -= F[m]*Q[j+m+1, t-m-1]
            Q[j,t]=val
    return Q
def ser(cM, cB, n, dt):
    cM = cM.astype(dt); cB = cB.astype(dt)
    Qs = np.zeros(n+1, dt); Qs[0]=1
    for m in range(1,n+1):
        Qs[m] = -sum((m - i/2)*cM[i]*Qs[m-i] for i in range(1,m+1))/m
    R = np.zeros(n+2, dt)
    for m in range(n+2):
        R[m] = (cM[m]-cB[m]) - sum(cM[i]*R[m-i] for i in range(1,m+1))
    S = np.zeros(n+1, dt); S[1:] = R[2:n+2]
    Ee = np.zeros(n+1, dt); Ee[0]=1
    for m in range(1,n+1):
        Ee[m] = sum(j*S[j]*Ee[m-j] for j in range(1,m+1))/(2*m)
    return sum(Qs[m]*Ee[n-m] for m in range(n+1)), Qs, Ee
cfgn = int(sys.argv[1]); ntr = int(sys.argv[2])
cfg = G.config(cfgn)
reps = cfg['reps']
if cfg['mixed'] and len(sys.argv) > 3:
    reps = np.concatenate([reps, reps]); C, v, eta, n = O.reduced_system(cfg['A'], cfg['gamma'], reps, mixed=False)
else:
    C, v, eta, n = O.reduced_system(cfg['A'], cfg['gamma'], reps, mixed=cfg['mixed'])
rng = np.random.default_rng(7)
print('cfg',cfgn,'d',C.shape[0],'n',n)
for tr in range(ntr):
    ks = [int(rng.integers(0, e+1)) for e in eta]; w = np.array([e-2*k for e,k in zip(eta,ks)])
    pass
    B = V.bordered(C, v, w, True)
    ntop = n+2
    HL = gh(B, LD); HD = gh(B, D)
    QLL = lab(HL, ntop, LD); QDD = lab(HD, ntop, D); QLD = lab(HL, ntop, D); QDL = lab(HD, ntop, LD)
    ref, Qs, Ee = ser(QLL[1], QLL[0], n, LD)
    def e(x): return float(abs(complex(x)-complex(ref))/abs(complex(ref)))
    allD = ser(QDD[1], QDD[0], n, D)[0]
    onlyH = ser(QDL[1], QDL[0], n, LD)[0]    # fp64 hessenberg, rest LD
    onlyL = ser(QLD[1], QLD[0], n, LD)[0]    # fp64 labudde only
    onlyS = ser(QLL[1], QLL[0], n, D)[0]     # fp64 series only
    cancel = float(sum(abs(complex(Qs[m]*Ee[n-m])) for m in range(n+1))/abs(complex(ref)))
    print(f"w-hw {int((w<0).sum())}: allD {e(allD):.1e}  H {e(onlyH):.1e}  LaB {e(onlyL):.1e}  ser {e(onlyS):.1e}  series-cancel {cancel:.1e}", flush=True)
