"""Regenerates case_<seed>_<index>.npz: the CSR and parameters of two cases of the
randomised sweep (tools/fuzz_parity.py --kinds pca --kmax 150 --smax 80) whose
power-iteration panel is graded over ~1e12: `python make_cases.py 3 93`, `2 41`."""
import sys, os, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tools'); sys.path.insert(0,'/root/repo/tests')
import oracle as orc
orc.build()
import importlib.util
spec=importlib.util.spec_from_file_location("fz","/root/repo/tools/fuzz_parity.py")
# avoid importing product: stub
import types
sys.modules['paper_1810_06825_b200']=types.ModuleType('paper_1810_06825_b200')
fz=importlib.util.module_from_spec(spec); spec.loader.exec_module(fz)
def replay(seed, target, kmax=150, smax=80):
    rng=np.random.default_rng(seed)
    for it in range(target+1):
        m, n = int(rng.integers(8, 3000)), int(rng.integers(8, 3000))
        lmax=min(m,n)
        k = int(rng.integers(1, max(2, min(lmax, kmax))))
        s = int(rng.integers(0, max(1, min(lmax - k, smax)) + 1)); s=min(s,lmax-k)
        q = int(rng.integers(2, 8))
        oA = fz.random_csr(rng, m, n)
        sd = int(rng.integers(0, 1 << 30))
        algo = orc.FRPCA if m <= n else orc.FRPCAT
        if m == n and rng.random() < 0.5: algo = orc.FRPCAT
    return oA, m,n,k,s,q,sd,algo
if __name__=="__main__":
    seed,target=int(sys.argv[1]),int(sys.argv[2])
    oA,m,n,k,s,q,sd,algo=replay(seed,target)
    print(m,n,k,s,q,sd,algo)
    o=orc.pca(oA,algo,k,s,seed=sd,passes=q)
    S=o["S"]; print("S1/Sk %.3g"%(S[0]/S[-1]), S[:3], S[-3:])
    rp,ci,va=oA.arrays(); np.savez("/root/repo/tests/golden/graded/case_%d_%d.npz"%(seed,target),rp=rp,ci=ci,va=va,m=m,n=n,k=k,s=s,q=q,seed=sd,algo=algo)
