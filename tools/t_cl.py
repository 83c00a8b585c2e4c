import os,sys,numpy as np
sys.path.insert(0,".")
import paper_2403_16013_b200 as mp
rng=np.random.default_rng(3)
for (m,n,l,k,d) in [(256,1024,64,2,6),(300,512,200,2,6),(128,64,96,2,2),(128,64,192,2,1)]:
    A=mp.random_matrix(m,n,k,rng); B=mp.random_matrix(n,l,k,rng)
    os.environ["MPC_OZAKI_GEMM"]="dgemm"; x=mp.rgemm_ozaki(A,B,d).data
    os.environ["MPC_OZAKI_GEMM"]="tc"; y=mp.rgemm_ozaki(A,B,d).data
    bad=np.argwhere((x!=y).any(axis=0))
    cols=sorted(set(bad[:,1].tolist())); rows=sorted(set(bad[:,0].tolist()))
    print((m,n,l,k,d),"bad",len(bad),"cols",cols[:3],cols[-3:] if cols else None,"rows",rows[:3],rows[-3:] if rows else None, flush=True)
