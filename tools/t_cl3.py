import os,sys,numpy as np
sys.path.insert(0,".")
import paper_2403_16013_b200 as mp
rng=np.random.default_rng(3)
m,n,l,k,d=128,64,480,2,1
A=mp.random_matrix(m,n,k,rng); B=mp.random_matrix(n,l,k,rng)
os.environ["MPC_OZAKI_GEMM"]="dgemm"; x=mp.rgemm_ozaki(A,B,d).data
os.environ["MPC_OZAKI_GEMM"]="tc"
for rep in range(3):
    y=mp.rgemm_ozaki(A,B,d).data
    print("tile ok:", ["1" if (x[:,:,t*48:(t+1)*48]==y[:,:,t*48:(t+1)*48]).all() else "0" for t in range(10)], flush=True)
