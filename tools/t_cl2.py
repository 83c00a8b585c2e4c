import os,sys,numpy as np
sys.path.insert(0,".")
import paper_2403_16013_b200 as mp
rng=np.random.default_rng(3)
m,n,l,k,d=128,64,96,2,1
A=mp.random_matrix(m,n,k,rng); B=mp.random_matrix(n,l,k,rng)
os.environ["MPC_OZAKI_GEMM"]="dgemm"; x=mp.rgemm_ozaki(A,B,d).data
os.environ["MPC_OZAKI_GEMM"]="tc"; y=mp.rgemm_ozaki(A,B,d).data
print("x[0,0,48:52]",x[0,0,48:52]); print("y[0,0,48:52]",y[0,0,48:52])
print("ratio", (y[0,:,48:]/x[0,:,48:])[:3,:4])
# hypothesis: only K-half computed
A2=A.data.copy(); A2[:, :, :32]=0
os.environ["MPC_OZAKI_GEMM"]="dgemm"; z=mp.rgemm_ozaki(mp.RealMatrix(A2),B,d).data
A3=A.data.copy(); A3[:, :, 32:]=0
w=mp.rgemm_ozaki(mp.RealMatrix(A3),B,d).data
print("match upper-K-half:", np.abs(z[0,:,48:]-y[0,:,48:]).max(), "lower:", np.abs(w[0,:,48:]-y[0,:,48:]).max())
