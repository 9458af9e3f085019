import numpy as np, sys
sys.path.insert(0,'/root/repo')
import paper_2603_24920_b200 as P, datagen
from oracle import oracle as O
for (n,d,L,K) in [(1000,128,4,16),(5000,256,4,16),(3000,96,6,16),(777,37,2,8),(300,100,3,12)]:
    D=datagen.generate(1,n=n,nq=4); X=np.ascontiguousarray(D['X'][:,:d])
    g=P.detlsh_build(X,L,K,256,42,opts=P.default_opts(proj_impl=1, sample_frac=0.1))
    A=g.A(); Po=O.project(A,X).astype(np.float64)
    for impl in (0,1):
        Pg=g.project(X,proj_impl=impl)
        scale=np.maximum(np.abs(Po), np.linalg.norm(X.astype(np.float64),axis=1,keepdims=True))
        print(n,d,L,K,'impl',impl,'max rel', (np.abs(Pg-Po)/scale).max(), flush=True)
