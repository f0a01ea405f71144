import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2010_03166_b200 as gsg, oracle as orc
ctx = gsg.Context(0)
def run(M,N,K,ta,tb,prec,fill=None):
    rng=np.random.default_rng(0)
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    if fill is not None: A[:]=fill; B[:]=1
    ref = orc.gemm(A,B,ta,tb)
    if prec: Ad=torch.from_numpy(A).cuda().bfloat16(); Bd=torch.from_numpy(B).cuda().bfloat16()
    else: Ad=torch.from_numpy(A).cuda(); Bd=torch.from_numpy(B).cuda()
    C=torch.full((M,N),float('nan'),device='cuda')
    ctx.gemm(Ad,Bd,C,transA=ta,transB=tb,precision=prec,K=K)
    torch.cuda.synchronize()
    c=C.cpu().numpy().astype(np.float64)
    err=np.abs(c-ref).max()/np.abs(ref).max()
    print(M,N,K,'ta',ta,'tb',tb,'prec',prec,'fill',fill,'maxabs',np.abs(c).max(),'err',err, 'c[0,:4]',c[0,:4],'ref',ref[0,:4], flush=True)
for prec in (0,1):
  for ta in (False,True):
    for tb in (False,True):
      run(128,128,32,ta,tb,prec,fill=1.0)
      run(128,128,32,ta,tb,prec)
      run(256,256,64,ta,tb,prec)
