import sys, numpy as np, torch
sys.path.insert(0,'.')
import oracle, synth
import paper_1812_02056_b200 as sf
for n in [130, 64, 256]:
  A=synth.gen_numpy("gaussian",n,seed=n)
  for s in [2, 4, 8]:
    Qo,Ro,_,_=oracle.qr(A,s)
    errs=[]
    for rep in range(4):
      dA=torch.from_numpy(A.T.copy()).cuda(); Q=torch.empty_like(dA); R=torch.empty_like(dA)
      info=torch.zeros(1,dtype=torch.int64,device='cuda')
      sf.qr_colmajor(n,s,dA,n,Q,n,R,n,info); torch.cuda.synchronize()
      Qg=Q.cpu().numpy().T
      bad=np.argwhere(np.abs(Qg-Qo)>1e-8)
      errs.append((float(np.abs(Qg-Qo).max()), bad[:1].tolist()))
    print(n, s, errs)
