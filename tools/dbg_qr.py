import sys, numpy as np, torch
sys.path.insert(0,'.')
import oracle, synth
import paper_1812_02056_b200 as sf
n=int(sys.argv[1]) if len(sys.argv)>1 else 130
A=synth.gen_numpy("gaussian",n,seed=n)
for s in [1,2,3,7,16,32,64,65,100,128,130]:
    if s>n: continue
    Qo,Ro,_,_=oracle.qr(A,s)
    dA=torch.from_numpy(A.T.copy()).cuda(); Q=torch.empty_like(dA); R=torch.empty_like(dA)
    info=torch.zeros(1,dtype=torch.int64,device='cuda')
    sf.qr_colmajor(n,s,dA,n,Q,n,R,n,info); torch.cuda.synchronize()
    Qg=Q.cpu().numpy().T; Rg=R.cpu().numpy().T
    print(s, int(info.item()), np.abs(Qg-Qo).max(), np.abs(Rg-Ro).max(), np.argwhere(np.abs(Qg-Qo)>1e-8)[:3].tolist())
