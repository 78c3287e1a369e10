import numpy as np, torch, time
rng=np.random.default_rng(0)
S,C,N=8,32,5119
Y=(rng.standard_normal((S,C,N))+1j*rng.standard_normal((S,C,N)))*np.exp(rng.standard_normal((S,C,1)))
Yd=torch.from_numpy(Y).cuda()
torch.cuda.synchronize(); t=time.time()
a,tau=torch.geqrf(Yd.conj().transpose(1,2).contiguous())
R=torch.triu(a[:, :C, :]).cpu().numpy()
torch.cuda.synchronize(); print('geqrf time', time.time()-t)
for s in range(S):
    U=np.linalg.svd(Y[s], full_matrices=False)[0]
    U2=np.linalg.svd(R[s].conj().T, full_matrices=False)[0]
    print(s, np.abs(U-U2).max(), np.diag(R[s])[:3])
Y=(rng.standard_normal((256,C,N))+1j*rng.standard_normal((256,C,N)))
Yd=torch.from_numpy(Y).cuda()
torch.cuda.synchronize(); t=time.time()
a,tau=torch.geqrf(Yd.conj().transpose(1,2).contiguous())
torch.cuda.synchronize(); print('geqrf 256 slices', time.time()-t)
