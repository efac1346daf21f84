import sys, os, numpy as np
sys.path.insert(0, '/root/repo')
import oracle, paper_1207_5558_b200 as S
O = oracle.Oracle()
rng = np.random.default_rng(1)
L_f, L_h = 8, 8
f = rng.standard_normal((L_f+1)**2) + 1j*rng.standard_normal((L_f+1)**2)
h = rng.standard_normal((L_h+1)**2) + 1j*rng.standard_normal((L_h+1)**2)
ref = O.forward_fast(f, L_f, False, h, L_h, False)
keys = sorted(ref, key=lambda t: (t[1], t[0]))   # engine order: m major, then l
with S.Plan(L_f, L_h) as p:
    _, vols = p.forward_capture(f, h, keys)
n = 2*L_h+1; nb = L_h+1; ncol = n*nb; NT = 16; MT = 16
ng = (len(keys)+MT-1)//MT; nct = (ncol+NT-1)//NT
bad = np.zeros((ng, nct), bool)
for i, k in enumerate(keys):
    d = np.abs(vols[k] - ref[k]).reshape(n, ncol).max(axis=0) > 1e-10*np.abs(ref[k]).max()
    for ct in range(nct):
        if d[ct*NT:(ct+1)*NT].any(): bad[i//MT, ct] = True
tiles = [(t % ng, t // ng) for t in range(ng*nct)]   # group-fastest order (ct_fast=0)?
print('grid', os.environ.get('SLSHT_CUDA_WS_GRID'), 'bad tiles', int(bad.sum()), 'of', ng*nct)
for ctf in (0, 1):
    order = [(t // nct, t % nct) if ctf else (t % ng, t // ng) for t in range(ng*nct)]
    pos = [i for i, (g, ct) in enumerate(order) if bad[g, ct]]
    print(' ct_fast', ctf, 'bad tile indices', pos[:40])
