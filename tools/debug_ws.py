import sys, numpy as np
sys.path.insert(0, '/root/repo')
import oracle, paper_1207_5558_b200 as S
O = oracle.Oracle()
rng = np.random.default_rng(1)
L_f, L_h = int(sys.argv[1]), int(sys.argv[2])
f = rng.standard_normal((L_f+1)**2) + 1j*rng.standard_normal((L_f+1)**2)
h = rng.standard_normal((L_h+1)**2) + 1j*rng.standard_normal((L_h+1)**2)
ref = O.forward_fast(f, L_f, False, h, L_h, False)
with S.Plan(L_f, L_h) as p:
    _, vols = p.forward_capture(f, h, sorted(ref))
bad = []
for k in sorted(ref):
    e = np.max(np.abs(vols[k] - ref[k])) / np.max(np.abs(ref[k]))
    if e > 1e-10: bad.append((k, e))
print('components', len(ref), 'bad', len(bad), bad[:10])
if bad:
    k = bad[0][0]; d = np.abs(vols[k] - ref[k]); idx = np.argwhere(d > 1e-10 * np.abs(ref[k]).max())
    print('bad idx (a,b,c) sample', idx[:10].tolist(), 'of', len(idx))
