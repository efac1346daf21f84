"""Digest fields vs the engine's own captured volumes: python tools/debug_digest.py L_f L_h lmax [real]"""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
import oracle
import paper_1207_5558_b200 as S

L_f, L_h, lmax = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
real = len(sys.argv) > 4 and sys.argv[4] == "real"
R = oracle.Reference()
f = R.random_coeffs(L_f, 11, real) if real else (np.random.default_rng(1).standard_normal((L_f+1)**2) + 1j*np.random.default_rng(2).standard_normal((L_f+1)**2))
h = R.random_coeffs(L_h, 12, real) if real else (np.random.default_rng(3).standard_normal((L_h+1)**2) + 1j*np.random.default_rng(4).standard_normal((L_h+1)**2))
lm = [(l, m) for l in range(lmax + 1) for m in range(-l, l + 1)]
with S.Plan(L_f, L_h, lmax=lmax, real_mode=real, materialize=True) as p:
    dig, vols = p.forward_capture(f, h, lm)
n = 2 * L_h + 1
bad = 0
for (l, m) in lm:
    v = vols[(l, m)]
    s2 = np.sum(np.abs(v) ** 2)
    d = dig[l * l + l + m]
    r0 = abs(d[0] - s2) / s2
    r1 = abs(d[1] - np.abs(v).max()) / np.abs(v).max()
    g0 = abs(complex(d[4], d[5]) - v.reshape(-1)[0]) / np.abs(v).max()
    if max(r0, r1, g0) > 1e-12:
        bad += 1
        if bad <= 8:
            print((l, m), 'rel s2 %.2e max %.2e g0 %.2e' % (r0, r1, g0))
print('components', len(lm), 'bad', bad)
