"""GPU volumes vs the C oracle for one (L_f, L_h, lmax, real) case: python tools/debug_vs_oracle.py L_f L_h lmax [real]"""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
import oracle
import paper_1207_5558_b200 as S

O = oracle.Oracle()
L_f, L_h, lmax = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
real = len(sys.argv) > 4 and sys.argv[4] == "real"
rng = np.random.default_rng(5)
if real:
    R = oracle.Reference()
    f = R.random_coeffs(L_f, 11, True)
    h = R.random_coeffs(L_h, 12, True)
else:
    f = rng.standard_normal((L_f + 1) ** 2) + 1j * rng.standard_normal((L_f + 1) ** 2)
    h = rng.standard_normal((L_h + 1) ** 2) + 1j * rng.standard_normal((L_h + 1) ** 2)
ref = O.forward_fast(f, L_f, real, h, L_h, real, lmax=lmax)
for mat in (False, True):
    with S.Plan(L_f, L_h, lmax=lmax, real_mode=real, materialize=mat, ring_bytes=64 << 20) as p:
        dig, vols = p.forward_capture(f, h, sorted(ref))
    bad = []
    for k in sorted(ref):
        e = np.max(np.abs(vols[k] - ref[k])) / np.max(np.abs(ref[k]))
        if e > 1e-10:
            bad.append((k, e))
    print('materialize', mat, 'components', len(ref), 'bad', len(bad), bad[:5])
    if bad:
        k = bad[0][0]
        d = np.abs(vols[k] - ref[k])
        idx = np.argwhere(d > 1e-10 * np.abs(ref[k]).max())
        print('  bad idx (a,b,c) sample', idx[:8].tolist(), 'of', len(idx))
    # digest sanity: sum |g|^2 vs the volumes
    for k in sorted(ref)[:50]:
        l, m = k
        s2 = np.sum(np.abs(ref[k]) ** 2)
        r = abs(dig[l * l + l + m, 0] - s2) / max(s2, 1e-300)
        if r > 1e-10:
            print('  digest s2 mismatch', k, r)
            break
