"""Developer smoke check: GPU engine vs the C oracle on a few small cases (prints errors)."""
import sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
import oracle
import paper_1207_5558_b200 as S

O = oracle.Oracle()
rng = np.random.default_rng(7)
def cg(L):
    n = S.coeff_count(L)
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)

# delta tables bitwise
for L in (0, 1, 8, 64):
    d = S.delta_tables(L); r = O.delta_tables(L)
    print('delta', L, 'max abs', np.abs(d - r).max(), 'bitwise', np.array_equal(d, r))

f = cg(6); h = cg(3)
mods = S.modulated_sht(S.SphCoeffs(6, f), [(0,0),(3,1),(9,-4),(5,5)], 3)
for i,(l,m) in enumerate([(0,0),(3,1),(9,-4),(5,5)]):
    ref = O.modulated_sht(f, 6, l, m, 3)
    print('mod', l, m, np.abs(mods[i]-ref).max(), np.abs(ref).max())

def cmp(Lf, Lh, real=False, emit=True, lmax=-1):
    if real:
        R = oracle.Reference()
        f = R.random_coeffs(Lf, 11, True); h, lam = R.eigenfunction_window(0.3, 0.7, Lh, 4)
    else:
        f = cg(Lf); h = cg(Lh)
    t = time.time()
    ref = O.forward_fast(f, Lf, real, h, Lh, real, lmax=lmax, emit_negative_m=emit)
    t1 = time.time()
    dist = {}
    S.forward_fast(S.SphCoeffs(Lf, f, real), S.SphCoeffs(Lh, h, real),
                   sink=lambda l, m, v: dist.__setitem__((l, m), v.copy()),
                   opts=S.ForwardOptions(lmax=lmax, emit_negative_m=emit))
    t2 = time.time()
    assert set(ref) == set(dist), (len(ref), len(dist))
    num = max(np.abs(dist[k] - ref[k]).max() for k in ref)
    den = max(np.abs(ref[k]).max() for k in ref)
    print(f'forward Lf={Lf} Lh={Lh} real={real}: comps {len(ref)} eps_inf {num/den:.3e} (oracle {t1-t:.2f}s gpu {t2-t1:.2f}s)')

cmp(3, 2); cmp(6, 3); cmp(4, 3, real=True); cmp(5, 3, real=True, emit=False); cmp(0, 0); cmp(3, 0); cmp(0, 3)
cmp(32, 8)
cmp(10, 23)   # n = 47 -> generic dense DFT path
cmp(8, 32, lmax=12)
cmp(4, 64, lmax=6)
