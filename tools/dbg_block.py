import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
from paper_2209_06700_b200.fem import build_hierarchy
from oracle.fem_qk import Hierarchy
for k, L in [(1, 3), (2, 3), (4, 2)]:
    h = build_hierarchy(3, L, k); o = Hierarchy(3, L, k)
    for nb in (1, 2, 3, 4, 5, 7):
        u = np.random.default_rng(1).standard_normal((nb, h.n))
        lams = np.linspace(0.5, 3, nb)
        ref = o.apply_shifted(L, lams, 0.1, u)
        got = h.apply_shifted(L, lams, 0.1, u)
        gotu = h.apply_shifted(L, 1.5, 0.1, u); refu = o.apply_shifted(L, 1.5, 0.1, u)
        errs = [float(np.abs(got[i]-ref[i]).max()/np.abs(ref).max()) for i in range(nb)]
        print(k, nb, ['%.1e' % e for e in errs], '%.1e' % (np.abs(gotu-refu).max()/np.abs(refu).max()))
