import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle'); sys.path.insert(0,'tests')
import paper_2409_11515_b200 as ck, pyoracle
from paper_2409_11515_b200 import configs
from test_gpu_golden import _column_scaled
P=pyoracle.Oracle('ref' if pyoracle.available('ref') else 'port')
for n in (500, 1000, 4000):
    m=_column_scaled(configs.ensemble_member(0,1,n=n))
    f=ck.lu_factorize(m,1e-14); rf=P.lu_factorize(m,1e-14)
    b=P.random_unit_vectors(1,n)[0]
    x=f.solve(b); xr=P.lu_solve(rf,b)
    t=f.transpose_solve(b); tr=P.lu_transpose_solve(rf,b)
    d=m.to_dense()
    print(n, f.kl, f.ku, 'solve rel', np.linalg.norm(x-xr)/np.linalg.norm(xr), 'tsolve rel', np.linalg.norm(t-tr)/np.linalg.norm(tr),
          'resid', np.linalg.norm(d@x-b), np.linalg.norm(d@xr-b), 'pivmin', f.pivot_min, rf.pivot_min)
    if n<=1000:
        perm,L,U=f.dense_factors()
        e=rf.export()
        print('  perm equal', np.array_equal(perm, e['row_perm']))
