import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2007_03179_b200 as G
from test_gpu_fuzz import _matrix
p = dict(m=242, k=1, density=0.2526492893766641, long_row=False, n=242, op='min', column_arg=False, hub=5, rpw=2, slices=2, pack=0, data=1)
rng = np.random.default_rng(p['data'])
a = _matrix(rng, p['m'], p['k'], p['density'], p['long_row'])
b = G.make_random_dense(p['k'], p['n'], p['data'] + 1)
for slices in (2, 0):
    for rpw in (2, 0):
        ex = G.ExecOptions(hub_threshold=p['hub'], rows_per_warp=rpw, col_slices=slices)
        try:
            c, arg = G.native_spmm_arg(a, b, G.KernelVariant.tuned(), G.reduce_op_by_name(p['op']), exec=ex, want_arg=True)
            print("ok", slices, rpw, flush=True)
        except Exception as e:
            print("FAIL", slices, rpw, e, flush=True)
            break
