import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1403_0240_b200 as P
g = np.load('tests/golden/run_pc2d.npz')

def make(mode):
    os.environ['RCB_ACCEPT'] = mode
    return P.RegionCompetition(g['image'], g['init'], P.EnergyConfig('pc', 'gauss'), P.SobolevParams(4.0),
                               P.OptimizerConfig('sobolev'))
A, B = make('dataflow'), make('rounds')
for it in range(25):
    la = A.labels
    ra, rb = A.iterate(), B.iterate()
    xa, xb = A.last_accepted, B.last_accepted
    if len(xa) != len(xb) or not np.array_equal(xa, xb):
        sa = set(map(tuple, xa.tolist())); sb = set(map(tuple, xb.tolist()))
        print('iteration', it + 1, 'df', len(xa), 'rounds', len(xb))
        print('only df:', sorted(sa - sb)[:10]); print('only rounds:', sorted(sb - sa)[:10])
        for (x, a, b) in sorted(sa - sb)[:3]:
            yy, xx = divmod(x, la.shape[1])
            print('site', x, (yy, xx), 'a', a, 'b', b)
            print(la[max(0, yy - 4):yy + 5, max(0, xx - 4):xx + 5])
            # order of this move within df acceptance list
            idx = [i for i, r in enumerate(xa.tolist()) if r[0] == x][0]
            print('df index', idx, 'neighbour moves before it in df:', [r for r in xa.tolist()[:idx] if abs(r[0] // la.shape[1] - yy) <= 3 and abs(r[0] % la.shape[1] - xx) <= 3])
        break
    assert np.array_equal(A.labels, B.labels)
else:
    print('no divergence')

# decision path of the divergent candidates (dataflow engine A)
import ctypes as C
n = C.c_int64(0)
cap = 200000
part = np.zeros(cap, np.int32); code = np.zeros(cap, np.int32)
P._lib.check(P._lib.lib.rcb_engine_debug_codes(A._h, P._lib.ptr(part), P._lib.ptr(code), cap, C.byref(n)))
xs, ow, cm, rk = A.last_candidates
for pos in range(n.value):
    q = part[pos]
    if int(xs[q]) in (608, 609) or pos < 3:
        print('pos', pos, 'particle', (int(xs[q]), int(ow[q]), int(cm[q])), 'code', int(code[pos]))
