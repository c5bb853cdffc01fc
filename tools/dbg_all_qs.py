import numpy as np, torch, sys
sys.path.insert(0,'.')
import oracle
from paper_2310_15711_b200 import hc
rng = np.random.default_rng(1)
y = rng.integers(0, 4, 50000, dtype=np.uint8)
yd = torch.from_numpy(y).cuda()
for path in (1, 2):
    for q in range(1, 9):
        for alpha in range(1, 16):
            for m in (q, 2*q+1, 128):
                x = y[777:777+m].copy()
                try:
                    got = hc.search(hc.prepare(x, q, alpha), yd, path=path).cpu().numpy()
                    ok = np.array_equal(got, oracle.brute(x, y))
                except Exception as e:
                    ok = repr(e)
                if ok is not True:
                    print('FAIL path', path, 'q', q, 'alpha', alpha, 'm', m, ok, flush=True)
print('done')
