import numpy as np, torch, sys
sys.path.insert(0,'.')
import oracle
from paper_2310_15711_b200 import hc
path=int(sys.argv[1])
rng = np.random.default_rng(52 + path)
for trial in range(120):
    sigma = int(rng.choice([2, 4, 20, 64, 256]))
    q = int(rng.integers(1, 9))
    m = int(rng.integers(q, 140))
    alpha = int(rng.integers(8, 13))
    n = int(rng.integers(0, 60_000))
    y = rng.integers(0, sigma, n, dtype=np.uint8)
    if n >= m and rng.random() < 0.8:
        o = int(rng.integers(0, n - m + 1))
        x = y[o:o + m].copy()
        for p in rng.integers(0, n - m + 1, 5):
            y[p:p + m] = x
    else:
        x = rng.integers(0, sigma, m, dtype=np.uint8)
    off = int(rng.integers(0, 16))
    print(trial, 'm',m,'q',q,'alpha',alpha,'n',n,'off',off, flush=True)
    h = hc.prepare(x, q, alpha)
    buf = torch.zeros(n + off + 1, dtype=torch.uint8, device="cuda")
    if n: buf[off:off+n] = torch.from_numpy(y).cuda()
    got = hc.search(h, buf[off:off+n], path=path).cpu().numpy()
    want = oracle.brute(x, y)
    assert np.array_equal(got, want)
