timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "random_small or plant or many_tiles or all_positions or ordering" 2>&1 | tail -2 > gpurun_out/parity.txt
python - <<'P' >> gpurun_out/parity.txt 2>&1
import numpy as np, torch, oracle
from paper_2310_15711_b200 import hc, inputs as I
rng = np.random.default_rng(5)
bad = 0
for t in range(60):
    n = int(rng.integers(1000, 300000)); sig = int(rng.choice([2, 4, 20]))
    y = rng.integers(0, sig, n, dtype=np.uint8); q = int(rng.integers(2, 7)); m = int(rng.integers(2*q, 40))
    o = int(rng.integers(0, n - m)); x = y[o:o+m].copy()
    for p in rng.integers(0, n - m, 20): y[p:p+m] = x
    yd = torch.from_numpy(y).cuda()
    got = hc.search(hc.prepare(x, q, 12), yd, path=hc.PATH_STREAM, stages=5, tile_bytes=int(rng.choice([256, 1024, 3072]))).cpu().numpy()
    bad += not np.array_equal(got, oracle.brute(x, y))
print("pair-loop random trials bad:", bad)
P
for r in 1 2; do for s in 2 5; do echo "== stages=$s"; python tools/profile_search.py --m 8 16 32 --reps 3 --path 3 --stages $s 2>&1 | grep -v "rep=0" | awk "{print \$1, \$6, \$8}"; done; done > gpurun_out/exp.txt 2>&1
