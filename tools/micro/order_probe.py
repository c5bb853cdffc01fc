import ctypes as C, os, numpy as np, torch
lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "liborder_probe.so"))
rng = np.random.default_rng(1)
for count in (300, 1000, 4144, 6000):
    keys = np.sort(rng.choice(1 << 28, count, replace=False)).astype(np.uint32)
    rng.shuffle(keys)
    pos = torch.from_numpy(np.concatenate([keys, np.zeros(4, np.uint32)]).view(np.int32)).cuda()
    dst = torch.empty(count, dtype=torch.int64, device="cuda")
    t = torch.zeros(2, dtype=torch.int64, device="cuda")
    for threads in (256, 512):
        for r in range(3):
            rc = lib.probe_order(C.c_void_p(pos.data_ptr()), count, C.c_void_p(dst.data_ptr()), C.c_void_p(t.data_ptr()), threads, 12 * count + 544 + 64)
        ok = np.array_equal(dst.cpu().numpy(), np.sort(keys).astype(np.int64))
        print(f"count={count} threads={threads} cycles={int(t[0])} us={int(t[0]) / 1965:.2f} ok={ok} rc={rc}", flush=True)
