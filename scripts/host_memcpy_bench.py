import ctypes, threading, time, numpy as np
n = 1 << 30
src = np.frombuffer(np.random.default_rng(0).bytes(n), dtype=np.uint8)
try:
    import torch
    dst = torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy()
    kind = 'pinned'
except Exception:
    dst = np.empty(n, dtype=np.uint8); kind = 'pageable'
dst[:] = 1
for T in (1, 2, 4, 8, 12, 16):
    best = 1e9
    for rep in range(3):
        def part(i):
            lo = n * i // T; hi = n * (i + 1) // T
            ctypes.memmove(dst.ctypes.data + lo, src.ctypes.data + lo, hi - lo)
        ths = [threading.Thread(target=part, args=(i,)) for i in range(T)]
        t0 = time.perf_counter()
        for t in ths: t.start()
        for t in ths: t.join()
        best = min(best, time.perf_counter() - t0)
    print(kind, T, 'threads', round(n / best / 1e9, 1), 'GB/s')
