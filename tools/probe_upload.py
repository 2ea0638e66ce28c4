import time, numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
n = 64 * 1_000_000 * 24
a = np.ones(n, dtype=np.uint8)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
for trial in range(2):
    t0 = time.time(); d.copy_(torch.from_numpy(a)); torch.cuda.synchronize(); print("pageable single", time.time() - t0)
def chunk(i, k=16):
    s = torch.cuda.Stream()
    lo, hi = i * n // k, (i + 1) * n // k
    with torch.cuda.stream(s):
        d[lo:hi].copy_(torch.from_numpy(a[lo:hi]), non_blocking=False)
    s.synchronize()
for k in (4, 16):
    t0 = time.time()
    with ThreadPoolExecutor(k) as ex: list(ex.map(lambda i: chunk(i, k), range(k)))
    torch.cuda.synchronize(); print("pageable threads", k, time.time() - t0)
t0 = time.time(); p = torch.empty(n, dtype=torch.uint8).pin_memory(); print("pin alloc", time.time() - t0)
t0 = time.time(); p.numpy()[:] = a; print("memcpy into pinned", time.time() - t0)
t0 = time.time(); d.copy_(p, non_blocking=True); torch.cuda.synchronize(); print("pinned copy", time.time() - t0)
t0 = time.time(); r = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, n, 0); print("register", time.time() - t0, r)
t0 = time.time(); d.copy_(torch.from_numpy(a)); torch.cuda.synchronize(); print("registered copy", time.time() - t0)
t0 = time.time(); torch.cuda.cudart().cudaHostUnregister(a.ctypes.data); print("unregister", time.time() - t0)
