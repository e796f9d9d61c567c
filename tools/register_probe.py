import time, ctypes, numpy as np, torch
cudart = torch.cuda.cudart()
n = 250_000 * 1024
x = np.random.default_rng(0).random(n)
y = np.empty(n)
torch.cuda.init()
for arr, name in ((x, "touched input"), (y, "fresh np.empty output")):
    t = time.perf_counter()
    r = cudart.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
    dt = time.perf_counter() - t
    print(f"cudaHostRegister {name} {arr.nbytes/1e9:.1f} GB: rc={r} {dt*1e3:.0f} ms ({arr.nbytes/dt/1e9:.1f} GB/s)")
    t = time.perf_counter(); cudart.cudaHostUnregister(arr.ctypes.data); print(f"  unregister {1e3*(time.perf_counter()-t):.0f} ms")
z = np.empty(n)
import threading
def par_copy(dst, src, T):
    parts = np.array_split(np.arange(n), T)
    def w(p): dst[p[0]:p[-1]+1] = src[p[0]:p[-1]+1]
    th = [threading.Thread(target=w, args=(p,)) for p in parts]
    [t.start() for t in th]; [t.join() for t in th]
for T in (1, 4, 8, 16):
    t = time.perf_counter(); par_copy(z, x, T); dt = time.perf_counter() - t
    print(f"host copy {T} threads: {x.nbytes/dt/1e9:.1f} GB/s")
import os; print("cpus", os.cpu_count())
