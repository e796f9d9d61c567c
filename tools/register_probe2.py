"""Host-side costs of staging alternatives on the GPU box (8.2 GB arrays):
cudaHostRegister in place (fresh / pre-touched), multi-threaded read scan and
memcpy throughput.  Usage: python tools/register_probe2.py"""
import ctypes
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
shape = (n, 1024)
nb = 8 * n * 1024
rt = ctypes.CDLL("libcudart.so.12") if False else None
torch.cuda.init()
cr = torch.cuda.cudart()


def tm(label, fn):
    t0 = time.perf_counter()
    r = fn()
    dt = time.perf_counter() - t0
    print(f"{label:55s} {dt * 1e3:9.1f} ms  {nb / dt / 1e9:7.1f} GB/s", flush=True)
    return r


x = np.random.default_rng(0).normal(size=shape)
for th in (1, 4, 8, 16):
    def scan(a=x, th=th):
        parts = np.array_split(a.reshape(-1), th * 4)
        with ThreadPoolExecutor(th) as ex:
            return all(ex.map(lambda p: bool(np.isfinite(p).all()), parts))
    tm(f"isfinite scan, {th} threads", scan)
y = np.empty_like(x)
y.fill(0)
for th in (1, 4, 8, 16):
    def cp(th=th):
        px, py = np.array_split(x.reshape(-1), th * 4), np.array_split(y.reshape(-1), th * 4)
        with ThreadPoolExecutor(th) as ex:
            list(ex.map(lambda ab: np.copyto(ab[1], ab[0]), zip(px, py)))
    tm(f"memcpy pre-touched, {th} threads", cp)
for th in (1, 8, 16):
    def fresh(th=th):
        z = np.empty_like(x)
        pz = np.array_split(z.reshape(-1), th * 4)
        with ThreadPoolExecutor(th) as ex:
            list(ex.map(lambda p: p.fill(0.0), pz))
        return z
    tm(f"first touch fresh array, {th} threads", fresh)


def reg(a, flags=0):
    r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, flags)
    assert int(r) == 0, r


def unreg(a):
    cr.cudaHostUnregister(a.ctypes.data)


tm("cudaHostRegister pre-touched input (x)", lambda: reg(x))
tm("cudaHostUnregister x", lambda: unreg(x))
tm("cudaHostRegister pre-touched input (x) again", lambda: reg(x))
tm("cudaHostUnregister x", lambda: unreg(x))
z = np.empty_like(x)
tm("cudaHostRegister FRESH array (untouched)", lambda: reg(z))
tm("cudaHostUnregister fresh", lambda: unreg(z))
d = torch.empty(shape, dtype=torch.float64, device="cuda")
reg(x)
tx = torch.from_numpy(x)
torch.cuda.synchronize()
tm("H2D from registered x", lambda: (d.copy_(tx, non_blocking=True), torch.cuda.synchronize()))
unreg(x)
tm("H2D from pageable x", lambda: (d.copy_(tx), torch.cuda.synchronize()))
