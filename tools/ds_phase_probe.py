"""Per-phase wall times of the device dataset codec (host orchestration vs
kernels); measurement helper, prints one JSON line."""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2601_03159_b200 import _abi, _native
from paper_2601_03159_b200.datafiles import _vp, format_dataset_to_device, _label_blob

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
torch.cuda.set_device(0)
_native.ensure_device(0)
x, data, headers, labels = bench.ds_text(n, 1024)
d_text = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
L = _native.lib()
st = _vp(torch.cuda.current_stream().cuda_stream)
res = {}


def tick(name, t0):
    torch.cuda.synchronize()
    res[name] = res.get(name, 0) + (time.perf_counter() - t0) * 1e3
    return time.perf_counter()


for it in range(4):
    if it == 1:
        res.clear()
    t = time.perf_counter()
    info = _abi.SaDatasetInfo()
    h = ctypes.c_void_p()
    _native.check(L.sa_dataset_open(_vp(d_text.data_ptr()), len(data), -1, 1, ctypes.byref(h), ctypes.byref(info), st))
    t = tick("open", t)
    v = torch.empty((info.n_series, info.length), dtype=torch.float64, device="cuda")
    _native.check(L.sa_dataset_values(h, _vp(v.data_ptr()), ctypes.byref(info)))
    t = tick("values", t)
    dh = torch.empty(max(info.header_bytes, 1), dtype=torch.uint8, device="cuda")
    dl = torch.empty(max(info.label_bytes, 1), dtype=torch.uint8, device="cuda")
    L.sa_dataset_headers(h, _vp(dh.data_ptr()))
    L.sa_dataset_labels(h, _vp(dl.data_ptr()))
    t = tick("gather", t)
    lab = tuple(dl[:info.label_bytes].cpu().numpy().tobytes().decode().split("\n")[:-1])
    t = tick("labels_host", t)
    L.sa_dataset_close(h)
    t = tick("close", t)
    blob, off = _label_blob(lab, len(lab))
    t = tick("label_blob_host", t)
    out = format_dataset_to_device(v, "ts", headers, lab)
    t = tick("format_total", t)
print(json.dumps({k: round(v / 3, 3) for k, v in res.items()}))
