"""Where does the end-to-end query time go?  PCIe copy rates (torch pinned
buffers) next to one host-pointer wt_tree_query per kind with its kernel time."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03372_b200 as W
from paper_2505_03372_b200 import _lib

dev = torch.device("cuda", 0)
x = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
y = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
for name, f in (("h2d", lambda: y.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(y, non_blocking=True))):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    print(f"{name}: {3 * (1 << 30) / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
# both directions at once (two streams): the e2e step moves 1.33 GB in and
# 0.57 GB out concurrently
x2 = torch.empty(1 << 29, dtype=torch.uint8).pin_memory()
y2 = torch.empty(1 << 29, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1):
        y.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        x2.copy_(y2, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"h2d 1 GiB + d2h 0.5 GiB concurrently: {3 * 1.5 * (1 << 30) / dt / 1e9:.1f} GB/s combined")
del x, y, x2, y2
n = 1 << 30
text = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
tree = W.construct(torch.from_numpy(text).to(dev))
m = 33_333_334
r = np.random.default_rng(1)
pos = torch.from_numpy(r.integers(0, n, m)).pin_memory().numpy()
sym = torch.from_numpy(r.integers(0, 256, m)).pin_memory().numpy()
for chunk in (1 << 20, 1 << 22, 1 << 24):
    for kind, ids, args in ((_lib.Q_ACCESS, None, pos), (_lib.Q_RANK, sym, pos)):
        out = _lib.pinned_empty(m, np.uint8 if kind == 0 else np.int64)
        bad = C.c_int64(-1)
        ms = C.c_float(0)
        for rep in range(2):
            t0 = time.perf_counter()
            _lib.check(_lib.lib.wt_tree_query(tree.handle, kind, _lib.ptr(ids), _lib.ptr(args),
                                              _lib.ptr(out), m, chunk, _lib.F_SYMBOLS, None,
                                              C.byref(bad), C.byref(ms)))
            dt = time.perf_counter() - t0
        inb = m * (8 if ids is None else 16)
        print(f"chunk 2^{chunk.bit_length()-1} kind {kind}: wall {dt*1e3:.1f} ms kernels {ms.value:.1f} ms "
              f"-> {m/dt/1e9:.2f} Gq/s; h2d {inb/1e9:.2f} GB d2h {out.nbytes/1e9:.2f} GB")
t0 = time.perf_counter()
a = W.access_batch(tree, pos, chunk_size=1 << 22)
print(f"access_batch API: {(time.perf_counter()-t0)*1e3:.1f} ms")
