"""A/B: host-pipeline query time with and without the pipeline stats events."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03372_b200 as W
from paper_2505_03372_b200 import _lib

n = 1 << 30
text = torch.randint(0, 256, (n,), dtype=torch.int32, device="cuda").to(torch.uint8)
t = W.construct(text)
m = 33_333_333
pos = torch.randint(0, n, (m,), device="cuda").cpu().pin_memory().numpy()
for chunk in (1 << 21, 1 << 23):
    for stats in (False, True, False, True):
        for sort in (True,):
            ts = []
            for _ in range(5):
                st = _lib.QueryStats() if stats else None
                t0 = time.perf_counter()
                out, bad = t.query(_lib.Q_ACCESS, None, pos, symbols=True, chunk=chunk, sort=sort, stats=st)
                ts.append(time.perf_counter() - t0)
            print(f"chunk {chunk} stats={stats} sort={sort}: {min(ts)*1e3:.2f} ms min, {np.median(ts)*1e3:.2f} med",
                  "" if st is None else f"h2d {st.h2d_ms:.2f} kern {st.kernel_ms:.2f} d2h {st.d2h_ms:.2f} tot {st.total_ms:.2f} peak {st.peak_records}")
