"""Per-kind end-to-end time through the public API (pinned host arrays)."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03372_b200 as W

n = 1 << 30
text = torch.randint(0, 256, (n,), dtype=torch.int32, device="cuda").to(torch.uint8)
t = W.construct(text)
m = 33_333_333
g = torch.Generator(device="cuda"); g.manual_seed(1)
pin = lambda x: x.cpu().pin_memory().numpy()
pos = pin(torch.randint(0, n, (m,), device="cuda", generator=g))
syms = pin(torch.randint(0, 256, (m,), device="cuda", generator=g))
rpos = pin(torch.randint(0, n + 1, (m,), device="cuda", generator=g))
occ = np.diff(t.cum_hist)
ks = np.ascontiguousarray(np.minimum(1 + (np.random.default_rng(0).random(m) * occ[syms]).astype(np.int64), occ[syms]))
ks = torch.from_numpy(ks).pin_memory().numpy()
chunk = 1 << 21
for name, fn in (("access", lambda: W.access_batch(t, pos, chunk_size=chunk, sort=True)),
                 ("rank", lambda: W.rank_batch(t, syms, rpos, chunk_size=chunk, sort=True)),
                 ("select", lambda: W.select_batch(t, syms, ks, chunk_size=chunk, sort=True))):
    ts = []
    for _ in range(6):
        r = W.BatchRunner(t, chunk, sort=True)
        b = W.QueryBatch(name, pos if name == "access" else (rpos if name == "rank" else ks),
                         None if name == "access" else syms, chunk)
        t0 = time.perf_counter()
        out = r.run(b)
        ts.append(time.perf_counter() - t0)
    print(f"{name}: {np.median(ts)*1e3:.2f} ms med, min {min(ts)*1e3:.2f}; stage {r.stage_seconds*1e3:.2f} "
          f"process {r.process_seconds*1e3:.2f} unstage {r.unstage_seconds*1e3:.2f} peak {r.staging_peak_records}")
    ts = []
    for _ in range(6):
        t0 = time.perf_counter(); out = fn(); ts.append(time.perf_counter() - t0)
    print(f"  {name} via *_batch: {np.median(ts)*1e3:.2f} ms; out pinned? {out.base is not None}")
