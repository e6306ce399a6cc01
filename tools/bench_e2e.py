"""e2e host-buffer batch timing by chunk size (iteration tool, not the bench):
    python tools/bench_e2e.py [--n-log 30] [--m 33333334] [--chunks 20,21,22]"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-log", type=int, default=30)
    ap.add_argument("--m", type=int, default=33_333_334)
    ap.add_argument("--chunks", default="20,21,22,23")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2505_03372_b200 as W
    n = 1 << a.n_log
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    text = torch.randint(0, 256, (n,), generator=g, device="cuda", dtype=torch.int32).to(torch.uint8)
    tree = W.construct(text)
    rng = np.random.default_rng(1)
    pin = lambda x: torch.from_numpy(x).pin_memory().numpy()
    c = pin(rng.integers(0, 256, a.m))
    p = pin(rng.integers(0, n + 1, a.m))
    occ = np.array(tree.cum_hist)[1:] - np.array(tree.cum_hist)[:-1]
    k = pin(1 + (rng.random(a.m) * occ[c]).astype(np.int64))
    pos = pin(rng.integers(0, n, a.m))
    for lg in [int(x) for x in a.chunks.split(",")]:
        ch = 1 << lg
        for kind, fn in (("access", lambda: W.access_batch(tree, pos, chunk_size=ch, sort=True)),
                         ("rank", lambda: W.rank_batch(tree, c, p, chunk_size=ch, sort=True)),
                         ("select", lambda: W.select_batch(tree, c, k, chunk_size=ch, sort=True))):
            fn()
            ts = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                r = fn()
                ts.append(time.perf_counter() - t0)
                del r
            t = min(ts)
            print(f"chunk 2^{lg} {kind:6s} {t*1e3:7.2f} ms  {a.m/t/1e9:.2f} G q/s", flush=True)


if __name__ == "__main__":
    main()
