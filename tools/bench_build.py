"""Quick device-side build timing for one config (iteration tool, not the bench).

    python tools/bench_build.py [--n-log 30] [--sigma 256] [--kind uniform|zipf|dna] [--u16]
"""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-log", type=int, default=30)
    ap.add_argument("--sigma", type=int, default=256)
    ap.add_argument("--kind", default="uniform")
    ap.add_argument("--declared", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_2505_03372_b200 as W
    from paper_2505_03372_b200 import _lib
    n = 1 << args.n_log
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    if args.kind == "uniform":
        dt = torch.uint8 if args.sigma <= 256 else torch.uint16
        hi = args.sigma
        text = torch.randint(0, hi, (n,), generator=g, device="cuda", dtype=torch.int32).to(dt)
    elif args.kind == "dna":
        lut = torch.tensor(list(b"ACGT"), dtype=torch.uint8, device="cuda")
        text = lut[torch.randint(0, 4, (n,), generator=g, device="cuda")]
    else:  # zipf 1.2 via numpy in chunks
        rng = np.random.default_rng(0)
        parts = [(np.minimum(rng.zipf(1.2, 1 << 26), args.sigma) - 1).astype(np.uint16)
                 for _ in range(max(1, n >> 26))]
        text = torch.from_numpy(np.concatenate(parts)[:n]).cuda()
    alpha = np.arange(args.sigma, dtype=np.uint16 if args.sigma > 256 else np.uint8)
    prof = (C.c_float * 32)()
    for r in range(args.reps + 2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tree = (W.construct_with_alphabet(text, alpha) if args.declared else W.construct(text))
        wall = (time.perf_counter() - t0) * 1e3
        _lib.lib.wt_tree_build_profile(tree.handle, prof, 32)
        lv = [prof[i] for i in range(1 + tree.num_levels)]
        print(f"rep {r}: device {tree.build_ms:8.3f} ms  wall {wall:8.2f} ms  pre {lv[0]:.3f}  "
              f"levels {' '.join(f'{x:.3f}' for x in lv[1:])}  sigma={tree.sigma} "
              f"-> {n / tree.build_ms / 1e6:.1f} Gsym/s", flush=True)
        del tree


if __name__ == "__main__":
    main()
