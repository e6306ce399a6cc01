"""Quick device-resident query timing (iteration tool, not the bench).
    python tools/bench_query.py [--n-log 30] [--sigma 256] [--m 33333334]"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-log", type=int, default=30)
    ap.add_argument("--sigma", type=int, default=256)
    ap.add_argument("--m", type=int, default=33_333_334)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--sort", action="store_true", help="WT_F_SORT: device sort by symbol")
    args = ap.parse_args()
    import torch
    import paper_2505_03372_b200 as W
    from paper_2505_03372_b200 import _lib
    n = 1 << args.n_log
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    dt = torch.uint8 if args.sigma <= 256 else torch.uint16
    text = torch.randint(0, args.sigma, (n,), generator=g, device="cuda", dtype=torch.int32).to(dt)
    tree = W.construct(text)
    print(f"built n=2^{args.n_log} sigma={tree.sigma} in {tree.build_ms:.2f} ms; "
          f"device bytes {tree.device_bytes/1e9:.2f} GB", flush=True)
    m = args.m
    occ = torch.from_numpy(np.diff(tree.cum_hist)).cuda()
    syms = torch.from_numpy(tree.alphabet.sorted_symbols.astype(np.int64)).cuda()
    pos = torch.randint(0, n, (m,), generator=g, device="cuda", dtype=torch.int64)
    rsym = syms[torch.randint(0, tree.sigma, (m,), generator=g, device="cuda")]
    rpos = torch.randint(0, n + 1, (m,), generator=g, device="cuda", dtype=torch.int64)
    sid = torch.randint(0, tree.sigma, (m,), generator=g, device="cuda")
    sid = sid[occ[sid] > 0]
    ssym = syms[sid]
    ks = torch.minimum(1 + (torch.rand(len(sid), generator=g, device="cuda", dtype=torch.float64)
                            * occ[sid]).long(), occ[sid])
    out_a = torch.empty(m, dtype=dt, device="cuda")
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    flags = _lib.F_DEVICE_PTRS | _lib.F_SYMBOLS | (_lib.F_SORT if args.sort else 0)
    bad = C.c_int64(-1)
    P = lambda t: C.c_void_p(t.data_ptr())
    for name, kind, ids, a, o in (("access", 0, None, pos, out_a), ("rank", 1, rsym, rpos, out),
                                  ("select", 2, ssym, ks, out)):
        ts = []
        for r in range(args.reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.check(_lib.lib.wt_tree_query(tree.handle, kind, P(ids) if ids is not None else None,
                                              P(a), P(o), a.numel(), 0, flags,
                                              C.c_void_p(st.cuda_stream), C.byref(bad), None), name)
            e1.record(st)
            torch.cuda.synchronize()
            assert bad.value == -1
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        print(f"{name:7s} {a.numel()/t/1e6:8.3f} Gq/s  ({t:.3f} ms for {a.numel()})", flush=True)
    k = 1 << 20
    host = text.cpu().numpy()
    assert np.array_equal(out_a[:k].cpu().numpy(), host[pos[:k].cpu().numpy()])
    print("access spot-check ok")


if __name__ == "__main__":
    main()
