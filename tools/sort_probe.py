"""How much do the query kernels gain from a FULL (symbol, argument) order
over the device sort's bucket order?  Times, per kind: the WT_F_SORT
path; the plain path on inputs pre-sorted by (symbol, argument) with torch
(results come out in sorted order: no permuted writes); the plain path on
inputs pre-sorted by bucket only (each bucket's queries shuffled).
    python tools/sort_probe.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2505_03372_b200 as W
    from paper_2505_03372_b200 import _lib
    n, m = 1 << 30, 33_333_334
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    text = torch.randint(0, 256, (n,), generator=g, device="cuda", dtype=torch.int32).to(torch.uint8)
    tree = W.construct(text)
    occ = torch.from_numpy(np.diff(tree.cum_hist)).cuda()
    syms = torch.from_numpy(tree.alphabet.sorted_symbols.astype(np.int64)).cuda()
    rsid = torch.randint(0, tree.sigma, (m,), generator=g, device="cuda")
    rpos = torch.randint(0, n + 1, (m,), generator=g, device="cuda", dtype=torch.int64)
    sid = torch.randint(0, tree.sigma, (m,), generator=g, device="cuda")
    ks = torch.minimum(1 + (torch.rand(m, generator=g, device="cuda", dtype=torch.float64)
                            * occ[sid]).long(), occ[sid])
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    bad = C.c_int64(-1)
    P = lambda t: C.c_void_p(t.data_ptr())

    def run(kind, ids, a, flags, reps=5):
        ts = []
        for r in range(reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.check(_lib.lib.wt_tree_query(tree.handle, kind, P(ids), P(a), P(out), m, 0,
                                              flags, C.c_void_p(st.cuda_stream), C.byref(bad), None), "q")
            e1.record(st)
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    base = _lib.F_DEVICE_PTRS | _lib.F_SYMBOLS
    for name, kind, ids_id, a, span in (("rank", 1, rsid, rpos, n + 1), ("select", 2, sid, ks, int(occ.max()))):
        t_sort = run(kind, syms[ids_id], a, base | _lib.F_SORT)
        key = ids_id * (1 << 40) + (a if kind == 1 else a - 1)
        o = torch.argsort(key)
        t_full = run(kind, syms[ids_id[o]].contiguous(), a[o].contiguous(), base)
        res = []
        for sub in (256, 4096, 65536):
            shift = 0
            while ((span - 1) >> shift) >= sub:
                shift += 1
            bkey = ids_id * sub + ((a if kind == 1 else a - 1) >> shift)
            o2 = torch.argsort(bkey * (1 << 24) + torch.randint(0, 1 << 24, (m,), generator=g, device="cuda"))
            res.append(run(kind, syms[ids_id[o2]].contiguous(), a[o2].contiguous(), base))
        # argument-block major, symbol minor (2^20 buckets): consecutive buckets
        # are the same stretch of the text for every symbol
        sarg = a if kind == 1 else a - 1
        if kind == 2:  # ordinal -> approximate text position k * n / occ
            sarg = (sarg.double() * n / occ[ids_id].double()).long()
        shift = 0
        while ((n - 1) >> shift) >= 4096:
            shift += 1
        bkey = (sarg >> shift) * 256 + ids_id
        o3 = torch.argsort(bkey * (1 << 24) + torch.randint(0, 1 << 24, (m,), generator=g, device="cuda"))
        res.append(run(kind, syms[ids_id[o3]].contiguous(), a[o3].contiguous(), base))
        t_plain = run(kind, syms[ids_id], a, base)
        # the cost of putting sorted-order results back in query order
        perm = o.to(torch.int64)
        dst = torch.empty_like(out)
        ts = []
        for r in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            dst.index_copy_(0, perm, out)
            e1.record(st)
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        print(f"{name:7s} F_SORT {t_sort:.3f} ms | presorted full {t_full:.3f} | by 2^16/2^20/2^24 buckets "
              f"{res[0]:.3f} / {res[1]:.3f} / {res[2]:.3f} | pos-major 2^20 {res[3]:.3f} | unsorted {t_plain:.3f} | "
              f"unpermute (index_copy_) {np.median(ts):.3f}", flush=True)


if __name__ == "__main__":
    main()
