"""End-to-end (pinned host arrays through access_batch / rank_batch /
select_batch, sorted) queries/s against the pipeline chunk size.
    python tools/e2e_chunks.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2505_03372_b200 as W
    n, m = 1 << 30, 33_333_334
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    text = torch.randint(0, 256, (n,), generator=g, device="cuda", dtype=torch.int32).to(torch.uint8)
    tree = W.construct(text)
    occ = torch.from_numpy(np.diff(tree.cum_hist)).cuda()
    syms = torch.from_numpy(tree.alphabet.sorted_symbols.astype(np.int64)).cuda()
    pin = lambda t: t.cpu().pin_memory().numpy()
    acc = pin(torch.randint(0, n, (m,), generator=g, device="cuda", dtype=torch.int64))
    rsym = pin(syms[torch.randint(0, tree.sigma, (m,), generator=g, device="cuda")])
    rpos = pin(torch.randint(0, n + 1, (m,), generator=g, device="cuda", dtype=torch.int64))
    sid = torch.randint(0, tree.sigma, (m,), generator=g, device="cuda")
    ssym = pin(syms[sid])
    ks = pin(torch.minimum(1 + (torch.rand(m, generator=g, device="cuda", dtype=torch.float64)
                                * occ[sid]).long(), occ[sid]))
    logs = [int(x) for x in os.environ.get("E2E_LOGS", "16,18,20,21,22").split(",")]
    for log in logs:
        c = 1 << log
        for srt in (False, True):
            ts = []
            for r in range(4):
                t0 = time.perf_counter()
                W.access_batch(tree, acc, chunk_size=c, sort=srt)
                W.rank_batch(tree, rsym, rpos, chunk_size=c, sort=srt)
                W.select_batch(tree, ssym, ks, chunk_size=c, sort=srt)
                if r >= 1:
                    ts.append(time.perf_counter() - t0)
            t = float(np.median(ts))
            print(f"chunk 2^{log} sort={srt}: {3 * m / t / 1e9:.3f} G q/s  ({t * 1e3:.1f} ms per 3 batches)",
                  flush=True)


if __name__ == "__main__":
    main()
