"""Diagnose the C3z device text vs the CPU golden recipe."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import large_cases as LC
n = 1 << 22
g = LC.zipf_torch(3, 65536, n, "cuda").cpu().numpy().view(np.uint16)
c = LC.zipf_np(3, 65536, 0, n)
print("prefix equal:", (g == c).all(), "mismatches:", int((g != c).sum()), g[:8], c[:8])
full = LC.zipf_torch(3, 65536, 1 << 30, "cuda")
hi = (full.view(torch.int16) < 0).sum().item()
print("full >= 32768 fraction:", hi / (1 << 30), hi)
import paper_2505_03372_b200 as W
for bm in ("0", "1"):
    os.environ["WT_BLOCK_MODE"] = bm
    t = W.construct_with_alphabet(full, np.arange(65536, dtype=np.uint16))
    print("block", bm, "total_ones", [int(r.total_ones) for r in t.rs][:4])
    del t
