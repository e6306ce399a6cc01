"""One launch (or one build / batch) of every CUDA kernel in libwt_b200.so at a
realistic size, for one `ncu --set full` capture of all of them
(scripts/gpu_ncu_all.sh; summary: profiles/rNN_ncu_all_kernels.txt).

  C2 build (u8, sigma=256, block mode)   hist8_blocks, block_l1, l1_scan, wlevel<u8,u8,1>, wpair, dirq
  2^24 u8 builds                          wlevel tile mode, wcount0; dir + qlayout (WT_DIRQ=0)
  u8 LUT build (sigma=200, 2^28)          hist8, wcount0, wlevel<u8,u8,lut>, wlast<lut>
  C3u-like build (u16, 2^28)              hist16p, hist16_fold, wlevel<u16,u16>
  declared alphabet with a stray symbol   first_outside
  queries, 1e7 per kind, sorted + not     qsort_key, qsort_scan_*, qsort_scatter, access/rank/select, qunsort, widen (host batches: narrow wire)
  build_index over 2^30 bits + queries    bits_directory, bits_query
  the building-block ops (wt_ops.cu)      map, encode, split_count/scan/scatter, pack_bits
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_03372_b200 as W  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(3)
rng = np.random.default_rng(3)

# C2 build
n = 1 << 30
text = torch.randint(0, 256, (n,), generator=g, device=dev, dtype=torch.int32).to(torch.uint8)
t = W.construct(text)
del text
# tile mode (2^24 symbols: too few L1 blocks for block mode) and the split
# directory (dir_kernel) + query layout (qlayout_kernel) path (WT_DIRQ=0)
text = torch.randint(0, 256, (1 << 24,), generator=g, device=dev, dtype=torch.int32).to(torch.uint8)
t24 = W.construct(text)
del t24
os.environ["WT_DIRQ"] = "0"
t24 = W.construct(text)
del t24
os.environ.pop("WT_DIRQ")
del text
# u8 LUT levels + per-tile counting (not block mode: 2^28 symbols, sigma=200)
text = torch.randint(0, 200, (1 << 28,), generator=g, device=dev, dtype=torch.int32).to(torch.uint8)
t200 = W.construct(text)
del text, t200
# u16
text = torch.randint(0, 65536, (1 << 28,), generator=g, device=dev, dtype=torch.int32).to(torch.int16)
t16 = W.construct(text)
del t16
# declared alphabet with one symbol outside it -> first_outside
try:
    W.construct_with_alphabet(text, np.arange(1, 65536, dtype=np.uint16))
except W.SymbolError:
    pass
del text
torch.cuda.empty_cache()
# queries on the C2 tree: 1e7 per kind, sorted and unsorted
m = 10_000_000
pos = rng.integers(0, n, m)
syms = rng.integers(0, 256, m)
rpos = rng.integers(0, n + 1, m)
occ = np.diff(t.cum_hist)
ks = np.minimum(1 + (rng.random(m) * occ[syms]).astype(np.int64), occ[syms])
for sort in (True, False):
    W.access_batch(t, pos, chunk_size=m, sort=sort)
    W.rank_batch(t, syms, rpos, chunk_size=m, sort=sort)
    W.select_batch(t, syms, ks, chunk_size=m, sort=sort)
del t
torch.cuda.empty_cache()
# stand-alone bit vector: build_index + rank / select
ba = W.build_bit_array([1 << 30])
ba.words[:] = rng.integers(0, 1 << 63, len(ba.words), dtype=np.int64).view(np.uint64)
idx = W.build_index(ba, 0)
idx.rank1_bulk(rng.integers(0, 1 << 30, 1 << 22))
idx.select1_bulk(rng.integers(1, idx.total_ones + 1, 1 << 22))
del idx, ba
# the reference's building blocks as device ops
txt = rng.integers(0, 256, 1 << 28).astype(np.uint8)
ids, amap = W.minimal_alphabet(txt)
amap.map_text(txt)
enc, hist = W.encode_and_histogram(ids, W.create_codes(256))
W.stable_sort_by_prefix(enc[: 1 << 24], 2, 8)
ba = W.build_bit_array([1 << 28])
W.fill_level(ba, 0, enc, 1 << 28, 8)
torch.cuda.synchronize()
print("every kernel launched")
