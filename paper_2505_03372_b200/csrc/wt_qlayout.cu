// wt_qlayout.cu -- query-side "rank line" layout of each level.
//
// Line i of a level = [ones before bit kQBits i | the next kQBits bits].
// One thread per line: the kQW data words are a straight copy (word
// aligned), the header comes from the level's reference directory
// (rank1 = L1 + L2 + popcount, rankselect.py:151-169) and the thread emits
// the select samples (line index of every 2^kQSelLog-th one / zero) that
// fall in its line.  The last line is a sentinel whose header is the level
// total.
#include "wt_common.cuh"
#include "wt_kernels.h"
#include "wt_rs.cuh"

namespace wt {

constexpr int QL_NT = 256;

__global__ void __launch_bounds__(QL_NT, 8) qlayout_kernel(LevelDev L, const u64* total, u32 l2_shift,
                                                       ulonglong2* __restrict__ lines, u64 n_lines,
                                                       u32* __restrict__ sel1, u64 cap1,
                                                       u32* __restrict__ sel0, u64 cap0) {
  const u64 i = (u64)blockIdx.x * QL_NT + threadIdx.x;
  const u32 lane = threadIdx.x & 31;
  L.total_ones = *total;
  const u64 b0 = i * kQBits;
  const u64 nw = (L.n_bits + 63) >> 6;
  u64 w[kQW];
  u32 pc = 0;
#pragma unroll
  for (int x = 0; x < kQW; ++x) {
    const u64 wi = (b0 >> 6) + x;
    w[x] = i < n_lines && wi < nw ? __ldg(L.words + wi) : 0ull;  // padding bits are zero
    pc += __popcll(w[x]);
  }
  // headers: one directory lookup per warp (its first line), then a warp
  // scan of the lines' popcounts -- the 32 lines are consecutive
  u64 first = 0;
  if (lane == 0) {
    const u64 fb = b0;
    first = i >= n_lines ? 0ull : fb >= L.n_bits ? L.total_ones : rank1_dev(L, fb, l2_shift);
  }
  first = __shfl_sync(0xffffffffu, first, 0);
  u32 inc = pc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= (u32)d) inc += y;
  }
  if (i >= n_lines) return;
  const u64 hdr = first + (inc - pc);
  ulonglong2* out = lines + i * kQLineU2;
  out[0] = make_ulonglong2(hdr, w[0]);
#pragma unroll
  for (int x = 1; x < kQLineU2; ++x) out[x] = make_ulonglong2(w[2 * x - 1], w[2 * x]);
  // samples: ordinals k = j * 2^kQSelLog + 1 in (hdr, hdr + pc] for ones, likewise zeros
  if (pc) {
    const u64 lo = hdr, hi = hdr + pc;
    for (u64 j = (lo + (1u << kQSelLog) - 1) >> kQSelLog; (j << kQSelLog) + 1 <= hi; ++j)
      if (j < cap1) sel1[j] = (u32)i;
  }
  if (b0 < L.n_bits) {
    const u64 valid = L.n_bits - b0 < (u64)kQBits ? L.n_bits - b0 : (u64)kQBits;
    const u64 zlo = b0 - hdr, zhi = zlo + (valid - pc);
    for (u64 j = (zlo + (1u << kQSelLog) - 1) >> kQSelLog; (j << kQSelLog) + 1 <= zhi; ++j)
      if (j < cap0) sel0[j] = (u32)i;
  }
}

u64 qlayout_lines(u64 n_bits) { return n_bits / kQBits + 1; }

cudaError_t launch_qlayout(const LevelDev& L, const u64* total, u32 l2_shift, ulonglong2* lines,
                           u64 n_lines, u32* sel1, u64 cap1, u32* sel0, u64 cap0, cudaStream_t st) {
  if (!n_lines) return cudaSuccess;
  const u64 blocks = (n_lines + QL_NT - 1) / QL_NT;
  qlayout_kernel<<<(unsigned)blocks, QL_NT, 0, st>>>(L, total, l2_shift, lines, n_lines, sel1, cap1,
                                                     sel0, cap0);
  return cudaGetLastError();
}

}  // namespace wt
