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

// ---------------------------------------------------------------------------
// dirq_kernel: the reference directory (L2 entries, select samples every
// `rate`-th one / zero, rankselect.py:495-532) and the query layout (lines +
// line samples) of one level in ONE streaming pass over its bits.  A CTA of
// 1024 threads owns 1024 consecutive lines = 3072 words = three whole L1
// blocks, so it starts on both a line and an L1 boundary: thread t holds
// line t (three words), a CTA scan of the line popcounts on top of l1[3 g]
// gives every line header; the L2 entry of word w = (ones before w) -
// l1[w >> 10].  Reference samples (~two of each kind per warp at rate 4096):
// a warp-uniform loop over the ordinals in the warp's range, the owning lane
// selects in its line.
// ---------------------------------------------------------------------------
constexpr int DQ_NT = 1024;  // threads = lines per CTA (3 L1 blocks: kQW = 3)
static_assert(kQW == 3, "dirq_kernel aligns three L1 blocks with 1024 lines of 3 words");

__device__ __forceinline__ u64 dq_next_multiple(u64 o, u64 rate, int rate_log) {
  if (rate_log >= 0) return ((o >> rate_log) + 1) << rate_log;
  return (o / rate + 1) * rate;
}

__global__ void __launch_bounds__(DQ_NT) dirq_kernel(const __grid_constant__ DirQParams Q) {
  const DirParams& P = Q.d;
  __shared__ u32 wsum[32];
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 nw = (P.m + 63) >> 6;
  const u64 n_l1 = (P.m + kL1Bits - 1) / kL1Bits;
  const u64 ncta = (Q.n_lines + DQ_NT - 1) / DQ_NT;
  const u32 l2m = (u32)((1ull << P.l2_log) >> 6) - 1u;  // L2 block = l2m + 1 words
  const u64 total = *Q.total;
  // the next group's words are loaded while this group is processed
  u64 wn[3];
  {
    const u64 w3 = ((u64)blockIdx.x * DQ_NT + tid) * 3;
#pragma unroll
    for (int x = 0; x < 3; ++x) wn[x] = w3 + x < nw ? __ldg(P.words + w3 + x) : 0ull;
  }
  for (u64 g = blockIdx.x; g < ncta; g += gridDim.x) {
    const u64 i = g * DQ_NT + tid;  // this thread's line
    const u64 w3 = i * 3;
    u64 w[3];
#pragma unroll
    for (int x = 0; x < 3; ++x) w[x] = wn[x];
    {
      const u64 w3n = (i + (u64)gridDim.x * DQ_NT) * 3;
#pragma unroll
      for (int x = 0; x < 3; ++x) wn[x] = w3n + x < nw ? __ldg(P.words + w3n + x) : 0ull;
    }
    const u64 cta1 = 3 * g < n_l1 ? __ldg(P.l1 + 3 * g) : total;  // ones before the CTA's first bit
    u32 pc[3];
#pragma unroll
    for (int x = 0; x < 3; ++x) pc[x] = __popcll(w[x]);
    const u32 c = pc[0] + pc[1] + pc[2];
    u32 inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= (u32)d) inc += y;
    }
    __syncthreads();  // wsum reuse
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      u32 v = wsum[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= (u32)d) v += y;
      }
      wsum[lane] = v;  // inclusive per warp
    }
    __syncthreads();
    const u32 wpre = warp ? wsum[warp - 1] : 0u;
    const u32 exl = inc - c;             // ones of the warp before this line
    const u64 hdr = cta1 + wpre + exl;   // ones of the level before line i
    const u64 b0 = i * kQBits;
    if (i < Q.n_lines) {
      ulonglong2* out = Q.lines + i * kQLineU2;
      out[0] = make_ulonglong2(hdr, w[0]);
      out[1] = make_ulonglong2(w[1], w[2]);
      // line samples: line of every 2^kQSelLog-th one / zero
      for (u64 j = (hdr + (1u << kQSelLog) - 1) >> kQSelLog; (j << kQSelLog) + 1 <= hdr + c; ++j)
        if (j < Q.cap1) Q.sel1[j] = (u32)i;
      if (b0 < P.m) {
        const u64 valid = min(P.m - b0, (u64)kQBits);
        const u64 zlo = b0 - hdr, zhi = zlo + (valid - c);
        for (u64 j = (zlo + (1u << kQSelLog) - 1) >> kQSelLog; (j << kQSelLog) + 1 <= zhi; ++j)
          if (j < Q.cap0) Q.sel0[j] = (u32)i;
      }
      // L2 entries of the line's words
      u64 pre = hdr;
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        const u64 wx = w3 + x;
        if (wx < nw && ((u32)wx & l2m) == 0)
          P.l2[(wx << 6) >> P.l2_log] = (u16)(pre - __ldg(P.l1 + (wx >> 10)));
        pre += pc[x];
      }
    }
    // reference samples: ordinals of the warp's range, owner by range
    const u32 vl = b0 < P.m ? (u32)min(P.m - b0, (u64)kQBits) : 0u;  // the line's valid bits
    const u64 zb = (b0 < P.m ? b0 : P.m) - hdr;                     // zeros before the line
    const u32 zl = vl - c;
#pragma unroll
    for (int kind = 0; kind < 2; ++kind) {
      const bool ones = kind == 0;
      const u64 bl = ones ? hdr : zb;
      const u32 cl = ones ? c : zl;
      const u64 bw = __shfl_sync(0xffffffffu, bl, 0);
      const u64 ew = __shfl_sync(0xffffffffu, bl + cl, 31);
      for (u64 qo = dq_next_multiple(bw, P.rate, P.rate_log); qo <= ew; qo += P.rate) {
        if (bl < qo && qo <= bl + cl) {
          u32 k = (u32)(qo - bl);
          u32 cw[3];
#pragma unroll
          for (int x = 0; x < 3; ++x) {
            const u32 vbx = vl > 64u * x ? min(64u, vl - 64u * x) : 0u;
            cw[x] = ones ? pc[x] : vbx - pc[x];
          }
          const u32 j = k > cw[0] ? (k > cw[0] + cw[1] ? 2u : 1u) : 0u;
          k -= j == 0 ? 0u : j == 1 ? cw[0] : cw[0] + cw[1];
          const u64 wv = j == 0 ? w[0] : j == 1 ? w[1] : w[2];
          const u32 vb = vl > 64u * j ? min(64u, vl - 64u * j) : 0u;
          const u64 wm = (ones ? wv : ~wv) & (vb >= 64 ? ~0ull : (1ull << vb) - 1ull);
          const u64 pos = ((w3 + j) << 6) + select_in_word64(wm, k);
          const u64 si = (P.rate_log >= 0 ? (qo >> P.rate_log) : qo / P.rate) - 1;
          u64* o = ones ? P.ones : P.zeros;
          if (si < (ones ? P.ones_cap : P.zeros_cap)) o[si] = pos;
        }
      }
    }
  }
}

cudaError_t launch_dirq(const DirQParams& p, int sms, cudaStream_t st) {
  if (!p.n_lines) return cudaSuccess;
  const u64 ncta = (p.n_lines + DQ_NT - 1) / DQ_NT;
  u64 blocks = ncta;
  if (blocks > (u64)sms * 2) blocks = (u64)sms * 2;
  dirq_kernel<<<(unsigned)blocks, DQ_NT, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_qlayout(const LevelDev& L, const u64* total, u32 l2_shift, ulonglong2* lines,
                           u64 n_lines, u32* sel1, u64 cap1, u32* sel0, u64 cap0, cudaStream_t st) {
  if (!n_lines) return cudaSuccess;
  const u64 blocks = (n_lines + QL_NT - 1) / QL_NT;
  qlayout_kernel<<<(unsigned)blocks, QL_NT, 0, st>>>(L, total, l2_shift, lines, n_lines, sel1, cap1,
                                                     sel0, cap0);
  return cudaGetLastError();
}

}  // namespace wt
