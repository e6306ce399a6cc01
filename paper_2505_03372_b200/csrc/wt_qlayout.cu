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
// line samples) of one level in ONE streaming pass over its bits.  A warp
// owns 1024 consecutive lines = 3072 words = three whole L1 blocks, so it
// starts on both a line and an L1 boundary: its running ones count starts at
// l1[3 g] and every line header is that count plus a warp scan.  Lane i of a
// step owns line i of the step (three words); four steps' loads go out
// first.  L2 entry of word w = (ones before w) - l1[w >> 10].
// ---------------------------------------------------------------------------
constexpr int DQ_NT = 256;
constexpr u32 DQ_LINES = 1024;  // lines per warp (3 L1 blocks: kQW = 3)
static_assert(kQW == 3, "dirq_kernel aligns three L1 blocks with 1024 lines of 3 words");

__device__ __forceinline__ u64 dq_next_multiple(u64 o, u64 rate, int rate_log) {
  if (rate_log >= 0) return ((o >> rate_log) + 1) << rate_log;
  return (o / rate + 1) * rate;
}

__global__ void __launch_bounds__(DQ_NT) dirq_kernel(const __grid_constant__ DirQParams Q) {
  const DirParams& P = Q.d;
  const u32 lane = threadIdx.x & 31;
  const u64 nw = (P.m + 63) >> 6;
  const u64 n_l1 = (P.m + kL1Bits - 1) / kL1Bits;
  const u64 nwarps = (Q.n_lines + DQ_LINES - 1) / DQ_LINES;
  const u32 l2m = (u32)((1ull << P.l2_log) >> 6) - 1u;  // L2 block = l2m + 1 words
  const u64 total = *Q.total;
  for (u64 g = (u64)blockIdx.x * (DQ_NT / 32) + (threadIdx.x >> 5); g < nwarps;
       g += (u64)gridDim.x * (DQ_NT / 32)) {
    const u64 line0 = g * DQ_LINES;
    u64 run = 3 * g < n_l1 ? __ldg(P.l1 + 3 * g) : total;  // ones before the warp's first bit
    constexpr int GRP = 4;
    for (u32 sg = 0; sg < DQ_LINES / 32; sg += GRP) {
    if (line0 + (u64)sg * 32 >= Q.n_lines) break;
    u64 wv[GRP][3];
#pragma unroll
    for (int g2 = 0; g2 < GRP; ++g2) {
      const u64 wi = (line0 + (u64)(sg + g2) * 32 + lane) * 3;
#pragma unroll
      for (int x = 0; x < 3; ++x) wv[g2][x] = wi + x < nw ? __ldg(P.words + wi + x) : 0ull;
    }
#pragma unroll
    for (int g2 = 0; g2 < GRP; ++g2) {
      const u64 i0 = line0 + (u64)(sg + g2) * 32;  // the step's first line (warp-uniform)
      if (i0 >= Q.n_lines) break;
      const u64 i = i0 + lane;
      const u64 w3 = i * 3;
      u64 w[3];
#pragma unroll
      for (int x = 0; x < 3; ++x) w[x] = wv[g2][x];
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
      const u32 tot = __shfl_sync(0xffffffffu, inc, 31);
      const u32 exl = inc - c;
      const u64 hdr = run + exl;  // ones before line i
      const u64 srun = run;       // ones before the step (warp-uniform)
      run += tot;
      const u64 b0 = i * kQBits;
      const bool live = i < Q.n_lines;
      // ---- query line + line samples (every 2^kQSelLog-th one / zero) -------
      if (live) {
        ulonglong2* out = Q.lines + i * kQLineU2;
        out[0] = make_ulonglong2(hdr, w[0]);
        out[1] = make_ulonglong2(w[1], w[2]);
        if (c) {
          for (u64 j = (hdr + (1u << kQSelLog) - 1) >> kQSelLog; (j << kQSelLog) + 1 <= hdr + c; ++j)
            if (j < Q.cap1) Q.sel1[j] = (u32)i;
        }
        if (b0 < P.m) {
          const u64 valid = min(P.m - b0, (u64)kQBits);
          const u64 zlo = b0 - hdr, zhi = zlo + (valid - c);
          for (u64 j = (zlo + (1u << kQSelLog) - 1) >> kQSelLog; (j << kQSelLog) + 1 <= zhi; ++j)
            if (j < Q.cap0) Q.sel0[j] = (u32)i;
        }
        // ---- L2 entries of the line's words --------------------------------
        u64 pre = hdr;
#pragma unroll
        for (int x = 0; x < 3; ++x) {
          const u64 wx = w3 + x;
          if (wx < nw && ((u32)wx & l2m) == 0)
            P.l2[(wx << 6) >> P.l2_log] = (u16)(pre - __ldg(P.l1 + (wx >> 10)));
          pre += pc[x];
        }
      }
      // ---- reference samples: ~one per kind per step, owner lane by range --
      const u64 sb0 = i0 * kQBits;  // the step's first bit
      if (sb0 < P.m) {
        const u64 vstep = min(P.m - sb0, (u64)(32 * kQBits));
        const u32 vl = b0 < P.m ? (u32)min(P.m - b0, (u64)kQBits) : 0u;  // the lane's valid bits
        const u32 zl = vl - c;
        const u32 zexl = (u32)(b0 - sb0) - exl;
#pragma unroll
        for (int kind = 0; kind < 2; ++kind) {
          const bool ones = kind == 0;
          const u64 base = ones ? srun : sb0 - srun;
          const u64 cnt = ones ? (u64)tot : vstep - tot;
          const u32 lo = ones ? exl : zexl, lc = ones ? c : zl;
          for (u64 qo = dq_next_multiple(base, P.rate, P.rate_log); qo <= base + cnt; qo += P.rate) {
            const u64 k = qo - base;  // 1-based in the step
            if (lo < k && k <= (u64)lo + lc) {
              u32 kk = (u32)(k - lo);
              u64 pos = 0;
#pragma unroll
              for (int x = 0; x < 3; ++x) {
                const u32 vb = vl > 64u * x ? min(64u, vl - 64u * x) : 0u;
                const u64 wm = (ones ? w[x] : ~w[x]) & (vb >= 64 ? ~0ull : (1ull << vb) - 1ull);
                const u32 pcx = __popcll(wm);
                if (kk > 0 && kk <= pcx) {
                  pos = ((w3 + x) << 6) + select_in_word64(wm, kk);
                  kk = 0;
                } else if (kk > 0) {
                  kk -= pcx;
                }
              }
              const u64 si = (P.rate_log >= 0 ? (qo >> P.rate_log) : qo / P.rate) - 1;
              u64* o = ones ? P.ones : P.zeros;
              if (si < (ones ? P.ones_cap : P.zeros_cap)) o[si] = pos;
            }
          }
        }
      }
    }
    }
  }
}

cudaError_t launch_dirq(const DirQParams& p, int sms, cudaStream_t st) {
  if (!p.n_lines) return cudaSuccess;
  const u64 nwarps = (p.n_lines + DQ_LINES - 1) / DQ_LINES;
  u64 blocks = (nwarps + (DQ_NT / 32) - 1) / (DQ_NT / 32);
  if (blocks > (u64)sms * 8) blocks = (u64)sms * 8;
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
