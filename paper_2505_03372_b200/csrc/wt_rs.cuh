// wt_rs.cuh -- device rank / select over one level's directory.
//
// rank1: Alg. 1 (rankselect.py:151-169): L1[p>>16] + L2[p>>l2_shift] + popcount
//        of the words between the L2 block start and p, masked last word;
//        p == n_bits -> total_ones.
// select: Alg. 2 (rankselect.py:229-367): sample window -> binary search over
//        L1 -> binary search over L2 -> word scan -> in-word select (popcount
//        halving, select_in_word32 in wt_common.cuh).
#pragma once
#include "wt_common.cuh"

namespace wt {

__device__ __forceinline__ u64 rank1_dev(const LevelDev& L, u64 p, u32 l2_shift) {
  if (p >= L.n_bits) return L.total_ones;
  u64 r = __ldg(L.l1 + (p >> 16)) + (u64)__ldg(L.l2 + (p >> l2_shift));
  const u64 wb = (p >> l2_shift) << (l2_shift - 6);
  const u64 we = p >> 6;
  for (u64 w = wb; w < we; ++w) r += __popcll(__ldg(L.words + w));
  const u32 rem = (u32)(p & 63);
  if (rem) r += __popcll(__ldg(L.words + we) & ((1ull << rem) - 1));
  return r;
}

// rank1 when the word holding p is already loaded (p < n_bits)
__device__ __forceinline__ u64 rank1_with_word(const LevelDev& L, u64 p, u32 l2_shift, u64 wp) {
  u64 r = __ldg(L.l1 + (p >> 16)) + (u64)__ldg(L.l2 + (p >> l2_shift));
  const u64 wb = (p >> l2_shift) << (l2_shift - 6);
  const u64 we = p >> 6;
  for (u64 w = wb; w < we; ++w) r += __popcll(__ldg(L.words + w));
  const u32 rem = (u32)(p & 63);
  if (rem) r += __popcll(wp & ((1ull << rem) - 1));
  return r;
}

template <bool kOnes>
__device__ __forceinline__ u64 select_dev(const LevelDev& L, u64 k, u32 l2_shift, u64 rate,
                                          int rate_log) {
  const u64* smp = kOnes ? L.ones : L.zeros;
  const u64 ns = kOnes ? L.n_ones : L.n_zeros;
  const u64 si = rate_log >= 0 ? (k >> rate_log) : k / rate;
  u64 lo_pos = 0, hi_pos = L.n_bits - 1;
  if (ns) {
    if (si >= 1) lo_pos = __ldg(smp + (si - 1 < ns ? si - 1 : ns - 1));
    if (si < ns) hi_pos = __ldg(smp + si);
  }
  u64 lo = lo_pos >> 16;
  u64 hi = hi_pos >> 16;
  if (hi > L.n_l1 - 1) hi = L.n_l1 - 1;
  while (lo < hi) {
    const u64 mid = (lo + hi + 1) >> 1;
    const u64 c = __ldg(L.l1 + mid);
    const u64 v = kOnes ? c : (mid << 16) - c;
    if (v < k) lo = mid; else hi = mid - 1;
  }
  {
    const u64 c = __ldg(L.l1 + lo);
    k -= kOnes ? c : (lo << 16) - c;
  }
  const u64 per = 65536ull >> l2_shift;
  const u64 base = lo * per;
  u64 jl = base;
  u64 jh = base + per < L.n_l2 ? base + per - 1 : L.n_l2 - 1;
  while (jl < jh) {
    const u64 mid = (jl + jh + 1) >> 1;
    const u64 c = __ldg(L.l2 + mid);
    const u64 v = kOnes ? c : ((mid - base) << l2_shift) - c;
    if (v < k) jl = mid; else jh = mid - 1;
  }
  {
    const u64 c = __ldg(L.l2 + jl);
    k -= kOnes ? c : ((jl - base) << l2_shift) - c;
  }
  u64 w = jl << (l2_shift - 6);
  while (true) {
    u64 x = __ldg(L.words + w);
    if (!kOnes) x = ~x;
    const u32 pc = __popcll(x);
    if (pc >= k) return (w << 6) + select_in_word64(x, (u32)k);
    k -= pc;
    ++w;
  }
}

}  // namespace wt

namespace wt {

// ---------------------------------------------------------------------------
// rank / select on the query-side rank-line layout (wt_qlayout.cu)
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 qline_of(u64 p, u32& w) {
  const u64 q = p >> 6;  // word index in the level
  u64 i;
  if (kQW == 7)
    i = __umul64hi(q, 0x2492492492492493ull);     // q / 7 (exact for q < 2^61)
  else if (kQW == 3)
    i = __umul64hi(q, 0xAAAAAAAAAAAAAAABull) >> 1;  // q / 3
  else
    i = q / kQW;
  w = (u32)(q - kQW * i);
  return i;
}

struct QLine {
  u64 hdr;
  u64 wd[kQW];
};

// L2 fetch-size hint of the query loads (WT_QL2: A/B knob; on B200 the
// sorted C2 batches ran 0.3-0.6 % faster with L2::128B / L2::256B, the
// random ones 3 % slower than with L2::64B)
#ifndef WT_QL2
#define WT_QL2 "L2::64B"
#endif

// Random 64-byte line reads: hint the L2 to fetch 64 B (LTC64B) instead of
// promoting the miss to a larger DRAM request -- every rank step is one
// line, so anything beyond it is wasted HBM bandwidth.
__device__ __forceinline__ ulonglong2 ld_line16(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.global.nc." WT_QL2 ".v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ u64 ld_u64_64b(const u64* p) {
  u64 v;
  asm volatile("ld.global.nc." WT_QL2 ".u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ u32 ld_u32_64b(const u32* p) {
  u32 v;
  asm volatile("ld.global.nc." WT_QL2 ".u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// batch streams (arguments in, results out): L2 evict-first, so the walk's
// lines keep the L2
__device__ __forceinline__ u64 l2_evict_first_policy() {
  u64 p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ i64 ld_stream_i64(const i64* a, u64 pol) {
  i64 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
               : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream_i64(i64* a, i64 v, u64 pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(a), "l"(v), "l"(pol)
               : "memory");
}

// one 64-byte line as two 256-bit loads (LDG.256, sm_100): half the LSU
// instructions of 16-byte loads, which kept the query kernels lg-throttled
__device__ __forceinline__ void ld_line32(const ulonglong2* p, u64& a, u64& b, u64& c, u64& d) {
  asm volatile("ld.global.nc." WT_QL2 ".v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(p));
}
static_assert(kQW == 3 || kQW == 7, "line width: one 32-byte sector or 64 bytes");
// one 32-byte line: one LDG.256; the L2::64B hint (the neighbouring line
// comes along) measured +3 % on random batches, neutral on sorted ones
__device__ __forceinline__ void ld_sector(const ulonglong2* p, u64& a, u64& b, u64& c, u64& d) {
  asm volatile("ld.global.nc." WT_QL2 ".v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(p));
}
__device__ __forceinline__ QLine qload(const QLevelDev& Q, u64 i) {
  const ulonglong2* L = Q.lines + i * kQLineU2;
  QLine r;
  if constexpr (kQW == 3) {
    ld_sector(L, r.hdr, r.wd[0], r.wd[1], r.wd[2]);
  } else {
    ld_line32(L, r.hdr, r.wd[0], r.wd[1], r.wd[2]);
    ld_line32(L + 2, r.wd[kQW - 4], r.wd[kQW - 3], r.wd[kQW - 2], r.wd[kQW - 1]);
  }
  return r;
}

// ones in the line before word w, plus the word itself
__device__ __forceinline__ u64 qline_prefix(const QLine& L, u32 w, u64& word) {
  u64 r = L.hdr;
  word = L.wd[0];
#pragma unroll
  for (int x = 0; x < kQW; ++x) {
    if ((u32)x < w) r += __popcll(L.wd[x]);
    if ((u32)x == w) word = L.wd[x];
  }
  return r;
}

// rank1(p) for p in [0, n_bits] (the sentinel line makes p == n_bits work)
__device__ __forceinline__ u64 qrank1(const QLevelDev& Q, u64 p) {
  u32 w;
  const u64 i = qline_of(p, w);
  const QLine L = qload(Q, i);
  u64 word;
  const u64 r = qline_prefix(L, w, word);
  const u32 rem = (u32)(p & 63);
  return r + (rem ? __popcll(word & ((1ull << rem) - 1)) : 0);
}

// rank1(p) and the bit at p (p < n_bits): one line
__device__ __forceinline__ u64 qrank1_bit(const QLevelDev& Q, u64 p, u32& bit) {
  u32 w;
  const u64 i = qline_of(p, w);
  const QLine L = qload(Q, i);
  u64 word;
  const u64 r = qline_prefix(L, w, word);
  const u32 rem = (u32)(p & 63);
  bit = (u32)(word >> rem) & 1u;
  return r + (rem ? __popcll(word & ((1ull << rem) - 1)) : 0);
}

template <bool kOnes>
__device__ __forceinline__ u64 qselect(const QLevelDev& Q, u64 k) {
  const u32* sel = kOnes ? Q.sel1 : Q.sel0;
  const u64 ns = kOnes ? Q.n_sel1 : Q.n_sel0;
  const u64 j = (k - 1) >> kQSelLog;
  u64 lo = ld_u32_64b(sel + j);
  u64 hi = j + 1 < ns ? (u64)ld_u32_64b(sel + j + 1) : Q.n_lines - 1;
  // the answer is the last line in [lo, hi] whose count before it is below
  // k: narrow by header probes to two candidates (dense bits: the samples are
  // already at most one line apart), then load both lines at once -- one
  // dependent step less than probing the second line's header first
  while (lo + 1 < hi) {
    const u64 mid = (lo + hi) >> 1;
    const u64 h = ld_u64_64b(reinterpret_cast<const u64*>(Q.lines + mid * kQLineU2));
    const u64 v = kOnes ? h : mid * kQBits - h;
    if (v < k) lo = mid; else hi = mid - 1;
  }
  QLine L = qload(Q, lo);
  if (hi > lo) {
    const QLine B = qload(Q, hi);
    const u64 v = kOnes ? B.hdr : hi * kQBits - B.hdr;
    if (v < k) {
      L = B;
      lo = hi;
    }
  }
  k -= kOnes ? L.hdr : lo * kQBits - L.hdr;
  // find the word first (predicated selects), then ONE in-word select: inside
  // the loop it would run once per distinct word index in the warp
  u32 wi = kQW - 1, kk = (u32)k;
  u64 ws = kOnes ? L.wd[kQW - 1] : ~L.wd[kQW - 1];
  bool done = false;
#pragma unroll
  for (int x = 0; x < kQW - 1; ++x) {
    const u64 word = kOnes ? L.wd[x] : ~L.wd[x];
    const u32 pc = __popcll(word);
    const bool here = !done && pc >= kk;
    wi = here ? (u32)x : wi;
    ws = here ? word : ws;
    kk -= (!done && !here) ? pc : 0u;
    done = done || here;
  }
  return lo * kQBits + 64 * wi + select_in_word64(ws, kk);
}

}  // namespace wt
