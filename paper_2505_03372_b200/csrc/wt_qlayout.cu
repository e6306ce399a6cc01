// wt_qlayout.cu -- query-side "rank line" layout of each level.
//
// Line i of a level = [ones before bit kQBits i | the next kQBits bits].
// One thread per line: the kQW data words are a straight copy (word
// aligned), the header comes from the level's reference directory
// (rank1 = L1 + L2 + popcount, rankselect.py:151-169) and the thread emits
// the select samples (line index of every 2^kQSelLog-th one / zero) that
// fall in its line.  The last line is a sentinel whose header is the level
// total.
#include <atomic>
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
// line samples) of one level in ONE streaming pass over its bits (replaces
// dir_kernel + qlayout_kernel on the build path).
//
// A 256-thread CTA owns 1024 consecutive lines = 3072 words = three whole L1
// blocks, so it starts on both a line and an L1 boundary and needs no look-up
// into a directory.  Thread t owns lines [4t, 4t + 4) = words [12t, 12t + 12)
// (six 16-byte loads, all in flight at once); one warp scan of the thread
// counts and one barrier for the warp sums give every line header on top of
// l1[3 g].  Each line leaves as one 32-byte store (a whole sector).  Inside
// the CTA everything is 32-bit: the L2 entry of word w is (ones of the CTA
// before w) - (l1[w >> 10] - l1[3 g]); a line holds at most three line
// samples of each kind.  Reference samples (~three of each kind per warp at
// rate 4096): a warp-uniform loop over the ordinals of the warp's range, the
// owning lane selects in its twelve words.
// ---------------------------------------------------------------------------
constexpr int DQ_NT = 256;                 // threads per CTA
constexpr int DQ_LPT = 4;                  // lines per thread
constexpr int DQ_WPT = DQ_LPT * 3;         // words per thread
constexpr int DQ_LINES = DQ_LPT * DQ_NT;   // lines per CTA
static_assert(kQW == 3 && DQ_LINES * kQW == 3 * (kL1Bits / 64),
              "dirq_kernel aligns three L1 blocks with 1024 lines of 3 words");
static_assert((1 << kQSelLog) >= kQBits / 3, "at most three line samples per line");

__device__ __forceinline__ u64 dq_next_multiple(u64 o, u64 rate, int rate_log) {
  if (rate_log >= 0) return ((o >> rate_log) + 1) << rate_log;
  return (o / rate + 1) * rate;
}

__device__ __forceinline__ void dq_store_line(ulonglong2* p, u64 a, u64 b, u64 c, u64 d) {
  asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d)
               : "memory");
}

// line samples of one kind: sel[j] = line for every j with j * 2^kQSelLog + 1
// in (before, before + cnt] (at most three: cnt <= 192), staged in shared
// memory as the CTA-local line at j - jbase (the CTA's first sample index)
// (32-bit: `rb` = the CTA's count before the line + (count before the CTA
// mod 2^kQSelLog), `ob` = (that residue + 2^kQSelLog - 1) >> kQSelLog)
__device__ __forceinline__ void dq_line_samples(u16* ss, u32 ob, u32 rb, u32 cnt, u32 line) {
  constexpr u32 SR = (1u << kQSelLog) - 1;
  const u32 j0 = (rb + SR) >> kQSelLog;
  const u32 k = ((rb + cnt + SR) >> kQSelLog) - j0;
  const u32 o = j0 - ob;
#pragma unroll
  for (u32 x = 0; x < 3; ++x)
    if (x < k) ss[o + x] = (u16)line;
}

__device__ __forceinline__ u32 dq_smem(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void dq_load_group(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(dq_smem(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dq_smem(dst)),
      "l"(src), "r"(bytes), "r"(dq_smem(bar))
      : "memory");
}
__device__ __forceinline__ void dq_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(dq_smem(bar)),
      "r"(parity)
      : "memory");
}

constexpr int DQ_GWORDS = 3 * (kL1Bits / 64);  // words per CTA group (3072)
constexpr int DQ_GBYTES = DQ_GWORDS * 8;       // 24 KiB
constexpr int DQ_SSEL = DQ_GWORDS * 64 / (1 << kQSelLog) + 4;  // line samples of one kind per CTA
constexpr int DQ_SMEM = 2 * DQ_GBYTES + 64 + 2 * DQ_SSEL * 2;  // group buffers, mbarriers, staged samples

// One group (CTA-local 32-bit arithmetic throughout).  FULL: every bit of the
// group lies inside the level (all groups but the level's last), so no bound
// checks.  The thread's words are in `w`; the group buffer `slot` may be
// refilled once every thread holds its words (after the scan barrier).
template <bool FULL>
__device__ __forceinline__ void dq_group(const DirQParams& Q, const u64 (&w)[DQ_WPT], u64 g, u32 slot,
                                         u32 (*wsum)[DQ_NT / 32], u16* ss1, u16* ss0, u64* buf,
                                         u64* mbar, u64 gfull, u64 total) {
  const DirParams& P = Q.d;
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 nw = (P.m + 63) >> 6;
  const u64 n_l1 = (P.m + kL1Bits - 1) / kL1Bits;
  const u32 l2m = (u32)((1ull << P.l2_log) >> 6) - 1u;  // L2 block = l2m + 1 words (<= 1024)
  const u32 l2wl = P.l2_log - 6;
  constexpr u32 SR = (1u << kQSelLog) - 1;
  const u64 gw0 = g * DQ_GWORDS;           // the CTA's first word
  const u64 w0 = gw0 + (u64)tid * DQ_WPT;  // this thread's first word
  const u64 l1a = FULL || 3 * g < n_l1 ? __ldg(P.l1 + 3 * g) : total;  // ones before the CTA
  const u32 d1 = FULL || 3 * g + 1 < n_l1 ? (u32)(__ldg(P.l1 + 3 * g + 1) - l1a) : 0u;
  const u32 d2 = FULL || 3 * g + 2 < n_l1 ? (u32)(__ldg(P.l1 + 3 * g + 2) - l1a) : 0u;
  u32 pc[DQ_WPT], c = 0;
#pragma unroll
  for (int j = 0; j < DQ_WPT; ++j) {
    pc[j] = __popcll(w[j]);
    c += pc[j];
  }
  u32 inc = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= (u32)d) inc += y;
  }
  if (lane == 31) wsum[slot][warp] = inc;
  __syncthreads();  // every thread holds its words: the buffer may be refilled
  if (tid == 0) {
    const u64 gg = g + 2 * (u64)gridDim.x;
    if (gg < gfull) dq_load_group(buf + slot * DQ_GWORDS, P.words + gg * DQ_GWORDS, DQ_GBYTES, &mbar[slot]);
  }
  u32 wpre = 0, ctot = 0;
#pragma unroll
  for (int k = 0; k < DQ_NT / 32; ++k) {
    const u32 x = wsum[slot][k];
    wpre += (u32)k < warp ? x : 0u;
    ctot += x;
  }
  const u32 rel0 = wpre + inc - c;  // ones of the CTA before this thread
  const u64 gb0 = gw0 << 6;
  // valid bits of this thread / of the CTA
  const u32 vt = FULL ? 64u * DQ_WPT : (w0 << 6) < P.m ? (u32)min(P.m - (w0 << 6), (u64)(64 * DQ_WPT)) : 0u;
  const u32 vg = FULL ? 64u * DQ_GWORDS : gb0 < P.m ? (u32)min(P.m - gb0, (u64)DQ_GWORDS * 64) : 0u;
  const u64 zg = (FULL || gb0 < P.m ? gb0 : P.m) - l1a;  // zeros before the CTA
  // the CTA's line samples: indices [jb, jb + n) of sel1 / sel0; per line the
  // 32-bit residue arithmetic of dq_line_samples
  const u32 r1 = (u32)l1a & SR, r0 = (u32)zg & SR;
  const u32 ob1 = (r1 + SR) >> kQSelLog, ob0 = (r0 + SR) >> kQSelLog;
  // ---- lines, line samples, L2 entries ---------------------------------------
  {
    u32 rel = rel0;
#pragma unroll
    for (int x = 0; x < DQ_LPT; ++x) {
      const u32 li = tid * DQ_LPT + x;  // line inside the CTA
      const u64 i = g * DQ_LINES + li;
      const u32 cl = pc[3 * x] + pc[3 * x + 1] + pc[3 * x + 2];
      const u32 vl = FULL ? (u32)kQBits
                          : vt > (u32)(kQBits * x) ? min(vt - (u32)(kQBits * x), (u32)kQBits) : 0u;
      if (FULL || i < Q.n_lines) {
        dq_store_line(Q.lines + i * kQLineU2, l1a + rel, w[3 * x], w[3 * x + 1], w[3 * x + 2]);
        dq_line_samples(ss1, ob1, r1 + rel, cl, li);
        if (FULL || vl) dq_line_samples(ss0, ob0, r0 + (li * (u32)kQBits - rel), vl - cl, li);
      }
      // L2 entries (3072 words per CTA: a multiple of every L2 block size)
      u32 pre = rel;
#pragma unroll
      for (int y = 0; y < 3; ++y) {
        const u32 lw = tid * DQ_WPT + 3 * x + y;  // word inside the CTA
        if ((lw & l2m) == 0 && (FULL || w0 + 3 * x + y < nw)) {
          const u32 blk = lw >> 10;
          P.l2[(gw0 + lw) >> l2wl] = (u16)(pre - (blk == 0 ? 0u : blk == 1 ? d1 : d2));
        }
        pre += pc[3 * x + y];
      }
      rel += cl;
    }
  }
  // ---- reference samples: each lane its own ordinals (at rate 4096 a lane
  // holds at most one of each kind; ~three lanes of a warp hold one) ---------
  const u64 hb = l1a + rel0;                                      // ones before this thread
  const u64 zbt = (FULL || (w0 << 6) < P.m ? (w0 << 6) : P.m) - hb;  // zeros before this thread
#pragma unroll
  for (int kind = 0; kind < 2; ++kind) {
    const bool ones = kind == 0;
    const u64 bl = ones ? hb : zbt;
    const u32 cl = ones ? c : vt - c;
    for (u64 qo = dq_next_multiple(bl, P.rate, P.rate_log); qo <= bl + cl; qo += P.rate) {
      // word j holding ordinal k: k > (kind's count of words 0..i) for i < j
      const u32 k = (u32)(qo - bl);
      u32 j = 0, before = 0, acc = 0;
#pragma unroll
      for (int i = 0; i < DQ_WPT - 1; ++i) {
        const u32 vb = FULL ? 64u : vt > 64u * i ? min(64u, vt - 64u * i) : 0u;
        acc += ones ? pc[i] : vb - pc[i];
        const bool past = k > acc;
        j += past ? 1u : 0u;
        before = past ? acc : before;
      }
      u64 wv = w[0];
#pragma unroll
      for (int i = 1; i < DQ_WPT; ++i) wv = j == (u32)i ? w[i] : wv;
      const u32 vb = FULL ? 64u : vt > 64u * j ? min(64u, vt - 64u * j) : 0u;
      wv = (ones ? wv : ~wv) & (vb >= 64 ? ~0ull : (1ull << vb) - 1ull);
      const u64 pos = ((w0 + j) << 6) + select_in_word64(wv, k - before);
      const u64 si = (P.rate_log >= 0 ? (qo >> P.rate_log) : qo / P.rate) - 1;
      u64* o = ones ? P.ones : P.zeros;
      if (si < (ones ? P.ones_cap : P.zeros_cap)) o[si] = pos;
    }
  }
  // ---- the staged line samples leave coalesced (sel_cap exceeds every index)
  __syncthreads();
  {
    const u32 gl = (u32)(g * DQ_LINES);
    const u64 jb1 = (l1a + SR) >> kQSelLog, jb0 = (zg + SR) >> kQSelLog;
    const u32 n1 = (u32)(((l1a + ctot + SR) >> kQSelLog) - jb1);
    const u32 n0 = (u32)(((zg + (vg - ctot) + SR) >> kQSelLog) - jb0);
    u32* s1 = Q.sel1 + jb1;
    u32* s0 = Q.sel0 + jb0;
    for (u32 x = tid; x < n1; x += DQ_NT) s1[x] = gl + ss1[x];
    for (u32 x = tid; x < n0; x += DQ_NT) s0[x] = gl + ss0[x];
  }
}

// Persistent: CTA b takes groups b, b + grid, ...; the next group's 24 KiB
// stream into the other shared buffer by one bulk copy (cp.async.bulk +
// mbarrier) while this one is processed, so each SM keeps ~100 KiB of reads in
// flight without spending registers on them.  The level's partial last
// group (its words end inside it) loads directly from global memory.
#ifndef DQ_MINB
#define DQ_MINB 3
#endif
__global__ void __launch_bounds__(DQ_NT, DQ_MINB) dirq_kernel(const __grid_constant__ DirQParams Q) {
  const DirParams& P = Q.d;
  extern __shared__ __align__(128) u8 dq_sm[];
  u64* buf = reinterpret_cast<u64*>(dq_sm);
  u64* mbar = reinterpret_cast<u64*>(dq_sm + 2 * DQ_GBYTES);
  u16* ss1 = reinterpret_cast<u16*>(dq_sm + 2 * DQ_GBYTES + 64);  // staged line samples
  u16* ss0 = ss1 + DQ_SSEL;
  __shared__ u32 wsum[2][DQ_NT / 32];
  const u32 tid = threadIdx.x;
  const u64 nw = (P.m + 63) >> 6;
  const u64 ng = (Q.n_lines + DQ_LINES - 1) / DQ_LINES;
  const u64 gfull = nw / DQ_GWORDS;                           // groups whose words all lie inside the level
  const u64 gbits = P.m / ((u64)DQ_GWORDS * 64);              // groups whose bits all do
  const u64 total = *Q.total;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(dq_smem(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(dq_smem(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (u32 k = 0; k < 2; ++k) {
      const u64 gg = blockIdx.x + (u64)k * gridDim.x;
      if (gg < gfull) dq_load_group(buf + k * DQ_GWORDS, P.words + gg * DQ_GWORDS, DQ_GBYTES, &mbar[k]);
    }
  }
  __syncthreads();
  u32 it = 0;
  for (u64 g = blockIdx.x; g < ng; g += gridDim.x, ++it) {
    const u32 slot = it & 1u;
    const u64 w0 = g * DQ_GWORDS + (u64)tid * DQ_WPT;  // this thread's first word
    u64 w[DQ_WPT];
    if (g < gfull) {
      dq_wait(&mbar[slot], (it >> 1) & 1u);
      const ulonglong2* src = reinterpret_cast<const ulonglong2*>(buf + slot * DQ_GWORDS + tid * DQ_WPT);
#pragma unroll
      for (int j = 0; j < DQ_WPT / 2; ++j) {
        const ulonglong2 v = src[j];
        w[2 * j] = v.x;
        w[2 * j + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < DQ_WPT; ++j) w[j] = w0 + j < nw ? __ldg(P.words + w0 + j) : 0ull;  // padding bits are zero
    }
    if (g < gbits)
      dq_group<true>(Q, w, g, slot, wsum, ss1, ss0, buf, mbar, gfull, total);
    else
      dq_group<false>(Q, w, g, slot, wsum, ss1, ss0, buf, mbar, gfull, total);
  }
}

cudaError_t launch_dirq(const DirQParams& p, int sms, cudaStream_t st, bool pdl) {
  if (!p.n_lines) return cudaSuccess;
  static std::atomic<int> per_sm_cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  const bool dev_ok = dev >= 0 && dev < 64;
  int per_sm = dev_ok ? per_sm_cache[dev].load(std::memory_order_acquire) : 0;
  if (per_sm <= 0) {  // the shared-memory opt-in belongs to the device context
    cudaError_t e = cudaFuncSetAttribute(dirq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DQ_SMEM);
    if (e != cudaSuccess) return e;
    per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dirq_kernel, DQ_NT, DQ_SMEM);
    if (per_sm < 1) per_sm = 1;
    if (dev_ok) per_sm_cache[dev].store(per_sm, std::memory_order_release);
  }
  const u64 ncta = (p.n_lines + DQ_LINES - 1) / DQ_LINES;
  const u64 cap = (u64)sms * per_sm;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ncta < cap ? ncta : cap));
  cfg.blockDim = dim3(DQ_NT);
  cfg.dynamicSmemBytes = DQ_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, dirq_kernel, p);
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
