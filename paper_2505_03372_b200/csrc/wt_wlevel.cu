// wt_wlevel.cu -- K2w: one fused pass per wavelet-tree level, WARP-granular tiles.
//
// Replaces, for level l, the reference's
//   stable_sort_by_prefix  (wtree.py:92-100)        -> one-pass stable per-node partition
//   fill_level / fill_region / _pack_span (wtree.py:103-107, bitvec.py:119-151)
//   build_index (rankselect.py:442-536): L2 entries and select samples
//   (L1 entries come from the per-L1-block scan that precedes the launch)
//
// Every warp owns whole tiles of 4 KiB of input (4096 u8 / 2048 u16
// elements) and never waits for another warp: no __syncthreads in the loop.
// Per tile:
//   0. the tile streams into a per-warp shared-memory ring (cp.async.bulk +
//      mbarrier), W_RING tiles ahead (one: 6 CTAs per SM fit);
//   1. lane rows: a tile is 16 (u8) / 8 (u16) rows of 256 elements, lane i
//      owns elements [8i, 8i + 8) of each row; one 8-bit mask per lane-row
//      (SWAR bit extraction, or `symbol >= thr` at a LUT level 0), packed warp
//      scans of the row counts; the masks are the tile's bit-vector bytes;
//   2. P1 (ones before the tile) = L1 prefix of its 65536-bit block + the
//      counts of the block's earlier tiles (counted by the previous level;
//      level 0 of a large u8 text: the warp walks whole blocks, "block mode");
//   3. single-node tile (the common case; two-node tiles at u16 codes): every
//      element goes to a warp-private staging buffer at its place in the
//      zeros run or the ones run (offsets congruent to the global destination
//      mod 16); each run body leaves as ONE cp.async.bulk shared -> global
//      store, heads / tails by lanes;
//   4. the staged runs are counted (AND + POPC) for the ones of the NEXT
//      level's bit per next-level tile / L1 block (a few atomics per run):
//      this is what makes step 2 possible for the next level without a
//      look-back;
//   5. L2 entries and select samples from (P1, in-tile prefix).
// Multi-node tiles (node boundaries inside the tile) store element by element.
// Destination of element j with bit b in node `key`:
//   b=1: one_base[key] + R1(j)        b=0: zero_base[key] + R0(j)
#include <atomic>
#include <cstdlib>
#include "wt_common.cuh"
#include "wt_kernels.h"

namespace wt {
namespace {

constexpr int W_NT = 128;
constexpr int W_WARPS = W_NT / 32;
#ifndef WT_W_RING
#define WT_W_RING 1
#endif
constexpr int W_RING = WT_W_RING;  // input tiles in flight per warp
#ifndef WT_W_NSTAGE
#define WT_W_NSTAGE 1
#endif
constexpr int W_NSTAGE = WT_W_NSTAGE;  // staging buffers per warp (1 | 2)
#ifndef WT_W_MINB
#define WT_W_MINB 6
#endif
constexpr int W_MINB = WT_W_MINB;  // __launch_bounds__ min CTAs per SM
#ifndef WT_W_MINB4
#define WT_W_MINB4 6
#endif
constexpr int W_MINB4 = WT_W_MINB4;  // the same for 4 KiB tiles (u8 input)
#ifndef WT_SAG
#define WT_SAG 0  // u8 levels: sheep-and-goats permutation scatter (measured slower than the cursors)
#endif
constexpr unsigned FULLM = 0xffffffffu;

// a warp tile is 2048 elements for both input widths (2 KiB of u8 / 4 KiB
// of u16), so per-tile costs are amortized alike and every level's tile
// counts have the same granularity
#ifndef WT_U8_TILE
#define WT_U8_TILE 4096
#endif
template <typename TIn>
struct WS {
  static constexpr int CH = 16 / (int)sizeof(TIn);          // elements per 16-byte chunk
  static constexpr int TILE = sizeof(TIn) == 1 ? WT_U8_TILE : 2048;  // elements per warp tile
  static constexpr int LOG = TILE == 4096 ? 12 : 11;
  static constexpr int BYTES = TILE * (int)sizeof(TIn);     // 2048 | 4096
  static constexpr int K = BYTES / 512;                     // 16-byte chunks per lane (4 | 8)
  static constexpr int TPL1 = kL1Bits / TILE;               // 32 tiles per L1 block
};

__device__ __forceinline__ u32 smem_addr(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void w_bulk_s2g(void* dst, const void* src, u32 bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void w_bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void w_bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void w_bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void w_bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void w_fence_proxy() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// bit `sh` of every element of WPC packed code words -> LSB-first mask
template <typename TC, int WPC>
__device__ __forceinline__ u32 wmask(const u32 (&cw)[WPC], u32 sh) {
  u32 m = 0;
  if (sizeof(TC) == 1) {
    // two words (8 elements) per multiply: bits at 8b (word 0) and 8b+4
    // (word 1) gather to bits 24..31 in element order
#pragma unroll
    for (int i = 0; i + 1 < WPC; i += 2) {
      const u32 y0 = (cw[i] >> sh) & 0x01010101u;
      const u32 y1 = (cw[i + 1] >> sh) & 0x01010101u;
      const u32 z = y1 * 16u + y0;
      m |= ((z * 0x01020408u) >> 24) << (4 * i);
    }
    if (WPC & 1) {
      const u32 y = (cw[WPC - 1] >> sh) & 0x01010101u;
      m |= ((y * 0x01020408u) >> 24) << (4 * (WPC - 1));
    }
  } else {
    // two words (4 elements) per step: z = y0 + 4*y1 holds bits 0, 16, 2, 18
    // for elements 0..3; (z | z >> 15) & 15 puts them in order
#pragma unroll
    for (int i = 0; i + 1 < WPC; i += 2) {
      const u32 y0 = (cw[i] >> sh) & 0x00010001u;
      const u32 y1 = (cw[i + 1] >> sh) & 0x00010001u;
      const u32 z = y1 * 4u + y0;
      m |= ((z | (z >> 15)) & 15u) << (2 * i);
    }
    if (WPC & 1) {
      const u32 y = (cw[WPC - 1] >> sh) & 0x00010001u;
      m |= ((y | (y >> 15)) & 3u) << (2 * (WPC - 1));
    }
  }
  return m;
}

template <typename TC, int WPC>
__device__ __forceinline__ u32 welem(const u32 (&cw)[WPC], int j) {
  if (sizeof(TC) == 1) return (cw[j >> 2] >> ((j & 3) * 8)) & 0xffu;
  return (cw[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
}

// 16 input bytes -> WPC code words (level 0 maps raw symbols through the LUT)
template <typename TIn, typename TC, bool kLut, int WPC>
__device__ __forceinline__ void wcodes(const uint4& q, const u16* slut, const u16* glut,
                                       u32 (&cw)[WPC]) {
  const u32 qw[4] = {q.x, q.y, q.z, q.w};
  if (!kLut) {
#pragma unroll
    for (int i = 0; i < WPC; ++i) cw[i] = qw[i];
  } else {
    constexpr int CH = 16 / (int)sizeof(TIn);
#pragma unroll
    for (int i = 0; i < WPC; ++i) cw[i] = 0;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const u32 raw = sizeof(TIn) == 1 ? (qw[j >> 2] >> ((j & 3) * 8)) & 0xffu
                                       : (qw[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
      const u32 code = sizeof(TIn) == 1 ? (u32)slut[raw] : (u32)__ldg(glut + raw);
      if (sizeof(TC) == 1)
        cw[j >> 2] |= code << ((j & 3) * 8);
      else
        cw[j >> 1] |= code << ((j & 1) * 16);
    }
  }
}

__device__ __forceinline__ uint4 w_load16(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// load one tile's 4 chunks per lane; bytes beyond the level are zero
template <typename TIn>
__device__ __forceinline__ void wload(const u8* in, u64 m, u32 t, int lane,
                                      uint4 (&q)[WS<TIn>::K]) {
  using S = WS<TIn>;
  const u64 t0 = (u64)t * S::TILE;
  const u8* base = in + t0 * sizeof(TIn);
  if (t0 + S::TILE <= m) {
#pragma unroll
    for (int k = 0; k < S::K; ++k) q[k] = w_load16(base + (k * 32 + lane) * 16);
  } else {
    const u64 bytes = (m - t0) * sizeof(TIn);
#pragma unroll
    for (int k = 0; k < S::K; ++k) {
      const u32 o = (u32)(k * 32 + lane) * 16;
      if (o + 16 <= bytes) {
        q[k] = w_load16(base + o);
      } else {
        u32 w[4] = {0, 0, 0, 0};
        for (u32 b = o; b < bytes && b < o + 16; ++b) w[(b - o) >> 2] |= (u32)base[b] << (8 * ((b - o) & 3));
        q[k] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
}

__device__ __forceinline__ u64 wnext_multiple(u64 o, u64 rate, int rate_log) {
  if (rate_log >= 0) return ((o >> rate_log) + 1) << rate_log;
  return (o / rate + 1) * rate;
}

}  // namespace

// Any tile the fast path does not take (the level's partial last tile, tiles
// spanning several nodes): loads from global memory, element-by-element
// destination stores, per-element next-level counts.
// returns the tile's ones (block mode: the caller's running count)
#ifndef WT_GT_UNROLL
#define WT_GT_UNROLL 1
#endif
constexpr int kGtUnroll = WT_GT_UNROLL;  // general_tile's per-element loop
template <typename TIn, typename TC, bool kLut, int MODE>
__device__ __noinline__ u32 general_tile(const WLevelParams& P, u32 t, const u16* slut, u64 p1_in) {
  constexpr bool kPair = MODE == 2, kBlk = MODE == 1;
  using S = WS<TIn>;
  constexpr int CH = S::CH, TILE = S::TILE, TPL1 = S::TPL1;
  constexpr int WPC = CH * (int)sizeof(TC) / 4;
  constexpr int NTILE_LOG = WS<TC>::LOG;  // next level's tile (its input = codes)
  const int lane = threadIdx.x & 31;
  const bool scatter = kPair || P.out != nullptr;
  const u8* in = reinterpret_cast<const u8*>(P.in);
  const u32 l2_chunks = (1u << P.l2_log) / CH;
  uint4 q[S::K];
  wload<TIn>(in, P.m, t, lane, q);
  u32 cw[S::K][WPC];
#pragma unroll
  for (int k = 0; k < S::K; ++k) wcodes<TIn, TC, kLut, WPC>(q[k], slut, P.lut, cw[k]);
    const u64 t0 = (u64)t * TILE;
    const u32 valid = (u32)min((u64)TILE, P.m - t0);
    // ---- P1: ones before the tile (block mode: the caller's running count) ---
    const u32 b = t / TPL1;
    const u32 tb = t - b * TPL1;  // tiles of the block before this one
    u32 pre = 0;
    if (p1_in == ~0ull) {
#pragma unroll
      for (int r = 0; r < (TPL1 + 31) / 32; ++r) {
        const u32 j = r * 32 + lane;
        if (j < tb) pre += __ldg(P.tile_counts + b * TPL1 + j);
      }
#pragma unroll
      for (int d = 16; d; d >>= 1) pre += __shfl_xor_sync(FULLM, pre, d);
    }
    const u64 l1v = __ldg(P.l1 + b);
    const u64 P1 = p1_in == ~0ull ? l1v + pre : p1_in;

    // ---- 1. codes, masks, in-tile scan ---------------------------------------
    u32 msk[S::K];
#pragma unroll
    for (int k = 0; k < S::K; ++k) {
      u32 mk = wmask<TC, WPC>(cw[k], P.shift_bit);
      const u32 e = (u32)(k * 32 + lane) * CH;
      if (e + CH > valid) mk &= e >= valid ? 0u : (1u << (valid - e)) - 1u;
      msk[k] = mk;
    }
    u32 r1c[S::K], ktot[S::K];
#pragma unroll
    for (int k = 0; k < S::K; k += 2) {
      const u32 x = (u32)__popc(msk[k]) | ((u32)__popc(msk[k + 1]) << 16);
      u32 inc = x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 y = __shfl_up_sync(FULLM, inc, d);
        if (lane >= d) inc += y;
      }
      const u32 tot = __shfl_sync(FULLM, inc, 31);
      const u32 ex = inc - x;
      r1c[k] = ex & 0xffffu;
      r1c[k + 1] = ex >> 16;
      ktot[k] = tot & 0xffffu;
      ktot[k + 1] = tot >> 16;
    }
    u32 tile_ones = 0;
#pragma unroll
    for (int k = 0; k < S::K; ++k) {
      r1c[k] += tile_ones;
      tile_ones += ktot[k];
    }

    // ---- bit-vector words -----------------------------------------------------
#pragma unroll
    for (int k = 0; k < S::K; ++k) {
      const u32 e = (u32)(k * 32 + lane) * CH;
      if (e < ((valid + 63u) & ~63u)) {  // through the level's last word: padding stays zero
        const u64 bit = t0 + e;
        if (CH == 16)
          reinterpret_cast<u16*>(P.words)[bit >> 4] = (u16)msk[k];
        else
          reinterpret_cast<u8*>(P.words)[bit >> 3] = (u8)msk[k];
      }
    }

    // ---- L2 entries ----------------------------------------------------------
    if (l2_chunks <= 32) {
      if ((lane & (l2_chunks - 1)) == 0) {
#pragma unroll
        for (int k = 0; k < S::K; ++k) {
          const u32 e = (u32)(k * 32 + lane) * CH;
          if (e < valid) P.l2[(t0 + e) >> P.l2_log] = (u16)(P1 + r1c[k] - l1v);
        }
      }
    } else if (lane == 0) {
      const u64 l2m = (1ull << P.l2_log) - 1;
#pragma unroll
      for (int k = 0; k < S::K; ++k) {
        const u64 g = t0 + (u64)k * 32 * CH;
        if (g < P.m && (g & l2m) == 0) P.l2[g >> P.l2_log] = (u16)(P1 + r1c[k] - l1v);
      }
    }

    // ---- select samples (rankselect.py:509-532) ------------------------------
#pragma unroll
    for (int kind = 0; kind < 2; ++kind) {
      const bool ones = kind == 0;
      const u64 base = ones ? P1 : t0 - P1;
      const u32 cnt = ones ? tile_ones : valid - tile_ones;
      u64* out = ones ? P.ones : P.zeros;
      const u64 cap = ones ? P.ones_cap : P.zeros_cap;
      for (u64 qo = wnext_multiple(base, P.rate, P.rate_log); qo <= base + cnt; qo += P.rate) {
        const u32 tt = (u32)(qo - base);  // 1-based ordinal inside the tile
        u32 kk = S::K - 1, acc = 0;  // k-row holding ordinal tt
#pragma unroll
        for (int k = 0; k < S::K; ++k) {
          const int rv = (int)valid - k * 32 * CH;
          const u32 row_valid = rv <= 0 ? 0u : (rv >= 32 * CH ? 32u * CH : (u32)rv);
          const u32 kc = ones ? ktot[k] : row_valid - ktot[k];
          if (tt <= acc + kc) { kk = k; break; }
          acc += kc;
        }
        // lane owning ordinal tt within k-row kk
        u32 pre_l = 0, cnt_l = 0, mk = 0;
#pragma unroll
        for (int k = 0; k < S::K; ++k) {
          if ((u32)k == kk) {
            const u32 e = (u32)(k * 32 + lane) * CH;
            const u32 vm = e >= valid ? 0u : (e + CH <= valid ? (CH == 16 ? 0xffffu : 0xffu)
                                                              : (1u << (valid - e)) - 1u);
            mk = ones ? msk[k] : (~msk[k] & vm);
            pre_l = ones ? r1c[k] : (u32)(k * 32 + lane) * CH - r1c[k];
            cnt_l = __popc(mk);
          }
        }
        const u32 own = __ballot_sync(FULLM, pre_l < tt && tt <= pre_l + cnt_l);
        if (own && lane == __ffs(own) - 1) {
          const u64 s = (P.rate_log >= 0 ? (qo >> P.rate_log) : qo / P.rate) - 1;
          if (s < cap) out[s] = t0 + (u64)(kk * 32 + lane) * CH + select_in_word32(mk, tt - pre_l);
        }
      }
    }

    if (!scatter) return tile_ones;

    {
      TC* gout = reinterpret_cast<TC*>(P.out);
      const u32 sh1 = P.shift_bit - 1;
      // (rolled loops: this path is rare on most levels, but where tiles
      // span many nodes -- Zipf texts, deep u16 levels -- the unrolled body
      // thrashed the instruction cache: ncu `no_instructions` 52 %)
#pragma unroll 1
      for (int k = 0; k < S::K; ++k) {
        const u32 e = (u32)(k * 32 + lane) * CH;
        u32 r1 = r1c[k];
#pragma unroll(kGtUnroll)
        for (int j = 0; j < CH; ++j) {
          // next-level ones, warp-aggregated per destination tile: lanes
          // whose element lands in the same next-level tile add together
          u32 tf = 0xffffffffu;
          if (e + j < valid) {
            const u32 v = welem<TC, WPC>(cw[k], j);
            const NodeEnt* ne = P.nodes + (v >> P.shift_key);
            const u32 bt = (msk[k] >> j) & 1u;
            const u64 dst = bt ? (u64)__ldg(&ne->one_base) + P1 + r1
                               : (u64)__ldg(&ne->zero_base) + (t0 + e + j - P1 - r1);
            if (dst < P.m_next) {
              if (kPair) {  // the last level's bit at its position (region zeroed)
                if ((v >> sh1) & 1u) {
                  atomicOr(reinterpret_cast<u32*>(P.next_words) + (dst >> 5), 1u << (dst & 31));
                  tf = (u32)(dst >> 16);
                }
              } else {
                gout[dst] = (TC)v;
                if ((v >> sh1) & 1u) tf = (u32)(dst >> (kBlk ? 16 : NTILE_LOG));
              }
            }
            r1 += bt;
          }
          const u32 key = tf != 0xffffffffu ? tf : 0x80000000u | (u32)lane;  // unique if none
          const unsigned peers = __match_any_sync(FULLM, key);
          if (tf != 0xffffffffu && lane == __ffs(peers) - 1) {
            if (kPair || kBlk) {  // per L1 block only
              atomicAdd(P.next_l1_counts + tf, (u32)__popc(peers));
            } else {
              atomicAdd(P.next_tile_counts + tf, (u32)__popc(peers));
              atomicAdd(P.next_l1_counts + (((u64)tf << NTILE_LOG) >> 16), (u32)__popc(peers));
            }
          }
        }
      }
    }
    return tile_ones;
}

// ---------------------------------------------------------------------------
// the kernel: full single-node tiles take the fast path below
// ---------------------------------------------------------------------------
// Fast-path layout: a tile is 8 rows of 256 input bytes; lane i owns bytes
// [8i, 8i + 8) of every row (CR = 8 / sizeof(TIn) elements).  Lane regions in
// a staged run then span ~128 bytes per row step, so the byte stores of one
// step fall in distinct banks.
template <typename TIn, typename TC>
struct WF {
  static constexpr int CR = 8;                               // elements per lane per row
  static constexpr int RE = 256;                             // elements per row
  static constexpr int ROWS = WS<TIn>::TILE / RE;            // 8
  static constexpr int LB = CR * (int)sizeof(TIn);           // input bytes per lane-row (8 | 16)
  static constexpr int LW = LB / 4;                          // input words per lane-row
  static constexpr int RB = 32 * LB;                         // input bytes per row
  static constexpr int WR = CR * (int)sizeof(TC) / 4;        // code words per lane-row
  static constexpr int STAGE = ((WS<TIn>::TILE * (int)sizeof(TC) + 128) + 127) & ~127;  // 4 runs
  static constexpr int WARP_SMEM = W_RING * WS<TIn>::BYTES + W_NSTAGE * STAGE + 64;
};

__device__ __forceinline__ void w_mbar_init(u64* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
}
__device__ __forceinline__ void w_load_tile(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void w_mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// codes of one lane-row (8 input elements, LW words) -> WR words
template <typename TIn, typename TC, bool kLut>
__device__ __forceinline__ void wrow_codes(const u32 (&v)[WF<TIn, TC>::LW], const u16* slut,
                                           const u16* glut, u32 (&cw)[WF<TIn, TC>::WR]) {
  constexpr int WR = WF<TIn, TC>::WR;
  if (!kLut) {
#pragma unroll
    for (int i = 0; i < WR; ++i) cw[i] = v[i];  // TIn == TC
  } else {
#pragma unroll
    for (int i = 0; i < WR; ++i) cw[i] = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const u32 raw = sizeof(TIn) == 1 ? (v[j >> 2] >> ((j & 3) * 8)) & 0xffu
                                       : (v[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
      const u32 code = sizeof(TIn) == 1 ? (u32)slut[raw] : (u32)__ldg(glut + raw);
      if (sizeof(TC) == 1)
        cw[j >> 2] |= code << ((j & 3) * 8);
      else
        cw[j >> 1] |= code << ((j & 1) * 16);
    }
  }
}

// one lane-row of the staged tile as LW words
template <int LW>
__device__ __forceinline__ void wrow_load(const u8* p, u32 (&v)[LW]) {
  if (LW == 2) {
    const uint2 x = *reinterpret_cast<const uint2*>(p);
    v[0] = x.x;
    v[LW - 1] = x.y;
  } else {
    const uint4 x = *reinterpret_cast<const uint4*>(p);
    v[0] = x.x; v[1 % LW] = x.y; v[2 % LW] = x.z; v[3 % LW] = x.w;
  }
}

// No "memory" clobber: the scatter's loads (ring rows, LUT) may be hoisted
// above these stores -- they read other buffers.  The stores stay ordered
// among themselves and before w_fence_proxy() (volatile asm, which clobbers
// memory) that publishes the staging buffer.
template <typename TC>
__device__ __forceinline__ void st_shared(u32 addr, u32 v) {
  if (sizeof(TC) == 1)
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v));
  else
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v));
}

// one element of a staged run, next-level bit
template <typename TC>
__device__ __forceinline__ u32 wbit_at(const u8* stage, u32 byte, u32 sh) {
  const u32 v = sizeof(TC) == 1 ? (u32)stage[byte] : (u32)*reinterpret_cast<const u16*>(stage + byte);
  return (v >> sh) & 1u;
}

// next-level ones of the zeros run (Z elements at stage byte zoff, global
// destination zdst) and of the ones run (O at ooff, odst), per next-level tile
// (a run spans <= 2 of them, <= 3 when kThree: u8 text -> u16 codes, whose
// next tiles are half as long) and L1 block.  Per run, one pass over its
// aligned 16-byte chunks (AND + POPC per word, no multiply), chunks wholly
// before a boundary also added to that boundary's prefix; element-wise passes
// for the run heads / tails and for the chunk holding a boundary.  Lanes 0..5
// add the counts.
template <typename TC>
__device__ __forceinline__ u32 wpop16(uint4 v, u32 msk) {
  return (u32)(__popc(v.x & msk) + __popc(v.y & msk)) + (u32)(__popc(v.z & msk) + __popc(v.w & msk));
}
template <typename TC, bool kThree>
__device__ __forceinline__ void wcount_tile(const u8* stage, u32 Z, u32 zoff, u64 zdst, u32 O,
                                            u32 ooff, u64 odst, u32 sh, int tile_log,
                                            u32* tcounts, u32* l1counts, int lane) {
  constexpr u32 SZ = sizeof(TC);
  constexpr u32 EPC = 16 / SZ;
  const u64 nt = 1ull << tile_log;
  const u32 msk = (sizeof(TC) == 1 ? 0x01010101u : 0x00010001u) << sh;
  // per run: head elements h, full chunks nf, tail start ts, boundaries b1 <= b2
  const u32 hz = min(Z, ((16u - (zoff & 15u)) & 15u) / SZ), nfz = (Z - hz) / EPC, tsz = hz + nfz * EPC;
  const u32 ho = min(O, ((16u - (ooff & 15u)) & 15u) / SZ), nfo = (O - ho) / EPC, tso = ho + nfo * EPC;
  const u32 b1z = min(Z, (u32)((((zdst >> tile_log) + 1) << tile_log) - zdst));
  const u32 b1o = min(O, (u32)((((odst >> tile_log) + 1) << tile_log) - odst));
  const u32 b2z = kThree ? min(Z, b1z + (u32)nt) : Z, b2o = kThree ? min(O, b1o + (u32)nt) : O;
  u32 az = 0, p1z = 0, p2z = 0, ao = 0, p1o = 0, p2o = 0;
  {
    const uint4* cz = reinterpret_cast<const uint4*>(stage + zoff + hz * SZ);
    const u32 c1 = b1z > hz ? (b1z - hz) / EPC : 0u, c2 = b2z > hz ? (b2z - hz) / EPC : 0u;
#pragma unroll 2
    for (u32 c = lane; c < nfz; c += 32) {
      const u32 x = wpop16<TC>(cz[c], msk);
      az += x;
      p1z += c < c1 ? x : 0u;
      if (kThree) p2z += c < c2 ? x : 0u;
    }
  }
  {
    const uint4* co = reinterpret_cast<const uint4*>(stage + ooff + ho * SZ);
    const u32 c1 = b1o > ho ? (b1o - ho) / EPC : 0u, c2 = b2o > ho ? (b2o - ho) / EPC : 0u;
#pragma unroll 2
    for (u32 c = lane; c < nfo; c += 32) {
      const u32 x = wpop16<TC>(co[c], msk);
      ao += x;
      p1o += c < c1 ? x : 0u;
      if (kThree) p2o += c < c2 ? x : 0u;
    }
  }
  // element-wise 1: heads and tails (lanes 0-7 z head, 8-15 z tail, 16-23 o head, 24-31 o tail;
  // EPC <= 16 so each is < 16 elements: two rounds)
#pragma unroll
  for (int rnd = 0; rnd < 2; ++rnd) {
    const u32 k = (lane & 7) + 8 * rnd;
    const bool one = lane >= 16, tail = (lane & 8) != 0;
    const u32 cnt = one ? O : Z, h = one ? ho : hz, ts = one ? tso : tsz;
    const u32 i = tail ? ts + k : k;
    const bool in = tail ? i < cnt : k < h;
    const u32 bt = in ? wbit_at<TC>(stage, (one ? ooff : zoff) + i * SZ, sh) : 0u;
    const u32 b1 = one ? b1o : b1z, b2 = one ? b2o : b2z;
    if (one) {
      ao += bt; p1o += i < b1 ? bt : 0u;
      if (kThree) p2o += i < b2 ? bt : 0u;
    } else {
      az += bt; p1z += i < b1 ? bt : 0u;
      if (kThree) p2z += i < b2 ? bt : 0u;
    }
  }
  // element-wise 2: the part before each boundary of the full chunk holding it
  // (lanes 0-7 b1z, 8-15 b2z, 16-23 b1o, 24-31 b2o; two rounds)
#pragma unroll
  for (int rnd = 0; rnd < 2; ++rnd) {
    const u32 k = (lane & 7) + 8 * rnd;
    const bool one = lane >= 16, second = (lane & 8) != 0;
    if (!kThree && second) continue;
    const u32 h = one ? ho : hz, ts = one ? tso : tsz;
    const u32 bb = one ? (second ? b2o : b1o) : (second ? b2z : b1z);
    const bool strad = bb > h && bb < ts && ((bb - h) % EPC) != 0;
    const u32 i = (strad ? h + ((bb - h) / EPC) * EPC : 0u) + k;
    const bool in = strad && i < bb;
    const u32 bt = in ? wbit_at<TC>(stage, (one ? ooff : zoff) + i * SZ, sh) : 0u;
    if (one) {
      if (second) p2o += bt; else p1o += bt;
    } else {
      if (second) p2z += bt; else p1z += bt;
    }
  }
  u32 q0 = az | (ao << 16), q1 = p1z | (p1o << 16), q2 = p2z | (p2o << 16);  // counts <= 4096
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    q0 += __shfl_xor_sync(FULLM, q0, d);
    q1 += __shfl_xor_sync(FULLM, q1, d);
    if (kThree) q2 += __shfl_xor_sync(FULLM, q2, d);
  }
  if (!kThree) q2 = q0;  // a run spans at most two next-level tiles: nothing past b2
  if (lane < 6) {
    const bool one = lane >= 3;
    const int seg = lane - (one ? 3 : 0);
    const u32 sft = one ? 16 : 0;
    const u32 a = (q0 >> sft) & 0xffffu, c1 = (q1 >> sft) & 0xffffu, c2 = (q2 >> sft) & 0xffffu;
    const u32 cc = seg == 0 ? c1 : seg == 1 ? c2 - c1 : a - c2;
    if (cc) {
      const u64 tf = ((one ? odst : zdst) >> tile_log) + seg;
      atomicAdd(tcounts + tf, cc);
      if (l1counts) atomicAdd(l1counts + ((tf << tile_log) >> 16), cc);
    }
  }
}

// Pair mode: the staged run of `cnt` codes at stage byte `soff` (soff = dst *
// sizeof(TC) mod 16) lands at positions [dst, dst + cnt) of the LAST level,
// whose bits are the codes' bit `sh`.  Every aligned 16-byte chunk of the
// staging is one aligned 16-bit (u8 codes) / 8-bit (u16) piece of that
// level's bit-vector: one SWAR gather per chunk, plain stores for the chunks
// inside the run, atomicOr for its (partial) first / last chunk -- the
// neighbouring runs own the other bits of those words (region zeroed before
// the launch).  The run's ones are added to the level's per-L1-block counts
// (a run of <= 4096 codes crosses at most one block boundary).
template <typename TC>
__device__ __forceinline__ void wpair_bits(const u8* stage, u32 cnt, u32 soff, u64 dst, u32 sh,
                                           u64* nwords, u32* l1counts, int lane) {
  constexpr u32 SZ = sizeof(TC), EPC = 16 / SZ;
  const u32 h = (soff & 15u) / SZ;  // chunk 0 elements before the run
  const u32 nch = (h + cnt + EPC - 1) / EPC;
  const u64 g0 = dst - h;           // chunk 0's first position (a multiple of EPC)
  const u8* base = stage + (soff & ~15u);
  const u64 bnd = ((dst >> 16) + 1) << 16;
  constexpr u32 FULLC = (1u << EPC) - 1u;
  u32 clo = 0, chi = 0;
  for (u32 c = lane; c < nch; c += 32) {
    const uint4 q = *reinterpret_cast<const uint4*>(base + 16 * c);
    const u32 cw[4] = {q.x, q.y, q.z, q.w};
    u32 m = wmask<TC, 4>(cw, sh);
    const u32 lo = c == 0 ? h : 0u;
    const u32 hi = min(EPC, h + cnt - c * EPC);
    const u32 vm = (FULLC >> (EPC - hi)) & ~((1u << lo) - 1u);
    m &= vm;
    const u64 g = g0 + (u64)c * EPC;
    if (vm == FULLC) {
      if (SZ == 1)
        reinterpret_cast<u16*>(nwords)[g >> 4] = (u16)m;
      else
        reinterpret_cast<u8*>(nwords)[g >> 3] = (u8)m;
    } else if (m) {
      atomicOr(reinterpret_cast<u32*>(nwords) + (g >> 5), m << (u32)(g & 31));
    }
    if (g >= bnd) chi += __popc(m); else clo += __popc(m);
  }
  u32 x = clo | (chi << 16);  // <= 4096 each
#pragma unroll
  for (int d = 16; d; d >>= 1) x += __shfl_xor_sync(FULLM, x, d);
  if (lane == 0 && (x & 0xffffu)) atomicAdd(l1counts + (dst >> 16), x & 0xffffu);
  if (lane == 1 && (x >> 16)) atomicAdd(l1counts + (bnd >> 16), x >> 16);
}

// MODE 0: next level counted per tile and per L1 block (tile mode); 1 (kBlk):
// this and the next level in block mode -- next-level ones counted per run in
// pass 1 (the staged runs are re-read only for a run crossing an L1 block);
// 2 (kPair): the next level is the last, its bits written from the staging.
template <typename TIn, typename TC, bool kLut, int MODE>
__global__ void __launch_bounds__(W_NT, WS<TIn>::BYTES > 2048 ? W_MINB4 : W_MINB)  // one 4 KiB ring slot per warp: 6 CTAs (80 registers; measured faster than 4 CTAs with two slots)
    wlevel_kernel(const __grid_constant__ WLevelParams P) {
  constexpr bool kPair = MODE == 2, kBlk = MODE == 1;
  using S = WS<TIn>;
  using F = WF<TIn, TC>;
  constexpr int TILE = S::TILE, TPL1 = S::TPL1;
  constexpr int CR = F::CR, RE = F::RE, ROWS = F::ROWS, WR = F::WR, LW = F::LW, LB = F::LB,
                RB = F::RB, TB = S::BYTES;
  constexpr u32 SZ = sizeof(TC);
  constexpr int NTILE_LOG = WS<TC>::LOG;  // next level's tile (its input = codes)
  extern __shared__ __align__(128) u8 smem_raw[];
  u16* slut = reinterpret_cast<u16*>(smem_raw);  // 256 entries (u8 text + LUT)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  u8* wbase = smem_raw + 512 + warp * F::WARP_SMEM;
  u8* ring = wbase;
  u8* stage0 = wbase + W_RING * TB;
  u64* mbar = reinterpret_cast<u64*>(wbase + W_RING * TB + W_NSTAGE * F::STAGE);

  // the scatter's copy of the LUT: code-sized entries at a static address, so
  // a lookup is one LDS [raw + imm] after one PRMT extracting the byte
  __shared__ TC slutc[kLut && sizeof(TIn) == 1 ? 256 : 1];
  if (kLut && sizeof(TIn) == 1) {
    for (int i = tid; i < 256; i += W_NT) {
      slut[i] = P.lut[i];
      slutc[i] = (TC)P.lut[i];
    }
    __syncthreads();
  }
  // u8 codes: sheep-and-goats PRMT selectors per 8-bit lane-row mask (zeros'
  // bytes first, then ones', each in order; nibble i = source byte of output i)
  constexpr bool kSag = sizeof(TC) == 1 && sizeof(TIn) == 1 && !kLut && WT_SAG;
  __shared__ uint2 ssag[kSag ? 256 : 1];
  if (kSag) {
    for (int i = tid; i < 256; i += W_NT) {
      u32 sel = 0, n = 0;
      for (u32 pass = 0; pass < 2; ++pass)
        for (u32 j = 0; j < 8; ++j)
          if ((((u32)i >> j) & 1u) == pass) sel |= j << (4 * n++);
      ssag[i] = make_uint2(sel & 0xffffu, sel >> 16);
    }
    __syncthreads();
  }
  const u32 ntiles = (u32)((P.m + TILE - 1) / TILE);
  const u32 nfull = (u32)(P.m / TILE);
  const u32 gw = blockIdx.x * W_WARPS + warp, nw = gridDim.x * W_WARPS;
  // kBlk at a LUT level 0: per-lane SIMD copies of the next bit's thresholds
  // (a threshold above every symbol value never compares true: enable mask 0)
  u32 nt[3] = {0, 0, 0}, ne[3] = {0, 0, 0};
  if (kBlk && kLut) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const u32 tv = P.nthr[i];
      const bool on = tv <= (sizeof(TIn) == 1 ? 0xffu : 0xffffu);
      nt[i] = on ? tv * (sizeof(TIn) == 1 ? 0x01010101u : 0x00010001u) : 0u;
      ne[i] = on ? 0xffffffffu : 0u;
    }
  }
  // Block mode (level 0 of a large u8 text, tile_counts == nullptr): a warp
  // takes whole L1 blocks and walks their tiles in order, so P1 is the L1
  // entry plus the warp's own running count -- no per-tile counting pass.
  const bool blockm = P.tile_counts == nullptr;
  auto tile_at = [&](u32 i) -> u32 {
    return blockm ? (gw + (i / TPL1) * nw) * TPL1 + i % TPL1 : gw + i * nw;
  };
  u32 run = 0;  // block mode: ones of the block's tiles before this one
  const bool scatter = kPair || P.out != nullptr;
  const u8* in = reinterpret_cast<const u8*>(P.in);

  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < W_RING; ++i) w_mbar_init(&mbar[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int i = 0; i < W_RING; ++i) {
      const u32 t = tile_at(i);
      if (t < nfull) w_load_tile(ring + i * TB, in + (u64)t * TB, TB, &mbar[i]);
    }
  }
  __syncwarp();

  u32 it = 0;
  for (u32 t = tile_at(0); t < ntiles; t = tile_at(++it)) {
    const u32 slot = it % W_RING;
    const u32 tnext = tile_at(it + W_RING);  // the tile this ring slot streams next
    if (blockm && t % TPL1 == 0) run = 0;
    if (t >= nfull) {  // the partial last tile
      general_tile<TIn, TC, kLut, MODE>(P, t, slut, blockm ? __ldg(P.l1 + t / TPL1) + run : ~0ull);
      if (scatter && lane == 0) w_bulk_commit();  // keep one bulk group per tile
      continue;
    }
    const u8* tin = ring + slot * TB;
    // ---- P1 (loads go out before the tile data is waited on) -----------------
    const u32 b = t / TPL1;
    const u32 tb = t - b * TPL1;
    u32 pre = 0;
    if (!blockm) {
#pragma unroll
      for (int r = 0; r < (TPL1 + 31) / 32; ++r) {
        const u32 j = r * 32 + lane;
        if (j < tb) pre += __ldg(P.tile_counts + b * TPL1 + j);
      }
    }
    const u64 l1v = __ldg(P.l1 + b);
    const u64 t0 = (u64)t * TILE;
    w_mbar_wait(&mbar[slot], (it / W_RING) & 1);

    // ---- single node? (first and last element of the tile) -------------------
    u32 fcode, lcode;
    {
      const u32 f = sizeof(TIn) == 1 ? (u32)tin[0] : (u32)reinterpret_cast<const u16*>(tin)[0];
      const u32 l = sizeof(TIn) == 1 ? (u32)tin[TILE - 1]
                                     : (u32)reinterpret_cast<const u16*>(tin)[TILE - 1];
      fcode = !kLut ? f : sizeof(TIn) == 1 ? (u32)slut[f] : (u32)__ldg(P.lut + f);
      lcode = !kLut ? l : sizeof(TIn) == 1 ? (u32)slut[l] : (u32)__ldg(P.lut + l);
    }
    const u32 fkey = fcode >> P.shift_key, lkey = lcode >> P.shift_key;
    // two nodes (a node boundary inside the tile -- at deep levels of large
    // alphabets most straddling tiles): keys are non-decreasing in the tile, so
    // `split` = first element of the second node, found by binary search
    u32 split = TILE;
    // (u16 codes only: at u8 codes node boundaries inside a tile are rare and
    // the extra code costs the single-node path registers)
    constexpr bool kTwoSeg = sizeof(TC) == 2;
    if (scatter && fkey != lkey && !kTwoSeg) split = 0;
    if (kTwoSeg && scatter && fkey != lkey) {
      u32 lo = 1, hi = TILE - 1;  // key(0) = fkey, key(TILE-1) = lkey
      while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        const u32 r = sizeof(TIn) == 1 ? (u32)tin[mid] : (u32)reinterpret_cast<const u16*>(tin)[mid];
        const u32 c = !kLut ? r : sizeof(TIn) == 1 ? (u32)slut[r] : (u32)__ldg(P.lut + r);
        if ((c >> P.shift_key) == fkey) lo = mid + 1; else hi = mid;
      }
      split = lo;
      const u32 r = sizeof(TIn) == 1 ? (u32)tin[split] : (u32)reinterpret_cast<const u16*>(tin)[split];
      const u32 c = !kLut ? r : sizeof(TIn) == 1 ? (u32)slut[r] : (u32)__ldg(P.lut + r);
      if ((c >> P.shift_key) != lkey) split = 0;  // three or more nodes
    }
    if (scatter && split == 0) {
      __syncwarp();
      if (lane == 0 && tnext < nfull)
        w_load_tile(ring + slot * TB, in + (u64)tnext * TB, TB, &mbar[slot]);
      run += general_tile<TIn, TC, kLut, MODE>(P, t, slut, blockm ? l1v + run : ~0ull);
      if (lane == 0) w_bulk_commit();  // keep one bulk group per tile
      continue;
    }
    if (!blockm) {
#pragma unroll
      for (int d = 16; d; d >>= 1) pre += __shfl_xor_sync(FULLM, pre, d);
    }
    const u64 P1 = l1v + (blockm ? run : pre);

    // ---- pass 1: masks and counts per row ------------------------------------
    u32 mrow[ROWS];
    u32 zc = 0, oc = 0;  // kBlk: next-level ones bound for the zeros / ones run
    u32 accT = 0, accO = 0;  // kBlk, codes: per-byte (halfword) next-level ones, of them in the ones run
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      u32 v[LW];
      wrow_load<LW>(tin + r * RB + lane * LB, v);
      u32 nm = 0;  // kBlk: the next level's bit of each element
      if (kLut) {
        // level 0 through the LUT: the level bit is the TOP code bit, i.e.
        // `symbol >= thr` (codes are monotone in symbols) -- a SIMD compare
        // of the raw symbols, no table lookups in this pass; the next bit is
        // the parity of (symbol >= nthr[i]) over the three thresholds of the
        // codes' top two bits
        if (sizeof(TIn) == 1) {
          const u32 t4 = P.thr * 0x01010101u;
          const u32 y0 = __vcmpgeu4(v[0], t4) & 0x01010101u, y1 = __vcmpgeu4(v[LW - 1], t4) & 0x01010101u;
          mrow[r] = P.thr > 0xffu ? 0u : ((y1 * 16u + y0) * 0x01020408u) >> 24;
          if (kBlk) {
            u32 y[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const u32 x = v[i % LW];
              y[i] = ((__vcmpgeu4(x, nt[0]) & ne[0]) ^ (__vcmpgeu4(x, nt[1]) & ne[1]) ^
                      (__vcmpgeu4(x, nt[2]) & ne[2])) & 0x01010101u;
            }
            nm = ((y[1] * 16u + y[0]) * 0x01020408u) >> 24;
          }
        } else {
          const u32 t2 = P.thr * 0x00010001u;
          u32 mm = 0;
#pragma unroll
          for (int i = 0; i + 1 < LW; i += 2) {
            const u32 y0 = __vcmpgeu2(v[i], t2) & 0x00010001u, y1 = __vcmpgeu2(v[i + 1], t2) & 0x00010001u;
            const u32 z = y1 * 4u + y0;  // bits 0, 16, 2, 18 -> elements 0, 1, 2, 3
            mm |= ((z | (z >> 15)) & 0xfu) << (2 * i);
            if (kBlk) {
              u32 y[2];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const u32 x = v[i + h];
                y[h] = ((__vcmpgeu2(x, nt[0]) & ne[0]) ^ (__vcmpgeu2(x, nt[1]) & ne[1]) ^
                        (__vcmpgeu2(x, nt[2]) & ne[2])) & 0x00010001u;
              }
              const u32 zn = y[1] * 4u + y[0];
              nm |= ((zn | (zn >> 15)) & 0xfu) << (2 * i);
            }
          }
          mrow[r] = P.thr > 0xffffu ? 0u : mm;
        }
      } else {
        u32 cw[WR];
        wrow_codes<TIn, TC, kLut>(v, slut, P.lut, cw);
        mrow[r] = wmask<TC, WR>(cw, P.shift_bit);
        if (kBlk) {  // SIMD byte / halfword counters (<= 32 per field over the tile)
          const u32 lm = sizeof(TC) == 1 ? 0x01010101u : 0x00010001u;
#pragma unroll
          for (int i = 0; i < WR; ++i) {
            const u32 y = (cw[i] >> P.shift_bit) & lm, nb = (cw[i] >> (P.shift_bit - 1)) & lm;
            accT += nb;
            accO += nb & y;
          }
        }
      }
      if (kBlk && kLut) {
        zc += __popc(nm & ~mrow[r] & 0xffu);
        oc += __popc(nm & mrow[r]);
      }
    }
    if (kBlk && !kLut) {  // fold the SIMD counters
      const u32 t = sizeof(TC) == 1 ? (accT * 0x01010101u) >> 24 : (accT & 0xffffu) + (accT >> 16);
      oc = sizeof(TC) == 1 ? (accO * 0x01010101u) >> 24 : (accO & 0xffffu) + (accO >> 16);
      zc = t - oc;
    }
    u32 r1[ROWS], rtot[ROWS];
    // four rows per warp scan, 8-bit fields: a lane-row holds <= 8 ones, so
    // every lane's inclusive field stays <= 248 except lane 31's (<= 256,
    // which may carry): the exclusive prefixes are read from lane - 1 and the
    // row totals are lane 31's exclusive prefix plus its own counts
    static_assert(ROWS % 4 == 0, "rows come in fours");
#ifndef WT_SCAN4
#define WT_SCAN4 1
#endif
#if WT_SCAN4
#pragma unroll
    for (int r = 0; r < ROWS; r += 4) {
      const u32 x = (u32)__popc(mrow[r]) | ((u32)__popc(mrow[r + 1]) << 8) |
                    ((u32)__popc(mrow[r + 2]) << 16) | ((u32)__popc(mrow[r + 3]) << 24);
      u32 inc = x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 y = __shfl_up_sync(FULLM, inc, d);
        if (lane >= d) inc += y;
      }
      u32 ex = __shfl_up_sync(FULLM, inc, 1);
      if (lane == 0) ex = 0;
      const u32 ex31 = __shfl_sync(FULLM, ex, 31), x31 = __shfl_sync(FULLM, x, 31);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        r1[r + i] = (ex >> (8 * i)) & 0xffu;
        rtot[r + i] = ((ex31 >> (8 * i)) & 0xffu) + ((x31 >> (8 * i)) & 0xffu);
      }
    }
#else
#pragma unroll
    for (int r = 0; r < ROWS; r += 2) {
      const u32 x = (u32)__popc(mrow[r]) | ((u32)__popc(mrow[r + 1]) << 16);
      u32 inc = x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 y = __shfl_up_sync(FULLM, inc, d);
        if (lane >= d) inc += y;
      }
      const u32 tot = __shfl_sync(FULLM, inc, 31);
      const u32 ex = inc - x;
      r1[r] = ex & 0xffffu;
      r1[r + 1] = ex >> 16;
      rtot[r] = tot & 0xffffu;
      rtot[r + 1] = tot >> 16;
    }
#endif
    u32 tile_ones = 0;
    u32 rstart[ROWS];  // ones of the tile before row r (warp-uniform)
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      rstart[r] = tile_ones;
      r1[r] += tile_ones;
      tile_ones += rtot[r];
    }
    run += tile_ones;

    // ---- bit-vector words: each lane-row mask is CR bits at t0 + r*RE + lane*CR
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
      reinterpret_cast<u8*>(P.words)[(t0 >> 3) + r * (RE / 8) + lane] = (u8)mrow[r];

    // L2 entries and samples here, or by dir_kernel after the launch (skip_dir)
    if (!P.skip_dir) {
    // ---- L2 entries: blocks start at lane-row boundaries (l2_bits >= 64) ------
    if ((1u << P.l2_log) >= (u32)RE) {  // at most one per row: lane r handles row r
      u32 rs = 0;  // ones before row `lane`
#pragma unroll
      for (int r = 0; r < ROWS; ++r) rs = lane == r ? rstart[r] : rs;
      const u64 g = t0 + (u64)lane * RE;
      if (lane < ROWS && (((u32)g) & ((1u << P.l2_log) - 1)) == 0)
        P.l2[g >> P.l2_log] = (u16)(P1 + rs - l1v);
    } else if (((lane * CR) & ((1u << P.l2_log) - 1)) == 0) {  // same lanes in every row
#pragma unroll
      for (int r = 0; r < ROWS; ++r)
        P.l2[(t0 + r * RE + lane * CR) >> P.l2_log] = (u16)(P1 + r1[r] - l1v);
    }

    // ---- select samples (rankselect.py:509-532) --------------------------------
#pragma unroll
    for (int kind = 0; kind < 2; ++kind) {
      const bool ones = kind == 0;
      const u64 base = ones ? P1 : t0 - P1;
      const u32 cnt = ones ? tile_ones : TILE - tile_ones;
      u64* out = ones ? P.ones : P.zeros;
      const u64 cap = ones ? P.ones_cap : P.zeros_cap;
      const u64 q0 = wnext_multiple(base, P.rate, P.rate_log);
      if (q0 > base + cnt) continue;
      for (u64 qo = q0; qo <= base + cnt; qo += P.rate) {
        const u32 tt = (u32)(qo - base);  // 1-based ordinal inside the tile
        // the row holding ordinal tt (warp-uniform), then its lane (ballot)
        u32 rr = 0;
#pragma unroll
        for (int r = 1; r < ROWS; ++r) {
          const u32 before = ones ? rstart[r] : (u32)(r * RE) - rstart[r];
          rr = before < tt ? (u32)r : rr;
        }
        u32 r1s = r1[0], ms = mrow[0];
#pragma unroll
        for (int r = 1; r < ROWS; ++r) {
          r1s = rr == (u32)r ? r1[r] : r1s;
          ms = rr == (u32)r ? mrow[r] : ms;
        }
        const u32 pre_l = ones ? r1s : rr * RE + lane * CR - r1s;
        const u32 mk = ones ? ms : (~ms & ((1u << CR) - 1u));
        const bool own = pre_l < tt && tt <= pre_l + __popc(mk);
        if (own) {
          const u64 sidx = (P.rate_log >= 0 ? (qo >> P.rate_log) : qo / P.rate) - 1;
          if (sidx < cap) out[sidx] = t0 + rr * RE + lane * CR + select_in_word32(mk, tt - pre_l);
        }
      }
    }

    }  // !skip_dir

    if (scatter) {
      // ---- pass 2: stable partition into the staged zeros / ones runs ----------
      u8* stage = stage0 + (W_NSTAGE == 2 ? (it & 1) : 0) * F::STAGE;
      const u32 sbase = smem_addr(stage);
      if (it >= (u32)W_NSTAGE) {
        if (lane == 0) {  // the bulk store that last read this buffer
          if (W_NSTAGE == 2) w_bulk_wait_read1(); else w_bulk_wait_read0();
        }
        __syncwarp();
      }
      const u32 tile_zeros = TILE - tile_ones;
      // ones before `split` (segment A = [0, split), B = [split, TILE))
      u32 onesA = tile_ones;
      if (kTwoSeg && split < (u32)TILE) {
        const u32 rs = split / RE, ls = (split % RE) / CR, js = split % CR;
        u32 v = 0;
#pragma unroll
        for (int r = 0; r < ROWS; ++r)
          if ((u32)r == rs) v = r1[r] + __popc(mrow[r] & ((1u << js) - 1u));
        onesA = __shfl_sync(FULLM, v, ls);
      }
      const u32 zerosA = split - onesA;
      const NodeEnt* ne = P.nodes + fkey;
      const u64 zdst = (u64)__ldg(&ne->zero_base) + (t0 - P1);
      const u64 odst = (u64)__ldg(&ne->one_base) + P1;
      const u32 zoff = (u32)((zdst * SZ) & 15);
      const u32 ooff = ((zoff + zerosA * SZ + 15) & ~15u) + (u32)((odst * SZ) & 15);
      const bool zlive = zerosA && zdst < P.m_next;
      const bool olive = onesA && odst < P.m_next;
      // segment B runs (empty when the tile lies in one node)
      const u32 onesB = tile_ones - onesA, zerosB = tile_zeros - zerosA;
      u64 zdstB = 0, odstB = 0;
      u32 zoffB = 0, ooffB = 0;
      if (kTwoSeg && split < (u32)TILE) {
        const NodeEnt* nb = P.nodes + lkey;
        zdstB = (u64)__ldg(&nb->zero_base) + (t0 + split - P1 - onesA);
        odstB = (u64)__ldg(&nb->one_base) + P1 + onesA;
        zoffB = ((ooff + onesA * SZ + 15) & ~15u) + (u32)((zdstB * SZ) & 15);
        ooffB = ((zoffB + zerosB * SZ + 15) & ~15u) + (u32)((odstB * SZ) & 15);
      }
      const bool zliveB = zerosB && zdstB < P.m_next;
      const bool oliveB = onesB && odstB < P.m_next;
      if (!kTwoSeg || split == (u32)TILE) {  // one node (the common case): two runs
        // loads stay ahead of the stores in program order (ptxas keeps shared
        // loads behind earlier shared stores it cannot disambiguate): the next
        // lane-row and this row's LUT lookups are issued before the stores
        // (u8 input only: at u16 the extra row of registers spills)
        constexpr bool kPre = sizeof(TIn) == 1;
        u32 vn[LW];
        if (kPre) wrow_load<LW>(tin + lane * LB, vn);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          u32 v[LW];
          if (kPre) {
#pragma unroll
            for (int i = 0; i < LW; ++i) v[i] = vn[i];
            if (r + 1 < ROWS) wrow_load<LW>(tin + (r + 1) * RB + lane * LB, vn);
          } else {
            wrow_load<LW>(tin + r * RB + lane * LB, v);
          }
          u32 cw[WR];
          if (!kLut) wrow_codes<TIn, TC, kLut>(v, slut, P.lut, cw);
          u32 lv[CR];
          if (kLut) {  // map each raw symbol
#pragma unroll
            for (int j = 0; j < CR; ++j)
              lv[j] = sizeof(TIn) == 1 ? (u32)slutc[__byte_perm(v[j >> 2], 0u, 0x4440u + (j & 3))]
                                       : (u32)__ldg(P.lut + ((v[j >> 1] >> ((j & 1) * 16)) & 0xffffu));
          }
          const u32 m = mrow[r];
          u32 oa = sbase + ooff + r1[r] * SZ;
          u32 za = sbase + zoff + ((u32)(r * RE + lane * CR) - r1[r]) * SZ;
          if (kSag) {
            // u8 codes: one sheep-and-goats byte permutation puts the row's
            // zeros first and its ones after them (both in order); output byte
            // k then goes to za + k (k < zeros) or oa - zeros + k -- no cursor
            // updates, one store per element
            const uint2 sg = ssag[m];
            const u32 p0 = __byte_perm(cw[0], cw[WR - 1], sg.x), p1 = __byte_perm(cw[0], cw[WR - 1], sg.y);
            const u32 nz = 8u - (u32)__popc(m);
            const u32 bo = oa - nz;
            const u32 therm = (1u << nz) - 1u;  // bit k: output byte k is a zero's
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const u32 val = (k < 4 ? p0 : p1) >> ((k & 3) * 8);
              st_shared<TC>(((therm >> k) & 1u ? za : bo) + k, val);
            }
          } else {
#pragma unroll
          for (int j = 0; j < CR; ++j) {
            // st.shared.u8/u16 keep the low bits: no masking of the element
            const u32 val = kLut ? lv[j]
                                 : sizeof(TC) == 1 ? cw[j >> 2] >> ((j & 3) * 8) : cw[j >> 1] >> ((j & 1) * 16);
            if (m & (1u << j)) {
              st_shared<TC>(oa, val);
              oa += SZ;
            } else {
              st_shared<TC>(za, val);
              za += SZ;
            }
          }
          }
        }
      } else {  // two nodes: four runs
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        u32 v[LW];
        wrow_load<LW>(tin + r * RB + lane * LB, v);
        u32 cw[WR];
        if (!kLut) wrow_codes<TIn, TC, kLut>(v, slut, P.lut, cw);
        const u32 m = mrow[r];
        const u32 e0 = (u32)(r * RE + lane * CR);
        const bool inB = e0 >= split;  // whole lane-row in segment B
        u32 oa = inB ? sbase + ooffB + (r1[r] - onesA) * SZ : sbase + ooff + r1[r] * SZ;
        u32 za = inB ? sbase + zoffB + ((e0 - split) - (r1[r] - onesA)) * SZ
                     : sbase + zoff + (e0 - r1[r]) * SZ;
        const u32 jsw = (!inB && e0 + CR > split) ? split - e0 : (u32)CR;  // switch to B inside
        auto element = [&](int j) {
          // st.shared.u8/u16 keep the low bits: no masking of the element
          u32 val;
          if (kLut) {  // map each raw symbol as it is stored
            val = sizeof(TIn) == 1 ? (u32)slutc[__byte_perm(v[j >> 2], 0u, 0x4440u + (j & 3))]
                                   : (u32)__ldg(P.lut + ((v[j >> 1] >> ((j & 1) * 16)) & 0xffffu));
          } else {
            val = sizeof(TC) == 1 ? cw[j >> 2] >> ((j & 3) * 8) : cw[j >> 1] >> ((j & 1) * 16);
          }
          if (m & (1u << j)) {
            st_shared<TC>(oa, val);
            oa += SZ;
          } else {
            st_shared<TC>(za, val);
            za += SZ;
          }
        };
        if (jsw == (u32)CR) {
#pragma unroll
          for (int j = 0; j < CR; ++j) element(j);
        } else {  // the one lane-row holding the node boundary
#pragma unroll
          for (int j = 0; j < CR; ++j) {
            if ((u32)j == jsw) {
              oa = sbase + ooffB;
              za = sbase + zoffB;
            }
            element(j);
          }
        }
      }
      }
      w_fence_proxy();
      __syncwarp();
      // the input slot is free: the tile three ahead streams into it
      if (lane == 0 && tnext < nfull)
        w_load_tile(ring + slot * TB, in + (u64)tnext * TB, TB, &mbar[slot]);
      if (kPair) {
        // the last level's bits straight from the staged runs
        const u32 sh1 = P.shift_bit - 1;
        if (zlive) wpair_bits<TC>(stage, zerosA, zoff, zdst, sh1, P.next_words, P.next_l1_counts, lane);
        if (olive) wpair_bits<TC>(stage, onesA, ooff, odst, sh1, P.next_words, P.next_l1_counts, lane);
        if (kTwoSeg && split < (u32)TILE) {
          if (zliveB) wpair_bits<TC>(stage, zerosB, zoffB, zdstB, sh1, P.next_words, P.next_l1_counts, lane);
          if (oliveB) wpair_bits<TC>(stage, onesB, ooffB, odstB, sh1, P.next_words, P.next_l1_counts, lane);
        }
        continue;
      }
      u8* gout = reinterpret_cast<u8*>(P.out);
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        if (rr >= 2 && (!kTwoSeg || split == (u32)TILE)) break;
        const bool live = rr == 0 ? zlive : rr == 1 ? olive : rr == 2 ? zliveB : oliveB;
        if (!live) continue;
        const u32 cnt = rr == 0 ? zerosA : rr == 1 ? onesA : rr == 2 ? zerosB : onesB;
        const u64 dst = rr == 0 ? zdst : rr == 1 ? odst : rr == 2 ? zdstB : odstB;
        const u32 soff = rr == 0 ? zoff : rr == 1 ? ooff : rr == 2 ? zoffB : ooffB;
        const u32 bytes = cnt * SZ;
        const u64 db = dst * SZ;
        u32 head = (u32)((16 - (db & 15)) & 15);
        if (head > bytes) head = bytes;
        const u32 body = (bytes - head) & ~15u;
        const u32 tail = bytes - head - body;
        if (lane < (int)head) gout[db + lane] = stage[soff + lane];
        if (lane >= 16 && lane < 16 + (int)tail) {
          const u32 o2 = head + body + (lane - 16);
          gout[db + o2] = stage[soff + o2];
        }
        if (lane == 0 && body) w_bulk_s2g(gout + db + head, stage + soff + head, body);
      }
      if (kBlk) {
        // next level's ones per L1 block: the pass-1 counts of each run, unless
        // the run crosses a block boundary (or the tile holds two nodes: its
        // pass-1 counts are not split by node) -- then the staged runs
        const bool two = kTwoSeg && split < (u32)TILE;
        const bool zx = zlive && ((zdst & 0xffffu) + zerosA > 65536u);
        const bool ox = olive && ((odst & 0xffffu) + onesA > 65536u);
        if (two || zx || ox) {
          wcount_tile<TC, false>(stage, zlive ? zerosA : 0u, zoff, zdst, olive ? onesA : 0u, ooff, odst,
                                 P.shift_bit - 1, 16, P.next_l1_counts, nullptr, lane);
          if (two)
            wcount_tile<TC, false>(stage, zliveB ? zerosB : 0u, zoffB, zdstB, oliveB ? onesB : 0u, ooffB,
                                   odstB, P.shift_bit - 1, 16, P.next_l1_counts, nullptr, lane);
        } else {
          u32 x = zc | (oc << 16);  // <= 4096 each
#pragma unroll
          for (int d = 16; d; d >>= 1) x += __shfl_xor_sync(FULLM, x, d);
          if (lane == 0 && zlive && (x & 0xffffu)) atomicAdd(P.next_l1_counts + (zdst >> 16), x & 0xffffu);
          if (lane == 1 && olive && (x >> 16)) atomicAdd(P.next_l1_counts + (odst >> 16), x >> 16);
        }
      } else {
      // next level's ones of both runs per next-level tile (<= 3 per run) and
      // L1 block, in one pass over the staged tile
      wcount_tile<TC, (WS<TIn>::TILE > WS<TC>::TILE)>(stage, zlive ? zerosA : 0u, zoff, zdst, olive ? onesA : 0u, ooff, odst,
                      P.shift_bit - 1, NTILE_LOG, P.next_tile_counts, P.next_l1_counts, lane);
      if (kTwoSeg && split < (u32)TILE)
        wcount_tile<TC, (WS<TIn>::TILE > WS<TC>::TILE)>(stage, zliveB ? zerosB : 0u, zoffB, zdstB, oliveB ? onesB : 0u, ooffB, odstB,
                        P.shift_bit - 1, NTILE_LOG, P.next_tile_counts, P.next_l1_counts, lane);
      }
      if (lane == 0) w_bulk_commit();  // one bulk group per scattering fast tile
    } else {
      __syncwarp();
      if (lane == 0 && tnext < nfull)
        w_load_tile(ring + slot * TB, in + (u64)tnext * TB, TB, &mbar[slot]);
    }
  }
  if (scatter && lane == 0) w_bulk_wait_all();
}

// ---------------------------------------------------------------------------
// the last level (nothing to partition): bits, L2 entries and samples only.
// Lane i owns input bytes [64i, 64i + 64) of a warp tile, so its mask is one
// contiguous 64-bit (u8 codes) / 32-bit (u16 codes) piece of the bit-vector
// and a single warp scan gives every L2 prefix.
// ---------------------------------------------------------------------------
template <typename TIn, typename TC, bool kLut>
__global__ void __launch_bounds__(256) wlast_kernel(const __grid_constant__ WLevelParams P) {
  using S = WS<TIn>;
  constexpr int TILE = S::TILE, TPL1 = S::TPL1;
  constexpr int CH = 16 / (int)sizeof(TIn);   // elements per 16-byte chunk
  constexpr int K = S::K;                     // 16-byte chunks per lane
  constexpr int E = K * CH;                   // elements per lane: 64
  constexpr int WPC = CH * (int)sizeof(TC) / 4;
  __shared__ u16 slut[kLut && sizeof(TIn) == 1 ? 256 : 1];
  const int tid = threadIdx.x, lane = tid & 31;
  if (kLut && sizeof(TIn) == 1) {
    for (int i = tid; i < 256; i += 256) slut[i] = P.lut[i];
    __syncthreads();
  }
  const u32 ntiles = (u32)((P.m + TILE - 1) / TILE);
  const u32 nfull = (u32)(P.m / TILE);
  const u32 nw = gridDim.x * 8;
  const u8* in = reinterpret_cast<const u8*>(P.in);
  const u64 l2m = (1ull << P.l2_log) - 1;
  // full tiles stream into a per-warp two-slot shared ring by TMA (bulk copy
  // + mbarrier); lanes then read their 128-byte slice with a per-lane chunk
  // rotation, so a warp's 16-byte reads spread over the banks
  constexpr int TB = S::BYTES;
  extern __shared__ __align__(128) u8 wl_smem[];
  u8* ring = wl_smem + (tid >> 5) * (2 * TB + 16);
  u64* mbar = reinterpret_cast<u64*>(ring + 2 * TB);
  const u32 gw = blockIdx.x * 8 + (tid >> 5);
  if (lane == 0) {
    w_mbar_init(&mbar[0]);
    w_mbar_init(&mbar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (u32 i = 0; i < 2; ++i)
      if (gw + i * nw < nfull) w_load_tile(ring + i * TB, in + (u64)(gw + i * nw) * TB, TB, &mbar[i]);
  }
  __syncwarp();
  u32 it = 0;
  for (u32 t = gw; t < ntiles; t += nw, ++it) {
    const u64 t0 = (u64)t * TILE;
    const u32 valid = (u32)min((u64)TILE, P.m - t0);
    // P1 loads first (independent of the data)
    const u32 b = t / TPL1, tb = t - b * TPL1;
    u32 pre = 0;
#pragma unroll
    for (int r = 0; r < (TPL1 + 31) / 32; ++r) {
      const u32 j = r * 32 + lane;
      if (j < tb) pre += __ldg(P.tile_counts + b * TPL1 + j);
    }
    const u64 l1v = __ldg(P.l1 + b);
    const u8* base = in + t0 * sizeof(TIn) + lane * (K * 16);
    const u32 e0 = (u32)lane * E;  // first element of this lane in the tile
    constexpr int NW = E / 64;     // bit-vector words per lane (1 | 2)
    u64 m[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) m[w] = 0;
    if (t < nfull) {  // full tile from the ring
      const u32 slot = it & 1u;
      w_mbar_wait(&mbar[slot], (it >> 1) & 1u);
      const u8* src = ring + slot * TB + lane * (K * 16);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const u32 c = ((u32)k + (u32)lane) % (u32)K;  // rotated chunk: banks spread
        const uint4 q = *reinterpret_cast<const uint4*>(src + c * 16);
        u32 cw[WPC];
        wcodes<TIn, TC, kLut, WPC>(q, slut, P.lut, cw);
        const u64 mk = (u64)wmask<TC, WPC>(cw, P.shift_bit);
        const u32 bit = c * CH;  // this chunk's first bit in the lane's slice
#pragma unroll
        for (int w = 0; w < NW; ++w)
          m[w] |= (bit >> 6) == (u32)w ? mk << (bit & 63) : 0ull;
      }
      __syncwarp();
      if (lane == 0 && t + 2 * nw < nfull)
        w_load_tile(ring + slot * TB, in + (u64)(t + 2 * nw) * TB, TB, &mbar[slot]);
    } else {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const u32 e = e0 + k * CH;
      uint4 q;
      if (e + CH <= valid) {
        q = __ldg(reinterpret_cast<const uint4*>(base + k * 16));
      } else {
        u32 w[4] = {0, 0, 0, 0};
        for (u32 bb = 0; bb < 16 && e * sizeof(TIn) + bb < valid * sizeof(TIn); ++bb)
          w[bb >> 2] |= (u32)base[k * 16 + bb] << (8 * (bb & 3));
        q = make_uint4(w[0], w[1], w[2], w[3]);
      }
      u32 cw[WPC];
      wcodes<TIn, TC, kLut, WPC>(q, slut, P.lut, cw);
      u32 mk = wmask<TC, WPC>(cw, P.shift_bit);
      if (e + CH > valid) mk &= e >= valid ? 0u : (1u << (valid - e)) - 1u;
      m[(k * CH) / 64] |= (u64)mk << ((k * CH) % 64);
    }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) pre += __shfl_xor_sync(FULLM, pre, d);
    const u64 P1 = l1v + pre;
    u32 wc[NW], c = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      wc[w] = __popcll(m[w]);
      c += wc[w];
    }
    u32 inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 y = __shfl_up_sync(FULLM, inc, d);
      if (lane >= d) inc += y;
    }
    const u32 tile_ones = __shfl_sync(FULLM, inc, 31);
    const u32 pl = inc - c;  // ones of the tile before this lane
    u32 before = pl;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const u32 ew = e0 + 64 * w;
      const u64 g = t0 + ew;
      if (ew < ((valid + 63u) & ~63u)) P.words[(g >> 6)] = m[w];
      if (ew < valid && (g & l2m) == 0) P.l2[g >> P.l2_log] = (u16)(P1 + before - l1v);
      before += wc[w];
    }
    // select samples (rankselect.py:509-532)
#pragma unroll
    for (int kind = 0; kind < 2; ++kind) {
      const bool ones = kind == 0;
      const u64 sb = ones ? P1 : t0 - P1;
      const u32 cnt = ones ? tile_ones : valid - tile_ones;
      const u64 q0 = wnext_multiple(sb, P.rate, P.rate_log);
      if (q0 > sb + cnt) continue;
      const u32 lvalid = e0 >= valid ? 0u : min((u32)E, valid - e0);
      const u32 lc = ones ? c : lvalid - c;
      const u32 lp = ones ? pl : e0 - pl;
      u64* out = ones ? P.ones : P.zeros;
      const u64 cap = ones ? P.ones_cap : P.zeros_cap;
      for (u64 qo = q0; qo <= sb + cnt; qo += P.rate) {
        u32 tt = (u32)(qo - sb);
        if (lp < tt && tt <= lp + lc) {
          tt -= lp;
          u32 pos = e0;
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const u32 ew = e0 + 64 * w;
            const u32 wv = ew >= valid ? 0u : min(64u, valid - ew);
            const u64 wm = ones ? m[w] : (~m[w] & (wv >= 64 ? ~0ull : ((1ull << wv) - 1)));
            const u32 pc = __popcll(wm);
            if (tt > 0 && tt <= pc) {
              pos = ew + select_in_word64(wm, tt);
              tt = 0;
            } else if (tt > 0) {
              tt -= pc;
            }
          }
          const u64 sidx = (P.rate_log >= 0 ? (qo >> P.rate_log) : qo / P.rate) - 1;
          if (sidx < cap) out[sidx] = t0 + pos;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Pair kernel: the last two levels in one pass (every code reaches the last
// level; WLevelParams::next_words).  Lane i owns the contiguous slice
// [E i, E i + E) of a warp tile (E = 128 u8 / 64 u16 elements), so its
// level-l mask is whole u64 words of that level's bit-vector (as in
// wlast_kernel), and its L2 entries / samples follow from one warp scan.
// The last level's bits are the next code bit of the tile's zeros-group and
// ones-group elements, each group in text order (S_{l+1} is the stable
// partition of S_l): every lane compacts its chunks' next-bit flags with
// PRMT selectors looked up by the 8-element mask (no byte scatter through
// shared memory), ORs each chunk's piece into the two group bit-strings in
// shared memory (its place = the lane's group prefix from the scan + the
// chunk's prefix inside the slice), and the warp writes the strings to the
// last level at the groups' destinations (words inside a run stored, the
// run's first / last word OR-ed: neighbouring runs share them).
// Chunk k of a lane is read from slice chunk k ^ (lane & 7): the 16-byte
// reads of a warp spread over all banks.
// ---------------------------------------------------------------------------
template <typename TIn, typename TC>
__device__ __forceinline__ void wp_codes(uint4& q, const u16* slut, const u16* glut, bool lut,
                                         const WLevelParams& P) {
  // 16 input bytes -> 16 code bytes (u8 codes) or 8 code halfwords (u16)
  if (!lut) return;
  if (sizeof(TIn) == 1 && P.plut_shift != 0xffu) {  // <= 8 symbols: a register table
    auto map4 = [&](u32 x) -> u32 {
      const u32 y = (x >> P.plut_shift) & 0x07070707u;  // 3-bit index per byte
      const u32 t = y | (y >> 4);                       // nibbles 0, 1 in byte 0; 2, 3 in byte 2
      return __byte_perm(P.plut_lo, P.plut_hi, __byte_perm(t, 0u, 0x4420u));
    };
    q = make_uint4(map4(q.x), map4(q.y), map4(q.z), map4(q.w));
  } else if (sizeof(TIn) == 1) {  // u8 text, u8 codes (L = 2 here)
    auto map4 = [&](u32 x) -> u32 {
      return (u32)slut[x & 0xffu] | ((u32)slut[(x >> 8) & 0xffu] << 8) |
             ((u32)slut[(x >> 16) & 0xffu] << 16) | ((u32)slut[x >> 24] << 24);
    };
    q = make_uint4(map4(q.x), map4(q.y), map4(q.z), map4(q.w));
  } else {
    auto g = [&](u32 x) -> u32 { return (u32)__ldg(glut + x); };
    if (sizeof(TC) == 1) {  // u16 text, u8 codes: 8 codes in the low 8 bytes
      auto map4 = [&](u32 x, u32 y) -> u32 {
        return g(x & 0xffffu) | (g(x >> 16) << 8) | (g(y & 0xffffu) << 16) | (g(y >> 16) << 24);
      };
      q = make_uint4(map4(q.x, q.y), map4(q.z, q.w), 0u, 0u);
    } else {
      auto map2 = [&](u32 x) -> u32 { return g(x & 0xffffu) | (g(x >> 16) << 16); };
      q = make_uint4(map2(q.x), map2(q.y), map2(q.z), map2(q.w));
    }
  }
}

// 8-element flag bytes (bit 0 of each byte = bit `sh` of the element's code)
// of step s of a code chunk: u8 codes 16 per chunk, u16 codes 8 per chunk
template <typename TC>
__device__ __forceinline__ void wp_flags(const uint4& q, int s, u32 sh, u32& f0, u32& f1) {
  if (sizeof(TC) == 1) {
    const u32 a = s ? q.z : q.x, b = s ? q.w : q.y;
    f0 = (a >> sh) & 0x01010101u;
    f1 = (b >> sh) & 0x01010101u;
  } else {
    const u32 a = (q.x >> sh) & 0x00010001u, b = (q.y >> sh) & 0x00010001u;
    const u32 c = (q.z >> sh) & 0x00010001u, d = (q.w >> sh) & 0x00010001u;
    f0 = __byte_perm(a, b, 0x6420);
    f1 = __byte_perm(c, d, 0x6420);
  }
}

// bit 0 of 8 flag bytes (elements 0..3 in f0, 4..7 in f1) -> 8-bit mask
__device__ __forceinline__ u32 wp_gather(u32 f0, u32 f1) {
  return (((f1 * 16u + f0) * 0x01020408u) >> 24) & 0xffu;
}

#ifndef WP_MINB
#define WP_MINB 3
#endif
template <typename TIn, typename TC, bool kLut>
__global__ void __launch_bounds__(256, WP_MINB) wpair_kernel(const __grid_constant__ WLevelParams P) {
  using S = WS<TIn>;
  constexpr int TILE = S::TILE, TPL1 = S::TPL1, TB = S::BYTES;
  constexpr int K = S::K;                    // 16-byte chunks per lane (8)
  constexpr int CE = TILE / 32 / K;          // elements per chunk (16 | 8)
  constexpr int E = K * CE;                  // elements per lane (128 | 64)
  constexpr int NW = E / 64;                 // level-l words per lane (2 | 1)
  constexpr int NS = CE / 8;                 // 8-element steps per chunk (2 | 1)
  constexpr int GW = TILE / 32 + 4;          // words of one group string (+ alignment; 2 GW % 4 == 0)
  static_assert(K == 8, "chunk rotation assumes 8 chunks per lane");
  // sheep-and-goats PRMT selectors of an 8-element step: output bytes = the
  // bytes whose mask bit is 0, in order, then those whose bit is 1 (selector
  // nibble i = source byte of output byte i)
  __shared__ uint2 csel[256];
  __shared__ u16 slut[kLut && sizeof(TIn) == 1 ? 256 : 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    u32 sel = 0, n = 0;
    for (u32 pass = 0; pass < 2; ++pass)
      for (u32 j = 0; j < 8; ++j)
        if (((tid >> j) & 1) == pass) sel |= j << (4 * n++);
    csel[tid] = make_uint2(sel & 0xffffu, sel >> 16);
    if (kLut && sizeof(TIn) == 1) slut[tid] = P.lut[tid];
    __syncthreads();
  }
  const u32 ntiles = (u32)((P.m + TILE - 1) / TILE);
  const u32 nfull = (u32)(P.m / TILE);
  const u32 gw = blockIdx.x * 8 + warp, nw = gridDim.x * 8;
  const bool blockm = P.tile_counts == nullptr;
  auto tile_at = [&](u32 i) -> u32 {
    return blockm ? (gw + (i / TPL1) * nw) * TPL1 + i % TPL1 : gw + i * nw;
  };
  const u8* in = reinterpret_cast<const u8*>(P.in);
  const u64 l2m = (1ull << P.l2_log) - 1;
  const u32 sh = P.shift_bit, sh1 = P.shift_bit - 1;
  extern __shared__ __align__(128) u8 wp_smem[];
  u8* ring = wp_smem + warp * (2 * TB + 16 + 2 * GW * 4);
  u64* mbar = reinterpret_cast<u64*>(ring + 2 * TB);
  u32* gbuf = reinterpret_cast<u32*>(ring + 2 * TB + 16);  // [2][GW]
  if (lane == 0) {
    w_mbar_init(&mbar[0]);
    w_mbar_init(&mbar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (u32 i = 0; i < 2; ++i) {
      const u32 t = tile_at(i);
      if (t < nfull) w_load_tile(ring + i * TB, in + (u64)t * TB, TB, &mbar[i]);
    }
  }
  __syncwarp();
  u32 run = 0, it = 0;
  for (u32 t = tile_at(0); t < ntiles; t = tile_at(++it)) {
    const u32 slot = it & 1u;
    const u32 tnext = tile_at(it + 2);
    if (blockm && t % TPL1 == 0) run = 0;
    const u32 b = t / TPL1, tb = t - b * TPL1;
    const u64 l1v = __ldg(P.l1 + b);
    if (t >= nfull) {  // the partial last tile
      general_tile<TIn, TC, kLut, 2>(P, t, slut, blockm ? l1v + run : ~0ull);
      continue;
    }
    u32 pre = 0;
    if (!blockm) {
#pragma unroll
      for (int r = 0; r < (TPL1 + 31) / 32; ++r) {
        const u32 j = r * 32 + lane;
        if (j < tb) pre += __ldg(P.tile_counts + b * TPL1 + j);
      }
#pragma unroll
      for (int d = 16; d; d >>= 1) pre += __shfl_xor_sync(FULLM, pre, d);
    }
    const u64 P1 = l1v + (blockm ? run : pre);
    const u64 t0 = (u64)t * TILE;
    const u8* tin = ring + slot * TB;
    w_mbar_wait(&mbar[slot], (it >> 1) & 1u);
    // ---- one node? (first and last element of the tile) --------------------
    u32 fkey, lkey;
    {
      const u32 f = sizeof(TIn) == 1 ? (u32)tin[0] : (u32)reinterpret_cast<const u16*>(tin)[0];
      const u32 l = sizeof(TIn) == 1 ? (u32)tin[TILE - 1] : (u32)reinterpret_cast<const u16*>(tin)[TILE - 1];
      const u32 fc = !kLut ? f : sizeof(TIn) == 1 ? (u32)slut[f] : (u32)__ldg(P.lut + f);
      const u32 lc = !kLut ? l : sizeof(TIn) == 1 ? (u32)slut[l] : (u32)__ldg(P.lut + l);
      fkey = fc >> P.shift_key;
      lkey = lc >> P.shift_key;
    }
    if (fkey != lkey) {  // node boundary inside the tile: element by element
      __syncwarp();
      if (lane == 0 && tnext < nfull) w_load_tile(ring + slot * TB, in + (u64)tnext * TB, TB, &mbar[slot]);
      run += general_tile<TIn, TC, kLut, 2>(P, t, slut, blockm ? l1v + run : ~0ull);
      continue;
    }
    // ---- pass A: the lane's slice (chunk k = slice chunk k ^ (lane & 7)) ---
    uint4 q[K];
    u64 m[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) m[w] = 0;
    const u8* src = tin + lane * (K * 16);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const u32 c = (u32)k ^ ((u32)lane & 7u);
      q[k] = *reinterpret_cast<const uint4*>(src + c * 16);
      wp_codes<TIn, TC>(q[k], slut, P.lut, kLut, P);
      u32 mk = 0;
#pragma unroll
      for (int s2 = 0; s2 < NS; ++s2) {
        u32 f0, f1;
        wp_flags<TC>(q[k], s2, sh, f0, f1);
        mk |= wp_gather(f0, f1) << (8 * s2);
      }
      const u32 bit = c * CE;
#pragma unroll
      for (int w = 0; w < NW; ++w) m[w] |= (bit >> 6) == (u32)w ? (u64)mk << (bit & 63) : 0ull;
    }
    __syncwarp();
    if (lane == 0 && tnext < nfull) w_load_tile(ring + slot * TB, in + (u64)tnext * TB, TB, &mbar[slot]);
    u32 wc[NW], cl = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      wc[w] = __popcll(m[w]);
      cl += wc[w];
    }
    u32 inc = cl;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 y = __shfl_up_sync(FULLM, inc, d);
      if (lane >= d) inc += y;
    }
    const u32 tile_ones = __shfl_sync(FULLM, inc, 31);
    const u32 pl = inc - cl;  // ones of the tile before this lane
    run += tile_ones;
    const u32 e0 = (u32)lane * E;
    // ---- level l: words, L2 entries, select samples (rankselect.py:495-532)
    {
      u32 before = pl;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const u64 g = t0 + e0 + 64 * w;
        P.words[g >> 6] = m[w];
        if ((g & l2m) == 0) P.l2[g >> P.l2_log] = (u16)(P1 + before - l1v);
        before += wc[w];
      }
#pragma unroll
      for (int kind = 0; kind < 2; ++kind) {
        const bool ones = kind == 0;
        const u64 sb = ones ? P1 : t0 - P1;
        const u32 cnt = ones ? tile_ones : TILE - tile_ones;
        const u64 q0 = wnext_multiple(sb, P.rate, P.rate_log);
        if (q0 > sb + cnt) continue;
        const u32 lc = ones ? cl : E - cl;
        const u32 lp = ones ? pl : e0 - pl;
        u64* out = ones ? P.ones : P.zeros;
        const u64 cap = ones ? P.ones_cap : P.zeros_cap;
        for (u64 qo = q0; qo <= sb + cnt; qo += P.rate) {
          u32 tt = (u32)(qo - sb);
          if (lp < tt && tt <= lp + lc) {
            tt -= lp;
            u32 pos = e0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
              const u64 wm = ones ? m[w] : ~m[w];
              const u32 pc = __popcll(wm);
              if (tt > 0 && tt <= pc) {
                pos = e0 + 64 * w + select_in_word64(wm, tt);
                tt = 0;
              } else if (tt > 0) {
                tt -= pc;
              }
            }
            const u64 sidx = (P.rate_log >= 0 ? (qo >> P.rate_log) : qo / P.rate) - 1;
            if (sidx < cap) out[sidx] = t0 + pos;
          }
        }
      }
    }
    // ---- the last level: the two group strings ------------------------------
    const NodeEnt* ne = P.nodes + fkey;
    const u64 zdst = (u64)__ldg(&ne->zero_base) + (t0 - P1);
    const u64 odst = (u64)__ldg(&ne->one_base) + P1;
    u32* gz = gbuf;
    u32* go = gbuf + GW;
    for (int i = lane; i < GW / 2; i += 32) reinterpret_cast<uint4*>(gbuf)[i] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    const u32 zb = (u32)(zdst & 31) + (e0 - pl);  // this lane's first bit in each string
    const u32 ob = (u32)(odst & 31) + pl;
    // chunks k and k + 1 are slice chunks c and c ^ 1: an adjacent pair, one
    // piece of <= 32 bits per group
#pragma unroll
    for (int k = 0; k < K; k += 2) {
      const u32 c = (u32)k ^ ((u32)lane & 7u);
      const u32 ce = c & ~1u;  // the pair's even chunk (first in the slice)
      const u32 bit = ce * CE;
      u32 ob4 = 0;  // ones of the slice before the pair
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const u32 lo = (u32)w * 64;
        const u64 mw = bit >= lo + 64 ? m[w] : bit <= lo ? 0ull : m[w] & ((1ull << (bit - lo)) - 1ull);
        ob4 += __popcll(mw);
      }
      u32 vz = 0, vo = 0, nz = 0, no = 0;
      // c & 1 == lane & 1 (k is even): odd lanes hold the pair's even chunk in q[k + 1]
      const bool odd = (lane & 1) != 0;
      uint4 qp[2];
      qp[0] = odd ? q[k + 1] : q[k];
      qp[1] = odd ? q[k] : q[k + 1];
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // even chunk first
        const u32 cb = (ce + h) * CE;
        const u64 mw = NW == 1 ? m[0] : ((cb >> 6) ? m[NW - 1] : m[0]);
        const u32 mk = (u32)(mw >> (cb & 63)) & ((1u << CE) - 1u);
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) {
          const u32 m8 = (mk >> (8 * s2)) & 0xffu;
          u32 f0, f1;
          wp_flags<TC>(qp[h], s2, sh1, f0, f1);
          const uint2 sg = csel[m8];
          const u32 v8 = wp_gather(__byte_perm(f0, f1, sg.x), __byte_perm(f0, f1, sg.y));
          const u32 c1 = __popc(m8), c0 = 8 - c1;
          vz |= (v8 & ((1u << c0) - 1u)) << nz;
          vo |= (v8 >> c0) << no;
          nz += c0;
          no += c1;
        }
      }
      const u32 pz = zb + (bit - ob4), po = ob + ob4;
      if (nz) {
        atomicOr(gz + (pz >> 5), vz << (pz & 31));
        if ((pz & 31) + nz > 32) atomicOr(gz + (pz >> 5) + 1, vz >> (32 - (pz & 31)));
      }
      if (no) {
        atomicOr(go + (po >> 5), vo << (po & 31));
        if ((po & 31) + no > 32) atomicOr(go + (po >> 5) + 1, vo >> (32 - (po & 31)));
      }
    }
    __syncwarp();
    // ---- write the group strings; the last level's ones per L1 block ------
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const u64 dst = g ? odst : zdst;
      const u32 cnt = g ? tile_ones : TILE - tile_ones;
      if (!cnt) continue;
      const u32* buf = g ? go : gz;
      const u32 b0 = (u32)(dst & 31), e = b0 + cnt;
      const u32 nwd = (e + 31) >> 5;
      // the first word of the next L1 block, relative to the string's first word
      const u32 wsplit = (u32)(((((dst >> 16) + 1) << 16) - (dst & ~31ull)) >> 5);
      u32* nw32 = reinterpret_cast<u32*>(P.next_words) + (dst >> 5);
      u32 x = 0;  // ones before the split | after << 16
      for (u32 w = lane; w < nwd; w += 32) {
        const u32 v = buf[w];
        if ((w == 0 && b0) || (w == nwd - 1 && (e & 31))) {
          if (v) atomicOr(nw32 + w, v);
        } else {
          nw32[w] = v;
        }
        x += (u32)__popc(v) << (w >= wsplit ? 16 : 0);
      }
#pragma unroll
      for (int d = 16; d; d >>= 1) x += __shfl_xor_sync(FULLM, x, d);
      if (lane == 0 && (x & 0xffffu)) atomicAdd(P.next_l1_counts + (dst >> 16), x & 0xffffu);
      if (lane == 1 && (x >> 16)) atomicAdd(P.next_l1_counts + (dst >> 16) + 1, x >> 16);
    }
    __syncwarp();  // the strings are re-zeroed by the next tile
  }
}

// ---------------------------------------------------------------------------
// level 0: ones per warp tile of the text's top code bit (streaming pass)
// ---------------------------------------------------------------------------
// Codes are monotone in the symbol (the minimal alphabet and the reduced-tree
// codes both preserve order, alphabet.py:94-111, :160-207), so the top code
// bit of a text symbol is simply `symbol >= thr`, thr = the smallest symbol
// whose code has it set: a SWAR byte / halfword compare, no LUT.
template <typename TIn>
__global__ void __launch_bounds__(256) wcount0_kernel(const TIn* __restrict__ text, u64 n, u32 thr,
                                                      u32* __restrict__ tile_counts,
                                                      u32* __restrict__ l1_counts) {
  using S = WS<TIn>;
  constexpr int CH = S::CH;
  const int lane = threadIdx.x & 31;
  const u32 ntiles = (u32)((n + S::TILE - 1) / S::TILE);
  const u32 t4 = sizeof(TIn) == 1 ? thr * 0x01010101u : thr * 0x00010001u;
  const bool none = thr > (sizeof(TIn) == 1 ? 0xffu : 0xffffu);
  for (u32 t = blockIdx.x * 8 + (threadIdx.x >> 5); t < ntiles; t += gridDim.x * 8) {
    uint4 q[S::K];
    wload<TIn>(reinterpret_cast<const u8*>(text), n, t, lane, q);
    const u64 t0 = (u64)t * S::TILE;
    u32 cnt = 0;
#pragma unroll
    for (int k = 0; k < S::K; ++k) {
      const u32 e = (u32)(k * 32 + lane) * CH;
      const u32 w4[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
      u32 c = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        c += sizeof(TIn) == 1 ? __popc(__vcmpgeu4(w4[i], t4)) >> 3
                              : __popc(__vcmpgeu2(w4[i], t4)) >> 4;
      if (t0 + e + CH > n) {  // tail: zero-filled bytes may compare >= thr only if thr == 0
        c = 0;
        for (int j = 0; j < CH && t0 + e + j < n; ++j) {
          const u32 raw = sizeof(TIn) == 1 ? (w4[j >> 2] >> ((j & 3) * 8)) & 0xffu
                                           : (w4[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
          c += raw >= thr;
        }
      }
      cnt += none ? 0u : c;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) cnt += __shfl_xor_sync(FULLM, cnt, d);
    if (lane == 0) {
      tile_counts[t] = cnt;
      if (cnt) atomicAdd(l1_counts + (t / S::TPL1), cnt);
    }
  }
}

// one CTA: exclusive scan of per-L1-block counts -> the level's L1 directory
// (ones before each 65536-bit block) and its total.  Thread t owns L1_QPT
// consecutive uint4 quads of counts per round (a round covers 2^14 blocks = a
// 2^30-bit level, so C2's levels take one round and ONE block scan: the
// earlier quad-per-thread rounds paid two barriers per 4096 blocks); sums
// inside a round fit 32 bits (2^14 blocks x 2^16 bits).  Counts are padded to
// a multiple of 4 with zeros by the caller's memset.
constexpr int L1_QPT = 4;
__global__ void __launch_bounds__(1024) l1_scan_kernel(const u32* __restrict__ counts, u64 n_l1,
                                                       u64* __restrict__ l1, u64* __restrict__ total) {
  __shared__ u32 wsum[32];
  // a programmatic dependent launched after this kernel (the previous level's
  // directory pass) needs nothing from it: release it at once
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 quads = (n_l1 + 3) / 4;
  const uint4* c4 = reinterpret_cast<const uint4*>(counts);
  u64 carry = 0;
  for (u64 base = 0; base < quads; base += 1024 * L1_QPT) {
    uint4 v[L1_QPT];
    u32 s = 0;
#pragma unroll
    for (int j = 0; j < L1_QPT; ++j) {
      const u64 q = base + (u64)tid * L1_QPT + j;
      v[j] = q < quads ? __ldg(c4 + q) : make_uint4(0, 0, 0, 0);
      s += v[j].x + v[j].y + v[j].z + v[j].w;
    }
    u32 inc = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 y = __shfl_up_sync(FULLM, inc, d);
      if (lane >= d) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    u32 ws = wsum[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 y = __shfl_up_sync(FULLM, ws, d);
      if (lane >= d) ws += y;
    }
    const u32 round_total = __shfl_sync(FULLM, ws, 31);
    const u32 wpre = __shfl_sync(FULLM, ws - wsum[lane], warp);
    u64 e = carry + wpre + (inc - s);
#pragma unroll
    for (int j = 0; j < L1_QPT; ++j) {
      const u64 q = base + (u64)tid * L1_QPT + j;
      const u64 e0 = e, e1 = e0 + v[j].x, e2 = e1 + v[j].y, e3 = e2 + v[j].z;
      e = e3 + v[j].w;
      if (q * 4 + 3 < n_l1) {
        reinterpret_cast<ulonglong2*>(l1)[q * 2] = make_ulonglong2(e0, e1);
        reinterpret_cast<ulonglong2*>(l1)[q * 2 + 1] = make_ulonglong2(e2, e3);
      } else if (q < quads) {
        const u64 ev[4] = {e0, e1, e2, e3};
        for (int i = 0; i < 4; ++i)
          if (q * 4 + i < n_l1) l1[q * 4 + i] = ev[i];
      }
    }
    carry += round_total;
    __syncthreads();  // wsum reuse
  }
  if (tid == 0) *total = carry;
}

// L2 entries and select samples of a level from its bit-vector and L1
// directory (rankselect.py:495-532): one 128-thread CTA per 65536-bit L1
// block, thread i owns words [8 i, 8 i + 8) (four 16-byte loads), a CTA scan
// of the threads' popcounts gives every L2 prefix; a thread selects only when
// an ordinal multiple of the rate falls in its 512 bits (~1 in 8 threads at
// rate 4096).  Full occupancy keeps enough loads in flight.
constexpr int D_NT = 128;
__global__ void __launch_bounds__(D_NT, 6) dir_kernel(const __grid_constant__ DirParams P) {
  __shared__ u32 wsum[D_NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 nw = (P.m + 63) >> 6;
  const u64 nblk = (P.m + kL1Bits - 1) / kL1Bits;
  const u32 l2m = (u32)((1ull << P.l2_log) >> 6) - 1u;  // L2 block = l2m + 1 words
  for (u64 b = blockIdx.x; b < nblk; b += gridDim.x) {
    const u64 w0 = b * (kL1Bits / 64) + 8 * (u64)tid;  // this thread's first word
    u32 pc[8], c = 0;
    if (w0 + 8 <= nw) {
      const ulonglong2* src = reinterpret_cast<const ulonglong2*>(P.words + w0);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const ulonglong2 v = __ldg(src + j);
        pc[2 * j] = __popcll(v.x);
        pc[2 * j + 1] = __popcll(v.y);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) pc[j] = w0 + j < nw ? __popcll(__ldg(P.words + w0 + j)) : 0u;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) c += pc[j];
    u32 inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 y = __shfl_up_sync(FULLM, inc, d);
      if (lane >= d) inc += y;
    }
    __syncthreads();  // wsum reuse across blocks
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    u32 wpre = 0;
#pragma unroll
    for (int k = 0; k < D_NT / 32; ++k) wpre += k < warp ? wsum[k] : 0u;
    const u32 ex = wpre + inc - c;  // ones of the block before word w0
    if (w0 < nw) {
      u32 pre = ex;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (w0 + j < nw && ((u32)(w0 + j) & l2m) == 0) P.l2[((w0 + j) << 6) >> P.l2_log] = (u16)pre;
        pre += pc[j];
      }
    }
    // select samples: ~two of each kind per warp step at rate 4096 -- a
    // warp-uniform loop over the sample ordinals in the warp's range; the
    // owning lane finds the word from its popcounts, loads it (L1) and selects
    const u64 l1v = __ldg(P.l1 + b);
    const u64 g0 = min(w0 << 6, P.m);
    const u32 valid = (u32)min((u64)512, P.m - g0);
    const u64 ob = l1v + ex, zb = g0 - ob;
    const u32 zc = valid - c;
#pragma unroll
    for (int kind = 0; kind < 2; ++kind) {
      const bool ones = kind == 0;
      const u64 bl = ones ? ob : zb;
      const u32 cl = ones ? c : zc;
      const u64 bw = __shfl_sync(FULLM, bl, 0);
      const u64 ew = __shfl_sync(FULLM, bl + cl, 31);
      for (u64 qo = wnext_multiple(bw, P.rate, P.rate_log); qo <= ew; qo += P.rate) {
        if (bl < qo && qo <= bl + cl) {
          // the word holding ordinal k: binary search over the word counts
          // (zeros: the valid bits of the word minus its ones)
          u32 k = (u32)(qo - bl);
          u32 cw[8];
#pragma unroll
          for (int x = 0; x < 8; ++x) {
            const u32 vbx = valid > 64u * x ? min(64u, valid - 64u * x) : 0u;
            cw[x] = ones ? pc[x] : vbx - pc[x];
          }
          const u32 q0c = cw[0] + cw[1] + cw[2] + cw[3];
          const bool hi4 = k > q0c;
          k -= hi4 ? q0c : 0u;
          const u32 a0 = hi4 ? cw[4] : cw[0], a1 = hi4 ? cw[5] : cw[1];
          const u32 a2 = hi4 ? cw[6] : cw[2], a3 = hi4 ? cw[7] : cw[3];
          const bool hi2 = k > a0 + a1;
          k -= hi2 ? a0 + a1 : 0u;
          const u32 b0 = hi2 ? a2 : a0;
          const bool hi1 = k > b0;
          k -= hi1 ? b0 : 0u;
          const u32 j = (hi4 ? 4u : 0u) + (hi2 ? 2u : 0u) + (hi1 ? 1u : 0u);
          const u32 vb = valid > 64u * j ? min(64u, valid - 64u * j) : 0u;
          const u64 wv = __ldg(P.words + w0 + j);
          const u64 wm = (ones ? wv : ~wv) & (vb >= 64 ? ~0ull : (1ull << vb) - 1ull);
          const u64 pos = ((w0 + j) << 6) + select_in_word64(wm, k);
          const u64 si = (P.rate_log >= 0 ? (qo >> P.rate_log) : qo / P.rate) - 1;
          u64* out = ones ? P.ones : P.zeros;
          if (si < (ones ? P.ones_cap : P.zeros_cap)) out[si] = pos;
        }
      }
    }
  }
}

namespace {
// pair kernel launch (MODE 2): 8 warps per CTA, per-warp ring + group strings
template <typename TIn, typename TC, bool kLut>
cudaError_t launch_pair(const WLevelParams& p, int sms, cudaStream_t st) {
  constexpr int GW = WS<TIn>::TILE / 32 + 4;
  const int smem = 8 * (2 * WS<TIn>::BYTES + 16 + 2 * GW * 4);
  auto kern = wpair_kernel<TIn, TC, kLut>;
  static std::atomic<int> cached[64];
  int dev = 0;
  cudaGetDevice(&dev);
  const bool dev_ok = dev >= 0 && dev < 64;
  int per_sm = dev_ok ? cached[dev].load(std::memory_order_acquire) : 0;
  if (per_sm <= 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
    if (per_sm < 1) per_sm = 1;
    if (dev_ok) cached[dev].store(per_sm, std::memory_order_release);
  }
  const u64 tiles = (p.m + WS<TIn>::TILE - 1) / WS<TIn>::TILE;
  const u64 units = p.tile_counts ? tiles : (tiles + WS<TIn>::TPL1 - 1) / WS<TIn>::TPL1;
  const u64 need = (units + 7) / 8;
  const u64 cap = (u64)sms * per_sm;
  kern<<<(unsigned)(need < cap ? need : cap), 256, smem, st>>>(p);
  return cudaGetLastError();
}

template <typename TIn, typename TC, bool kLut, int MODE>
cudaError_t launch_w(const WLevelParams& p, int sms, cudaStream_t st) {
  constexpr bool kPair = MODE == 2;
  // the pair kernel handles u8 codes from either input and u16 codes from u16 input
  if (kPair && !(sizeof(TIn) == 2 && sizeof(TC) == 1 && !kLut) && !(sizeof(TIn) == 1 && sizeof(TC) == 2)) {
    const char* e = getenv("WT_PAIR_KERNEL");  // "stage": the staging variant (A/B)
    if (!(e && e[0] == 's')) return launch_pair<TIn, TC, kLut>(p, sms, st);
  }
  const size_t smem = 512 + (size_t)W_WARPS * WF<TIn, TC>::WARP_SMEM;
  auto kern = wlevel_kernel<TIn, TC, kLut, MODE>;
  // attribute + occupancy once per device (host cost off the per-level path)
  // (per device: attributes and occupancy belong to a device context;
  // racing first calls only repeat idempotent work)
  static std::atomic<int> cached[64];
  static std::atomic<bool> lattr[64];
  int dev = 0;
  cudaGetDevice(&dev);
  const bool dev_ok = dev >= 0 && dev < 64;
  int per_sm = dev_ok ? cached[dev].load(std::memory_order_acquire) : 0;
  if (per_sm <= 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W_NT, smem);
    if (per_sm < 1) per_sm = 1;
    if (dev_ok) cached[dev].store(per_sm, std::memory_order_release);
  }
  const u64 tiles = (p.m + WS<TIn>::TILE - 1) / WS<TIn>::TILE;
  if (!p.out && !kPair) {  // the last level: no partition
    u64 blocks = (tiles + 7) / 8;
    if (blocks > (u64)sms * 8) blocks = (u64)sms * 8;
    const int lsmem = 8 * (2 * WS<TIn>::BYTES + 16);
    if (!dev_ok || !lattr[dev].load(std::memory_order_acquire)) {
      cudaError_t e = cudaFuncSetAttribute(wlast_kernel<TIn, TC, kLut>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, lsmem);
      if (e != cudaSuccess) return e;
      if (dev_ok) lattr[dev].store(true, std::memory_order_release);
    }
    wlast_kernel<TIn, TC, kLut><<<(unsigned)blocks, 256, lsmem, st>>>(p);
    return cudaGetLastError();
  }
  // block mode: one warp per L1 block is all the parallelism there is
  const u64 units = p.tile_counts ? tiles : (tiles + WS<TIn>::TPL1 - 1) / WS<TIn>::TPL1;
  const u64 need = (units + W_WARPS - 1) / W_WARPS;
  const u64 cap = (u64)sms * per_sm;
  kern<<<(unsigned)(need < cap ? need : cap), W_NT, smem, st>>>(p);
  return cudaGetLastError();
}
}  // namespace

namespace {
template <int MODE>
cudaError_t launch_wlevel_t(const WLevelParams& p, int in_bytes, int code_bytes, bool lut, int sms,
                            cudaStream_t st) {
  if (in_bytes == 1 && code_bytes == 1)
    return lut ? launch_w<u8, u8, true, MODE>(p, sms, st) : launch_w<u8, u8, false, MODE>(p, sms, st);
  if (in_bytes == 1 && code_bytes == 2) return launch_w<u8, u16, true, MODE>(p, sms, st);
  if (in_bytes == 2 && code_bytes == 1) return launch_w<u16, u8, true, MODE>(p, sms, st);
  if (in_bytes == 2 && code_bytes == 2)
    return lut ? launch_w<u16, u16, true, MODE>(p, sms, st) : launch_w<u16, u16, false, MODE>(p, sms, st);
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_wlevel(const WLevelParams& p, int in_bytes, int code_bytes, bool lut, int sms,
                          cudaStream_t st) {
  if (p.m == 0) return cudaSuccess;
  if (p.next_words) return launch_wlevel_t<2>(p, in_bytes, code_bytes, lut, sms, st);
  if (p.next_block) return launch_wlevel_t<1>(p, in_bytes, code_bytes, lut, sms, st);
  return launch_wlevel_t<0>(p, in_bytes, code_bytes, lut, sms, st);
}

cudaError_t launch_wcount0(const void* text, u64 n, int in_bytes, u32 thr, u32* tile_counts,
                           u32* l1_counts, int sms, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const u32 tiles = wlevel_tiles(n, in_bytes);
  u64 blocks = (tiles + 7) / 8;
  if (blocks > (u64)sms * 16) blocks = (u64)sms * 16;
  if (in_bytes == 1)
    wcount0_kernel<u8><<<(unsigned)blocks, 256, 0, st>>>((const u8*)text, n, thr, tile_counts, l1_counts);
  else
    wcount0_kernel<u16><<<(unsigned)blocks, 256, 0, st>>>((const u16*)text, n, thr, tile_counts, l1_counts);
  return cudaGetLastError();
}

cudaError_t launch_dir(const DirParams& p, int sms, cudaStream_t st) {
  if (p.m == 0) return cudaSuccess;
  const u64 nblk = (p.m + kL1Bits - 1) / kL1Bits;
  u64 blocks = nblk;
  if (blocks > (u64)sms * 16) blocks = (u64)sms * 16;
  dir_kernel<<<(unsigned)blocks, D_NT, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_l1_scan(const u32* counts, u64 n_l1, u64* l1, u64* total, cudaStream_t st) {
  l1_scan_kernel<<<1, 1024, 0, st>>>(counts, n_l1, l1, total);
  return cudaGetLastError();
}

u64 wlevel_warp_slots(int sms) {
  int per_sm = 1;
  const size_t smem = 512 + (size_t)W_WARPS * WF<u8, u8>::WARP_SMEM;
  auto kern = wlevel_kernel<u8, u8, false, 0>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W_NT, smem) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 1;
  }
  return (u64)sms * (per_sm < 1 ? 1 : per_sm) * W_WARPS;
}

u32 wlevel_tiles(u64 m, int in_bytes) {
  const u64 t = in_bytes == 1 ? WS<u8>::TILE : WS<u16>::TILE;
  return (u32)((m + t - 1) / t);
}

}  // namespace wt
