// wt_level.cu -- K2: one fused pass per wavelet-tree level (persistent, TMA-pipelined).
//
// Replaces, for level l, the reference's
//   stable_sort_by_prefix  (wtree.py:92-100)        -> one-pass stable per-node partition
//   fill_level / fill_region / _pack_span (wtree.py:103-107, bitvec.py:119-151)
//                                                   -> SWAR bit extraction, 16-bit stores
//   build_index phases 1-2 (rankselect.py:456-504)  -> in-tile scan + decoupled look-back
//   build_index samples   (rankselect.py:509-532)   -> emitted by the tile holding them
//
// No look-back: the global ones prefix of every tile is known before the
// level starts.  Level l's scatter counts, from the runs it stages, the ones
// of level l+1 per destination tile (a few atomics per tile), and a one-CTA
// scan turns those counts into level l+1's tile prefixes (and its L1
// entries); level 0's counts come from a streaming count pass over the text.
// Persistent CTAs walk tiles in any order.  Per tile:
//   0. the NEXT tile's input is already streaming into the other shared
//      buffer (cp.async.bulk + mbarrier, issued one iteration ahead);
//   1. per 16-byte chunk: SWAR extraction of the level bit -> 16/8-bit mask,
//      packed warp scans + block scan of the ones; packed bit words stored;
//   2. each node segment of the tile leaves as a zeros run and a ones run
//      (destinations stay in the node's range, and every
//      (node, bit) run is contiguous).  Runs are staged in shared memory at
//      offsets congruent to their global destination mod 16, so each run body
//      goes out as ONE cp.async.bulk shared->global store;
//   3. L2 entries and select samples from (tile prefix, in-tile prefix);
//   4. per run, the ones of the next level's bit, split at the next level's
//      tile boundaries, are added to next_counts.
// Destination of element j with bit b in node `key`:
//   b=1: one_base[key] + R1(j)        b=0: zero_base[key] + R0(j)
#include "wt_common.cuh"
#include "wt_kernels.h"

namespace wt {

#ifndef WT_LV_NT
#define WT_LV_NT 256
#endif
constexpr int LV_NT = WT_LV_NT;
constexpr int LV_CPT = 4;      // 16-byte input chunks per thread per tile
constexpr int LV_MAXSEG = 64;  // node segments per tile staged; more -> direct stores
constexpr int LV_SEGPAD = 48;  // staging slack per segment (two 16-byte alignments)
constexpr unsigned FULL = 0xffffffffu;

template <typename TIn>
struct LvShape {
  static constexpr int CH = 16 / (int)sizeof(TIn);        // elements per chunk
  static constexpr int TILE = LV_NT * LV_CPT * CH;        // 16384 (u8) | 8192 (u16)
  static constexpr int TPL1 = kL1Bits / TILE;             // tiles per L1 block
  static constexpr int IN_BYTES = TILE * (int)sizeof(TIn);  // 16 KB
};

template <typename TIn, typename TC>
struct LvSmem {
  alignas(128) u8 in[2][LvShape<TIn>::IN_BYTES];
  alignas(128) u8 stage[LvShape<TIn>::TILE * sizeof(TC) + LV_SEGPAD * LV_MAXSEG + 64];
  u64 mbar[2];
  u32 warp_tot[LV_NT / 32];
  u32 warp_nb[LV_NT / 32];
  u32 fkey, lkey, nseg;
  u16 seg_start[LV_MAXSEG + 1];
  u16 seg_r1[LV_MAXSEG + 1];
  u16 seg_key[LV_MAXSEG + 1];
  u16 seg_zoff[LV_MAXSEG];
  u16 seg_ooff[LV_MAXSEG];
  u64 seg_zdst[LV_MAXSEG];
  u64 seg_odst[LV_MAXSEG];
  u32 cnt[8];                    // fast path: next-level ones per (run, tile)
  u16 chunk_r1[LV_NT * LV_CPT];  // in-tile ones before each chunk
  u16 chunk_m[LV_NT * LV_CPT];   // level-bit mask of each chunk
  u16 lut[256];
};

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + bulk async copies
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 smem_u32(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, u32 bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// element helpers
// ---------------------------------------------------------------------------
// bit `sh` of every packed element of one u32 word, LSB-first
template <typename TC>
__device__ __forceinline__ u32 word_bits(u32 w, u32 sh) {
  if (sizeof(TC) == 1) {
    const u32 y = (w >> sh) & 0x01010101u;
    return (y * 0x01020408u) >> 24;  // 4 bits
  } else {
    const u32 y = (w >> sh) & 0x00010001u;
    return (y | (y >> 15)) & 3u;  // 2 bits
  }
}

// load chunk c of the tile from shared memory as codes (u32 words), zeroing
// elements at or beyond `valid`; level 0 maps raw symbols through the LUT.
template <typename TIn, typename TC, bool kLut>
__device__ __forceinline__ void load_chunk(const u8* in, u32 c, u32 valid, const u16* slut,
                                           const u16* glut,
                                           u32 (&cw)[LvShape<TIn>::CH * sizeof(TC) / 4]) {
  constexpr int CH = LvShape<TIn>::CH;
  constexpr int WPC = CH * (int)sizeof(TC) / 4;
  const uint4 q = *reinterpret_cast<const uint4*>(in + c * 16);
  const u32 qw[4] = {q.x, q.y, q.z, q.w};
  const u32 e = c * CH;
  if (!kLut) {
#pragma unroll
    for (int i = 0; i < 4; ++i) cw[i] = qw[i];
  } else {
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
  if (e + CH > valid) {  // tail of the last tile: clear invalid elements
    constexpr int EPW = 4 / (int)sizeof(TC);
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      if (e + j >= valid) {
        const int wi = j / EPW, sh = (j % EPW) * 8 * (int)sizeof(TC);
        cw[wi] &= ~((sizeof(TC) == 1 ? 0xffu : 0xffffu) << sh);
      }
    }
  }
}

template <typename TC>
__device__ __forceinline__ u32 elem(const u32* cw, int j) {
  if (sizeof(TC) == 1) return (cw[j >> 2] >> ((j & 3) * 8)) & 0xffu;
  return (cw[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
}

template <typename TIn, typename TC, bool kLut>
__device__ __forceinline__ u32 code_at(const u8* in, u32 e, const u16* slut, const u16* glut) {
  const u32 raw = sizeof(TIn) == 1 ? (u32)in[e] : (u32)reinterpret_cast<const u16*>(in)[e];
  if (!kLut) return raw;
  return sizeof(TIn) == 1 ? (u32)slut[raw] : (u32)__ldg(glut + raw);
}

__device__ __forceinline__ u64 next_multiple(u64 o, u64 rate, int rate_log) {
  if (rate_log >= 0) return ((o >> rate_log) + 1) << rate_log;
  return (o / rate + 1) * rate;
}

// select samples of one chunk: ordinals (o0, o0 + popc(mask)], first candidate q
__device__ __forceinline__ void emit_samples(u64* __restrict__ out, u64 cap, u64 o0, u32 mask,
                                             u64 q, u64 rate, int rate_log, u64 pos0) {
  const u32 cnt = __popc(mask);
  if (!cnt || q > o0 + cnt) return;
  if (q <= o0) q += ((o0 + 1 - q + rate - 1) / rate) * rate;
  for (; q <= o0 + cnt; q += rate) {
    const u64 s = (rate_log >= 0 ? (q >> rate_log) : q / rate) - 1;
    if (s < cap) out[s] = pos0 + select_in_word32(mask, (u32)(q - o0));
  }
}

// ---------------------------------------------------------------------------
template <typename TIn, typename TC, bool kLut>
__global__ void __launch_bounds__(LV_NT, 768 / LV_NT) level_kernel(const LevelParams P) {
  using S = LvShape<TIn>;
  constexpr int CH = S::CH, TILE = S::TILE, CPT = LV_CPT;
  constexpr int WPC = CH * (int)sizeof(TC) / 4;
  constexpr u32 SZ = sizeof(TC);
  constexpr u32 NTILE = (u32)LvShape<TC>::TILE;  // next level's tile (its input = codes)
  extern __shared__ __align__(128) u8 smem_raw[];
  LvSmem<TIn, TC>& sm = *reinterpret_cast<LvSmem<TIn, TC>*>(smem_raw);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 ntiles = (u32)((P.m + TILE - 1) / TILE);
  const bool scatter = P.out != nullptr;

  auto issue_load = [&](u32 t, int slot) {
    const u64 t0 = (u64)t * TILE;
    const u64 bytes = min((u64)TILE, P.m - t0) * sizeof(TIn);
    const u32 bulk = (u32)(bytes & ~15ull);
    if (bulk) {
      mbar_expect_tx(&sm.mbar[slot], bulk);
      bulk_g2s(sm.in[slot], reinterpret_cast<const u8*>(P.in) + t0 * sizeof(TIn), bulk,
               &sm.mbar[slot]);
    }
  };

  if (kLut && sizeof(TIn) == 1)
    for (int i = tid; i < 256; i += LV_NT) sm.lut[i] = P.lut[i];
  if (tid == 0) {
    mbar_init(&sm.mbar[0], 1);
    mbar_init(&sm.mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x < ntiles) issue_load(blockIdx.x, 0);
  }
  __syncthreads();

  u32 phase = 0;  // bit s = parity of the next wait on mbar[s]
  for (u32 it = 0;; ++it) {
    const int slot = it & 1;
    const u32 tile = blockIdx.x + it * gridDim.x;
    if (tile >= ntiles) break;
    if (tid == 0 && tile + gridDim.x < ntiles) issue_load(tile + gridDim.x, slot ^ 1);
    const u64 t0 = (u64)tile * TILE;
    const u32 valid = (u32)min((u64)TILE, P.m - t0);
    const u64 P1 = __ldg(P.prefix + tile);                             // ones before the tile
    const u64 l1v = __ldg(P.prefix + (tile / S::TPL1) * S::TPL1);      // ones before its L1 block
    u8* in = sm.in[slot];
    if ((valid * sizeof(TIn)) & ~15u) {
      mbar_wait(&sm.mbar[slot], (phase >> slot) & 1);
      phase ^= 1u << slot;
    }
    if (tid < 8) sm.cnt[tid] = 0;
    if (tid == 0) {
      // remainder bytes the bulk copy could not take (last tile only)
      const u32 bulk = (valid * (u32)sizeof(TIn)) & ~15u;
      for (u32 b = bulk; b < valid * sizeof(TIn); ++b)
        in[b] = reinterpret_cast<const u8*>(P.in)[t0 * sizeof(TIn) + b];
    }
    __syncthreads();

    // ---- 1. masks, counts, in-tile scan ------------------------------------
    u32 msk[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const u32 c = (u32)((warp * CPT + k) * 32 + lane);
      u32 cw[WPC];
      load_chunk<TIn, TC, kLut>(in, c, valid, sm.lut, P.lut, cw);
      u32 m = 0;
      constexpr int EPW = 4 / (int)SZ;
#pragma unroll
      for (int i = 0; i < WPC; ++i) m |= word_bits<TC>(cw[i], P.shift_bit) << (i * EPW);
      msk[k] = m;
    }
    if (tid == 0) {
      sm.fkey = code_at<TIn, TC, kLut>(in, 0, sm.lut, P.lut) >> P.shift_key;
      sm.lkey = code_at<TIn, TC, kLut>(in, valid - 1, sm.lut, P.lut) >> P.shift_key;
    }
    u32 r1c[CPT], rowtot[CPT];
#pragma unroll
    for (int k = 0; k < CPT; k += 2) {
      const u32 x = (u32)__popc(msk[k]) | ((u32)__popc(msk[k + 1]) << 16);
      u32 inc = x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 y = __shfl_up_sync(FULL, inc, d);
        if (lane >= d) inc += y;
      }
      const u32 tot = __shfl_sync(FULL, inc, 31);
      const u32 ex = inc - x;
      r1c[k] = ex & 0xffffu;
      r1c[k + 1] = ex >> 16;
      rowtot[k] = tot & 0xffffu;
      rowtot[k + 1] = tot >> 16;
    }
    {
      u32 run = 0;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        r1c[k] += run;
        run += rowtot[k];
      }
      if (lane == 0) sm.warp_tot[warp] = run;
    }
    __syncthreads();
    u32 tile_ones = 0, wbase = 0;
#pragma unroll
    for (int w = 0; w < LV_NT / 32; ++w) {
      const u32 t = sm.warp_tot[w];
      wbase += (w < warp) ? t : 0;
      tile_ones += t;
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      r1c[k] += wbase;
      const u32 c = (u32)((warp * CPT + k) * 32 + lane);
      sm.chunk_r1[c] = (u16)r1c[k];
      sm.chunk_m[c] = (u16)msk[k];
    }
    const bool single = sm.fkey == sm.lkey;

    // ---- 2b. packed bit words (independent of P1) -----------------------------
    {
      const u64 region_bits = ((P.m + 63) >> 6) << 6;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const u32 c = (u32)((warp * CPT + k) * 32 + lane);
        const u64 bitoff = t0 + (u64)c * CH;
        if (bitoff < region_bits) {
          if (CH == 16)
            reinterpret_cast<u16*>(P.words)[bitoff >> 4] = (u16)msk[k];
          else
            reinterpret_cast<u8*>(P.words)[bitoff >> 3] = (u8)msk[k];
        }
      }
    }

    // ---- L2 entries and select samples (both paths) -------------------------
    auto emit_directory = [&]() {
    {
      const u32 l2_mask = (1u << P.l2_log) - 1;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const u32 c = (u32)((warp * CPT + k) * 32 + lane);
        const u64 g = t0 + (u64)c * CH;
        if (g < P.m && (g & l2_mask) == 0) P.l2[g >> P.l2_log] = (u16)(P1 + r1c[k] - l1v);
      }
      // select samples: one warp per kind locates the sampled ordinals of
      // the tile through the per-chunk prefix table (rankselect.py:509-532)
      if (warp >= LV_NT / 32 - 2) {
        const bool ones = warp == LV_NT / 32 - 1;
        const u64 base = ones ? P1 : t0 - P1;             // ordinals before the tile
        const u32 cnt = ones ? tile_ones : valid - tile_ones;
        u64* out = ones ? P.ones : P.zeros;
        const u64 cap = ones ? P.ones_cap : P.zeros_cap;
        const u64 q0 = next_multiple(base, P.rate, P.rate_log);
        for (u64 q = q0 + (u64)lane * P.rate; q <= base + cnt; q += 32 * P.rate) {
          const u32 t = (u32)(q - base);  // 1-based ordinal inside the tile
          u32 lo = 0, hi = LV_NT * CPT - 1;
          while (lo < hi) {  // last chunk whose prefix is below t
            const u32 mid = (lo + hi + 1) >> 1;
            const u32 pre = ones ? sm.chunk_r1[mid] : mid * CH - sm.chunk_r1[mid];
            if (pre < t) lo = mid; else hi = mid - 1;
          }
          const u32 pre = ones ? sm.chunk_r1[lo] : lo * CH - sm.chunk_r1[lo];
          u32 mk = sm.chunk_m[lo];
          if (!ones) {
            const u32 e = lo * CH;
            mk = ~mk & (valid - e >= (u32)CH ? (1u << CH) - 1 : (1u << (valid - e)) - 1);
          }
          const u64 sidx = (P.rate_log >= 0 ? (q >> P.rate_log) : q / P.rate) - 1;
          if (sidx < cap) out[sidx] = t0 + lo * CH + select_in_word32(mk, t - pre);
        }
      }
    }

    };

    if (scatter && single) {
      // ---- fast path: the whole tile lies in one node ----------------------
      // Both runs' destinations, staging offsets and next-level tile
      // boundaries are computed redundantly by every thread (no run table).
      const u32 tile_zeros = valid - tile_ones;
      const NodeEnt* ne = P.nodes + sm.fkey;
      const u64 zdst = (u64)__ldg(&ne->zero_base) + (t0 - P1);
      const u64 odst = (u64)__ldg(&ne->one_base) + P1;
      const u32 zoff = (u32)((zdst * SZ) & 15);
      const u32 ooff = ((zoff + tile_zeros * SZ + 15) & ~15u) + (u32)((odst * SZ) & 15);
      const bool zlive = tile_zeros && zdst < P.m_next;
      const bool olive = tile_ones && odst < P.m_next;
      const u32 zb1 = (u32)((zdst / NTILE + 1) * NTILE - zdst), zb2 = zb1 + NTILE;
      const u32 ob1 = (u32)((odst / NTILE + 1) * NTILE - odst), ob2 = ob1 + NTILE;
      const u32 sh1 = P.shift_bit - 1;
      u32 cz0 = 0, cz1 = 0, cz2 = 0, co0 = 0, co1 = 0, co2 = 0;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const u32 c = (u32)((warp * CPT + k) * 32 + lane);
        const u32 e = c * CH;
        if (e >= valid) continue;
        u32 cw[WPC];
        load_chunk<TIn, TC, kLut>(in, c, valid, sm.lut, P.lut, cw);
        const u32 m = msk[k];
        u32 oslot = ooff + r1c[k] * SZ;
        u32 zslot = zoff + (e - r1c[k]) * SZ;
        if (e + CH <= valid) {
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const u32 v = elem<TC>(cw, j);
            if (m & (1u << j)) {
              *reinterpret_cast<TC*>(sm.stage + oslot) = (TC)v;
              oslot += SZ;
            } else {
              *reinterpret_cast<TC*>(sm.stage + zslot) = (TC)v;
              zslot += SZ;
            }
          }
        } else {
          for (int j = 0; j < CH && e + j < valid; ++j) {
            const u32 v = elem<TC>(cw, j);
            const u32 b = (m >> j) & 1u;
            *reinterpret_cast<TC*>(sm.stage + (b ? oslot : zslot)) = (TC)v;
            oslot += b * SZ;
            zslot += (b ^ 1u) * SZ;
          }
        }
        // next level's ones of this chunk, per run and destination tile
        u32 m1 = 0;
        constexpr int EPW = 4 / (int)SZ;
#pragma unroll
        for (int i = 0; i < WPC; ++i) m1 |= word_bits<TC>(cw[i], sh1) << (i * EPW);
        const u32 vm = valid - e >= (u32)CH ? (1u << CH) - 1 : (1u << (valid - e)) - 1;
        if (zlive) {
          const u32 zm = ~m & vm, i0 = e - r1c[k], nz = __popc(zm);
          const u32 hits = m1 & zm;
          if (i0 + nz <= zb1) {
            cz0 += __popc(hits);
          } else if (i0 >= zb1 && i0 + nz <= zb2) {
            cz1 += __popc(hits);
          } else {  // a boundary falls inside this chunk's zeros
            const u32 k1 = min(nz, zb1 > i0 ? zb1 - i0 : 0u), k2 = min(nz, zb2 > i0 ? zb2 - i0 : 0u);
            const u32 b1m = k1 ? (k1 >= nz ? zm : zm & ((2u << select_in_word32(zm, k1)) - 1)) : 0u;
            const u32 b2m = k2 ? (k2 >= nz ? zm : zm & ((2u << select_in_word32(zm, k2)) - 1)) : 0u;
            cz0 += __popc(hits & b1m);
            cz1 += __popc(hits & b2m & ~b1m);
            cz2 += __popc(hits & ~b2m);
          }
        }
        if (olive) {
          const u32 om = m, i0 = r1c[k], no = __popc(om);
          const u32 hits = m1 & om;
          if (i0 + no <= ob1) {
            co0 += __popc(hits);
          } else if (i0 >= ob1 && i0 + no <= ob2) {
            co1 += __popc(hits);
          } else {
            const u32 k1 = min(no, ob1 > i0 ? ob1 - i0 : 0u), k2 = min(no, ob2 > i0 ? ob2 - i0 : 0u);
            const u32 b1m = k1 ? (k1 >= no ? om : om & ((2u << select_in_word32(om, k1)) - 1)) : 0u;
            const u32 b2m = k2 ? (k2 >= no ? om : om & ((2u << select_in_word32(om, k2)) - 1)) : 0u;
            co0 += __popc(hits & b1m);
            co1 += __popc(hits & b2m & ~b1m);
            co2 += __popc(hits & ~b2m);
          }
        }
      }
      fence_proxy_async();
#pragma unroll
      for (int d = 16; d; d >>= 1) {
        cz0 += __shfl_xor_sync(FULL, cz0, d);
        cz1 += __shfl_xor_sync(FULL, cz1, d);
        cz2 += __shfl_xor_sync(FULL, cz2, d);
        co0 += __shfl_xor_sync(FULL, co0, d);
        co1 += __shfl_xor_sync(FULL, co1, d);
        co2 += __shfl_xor_sync(FULL, co2, d);
      }
      if (lane == 0) {
        if (cz0) atomicAdd(&sm.cnt[0], cz0);
        if (cz1) atomicAdd(&sm.cnt[1], cz1);
        if (cz2) atomicAdd(&sm.cnt[2], cz2);
        if (co0) atomicAdd(&sm.cnt[3], co0);
        if (co1) atomicAdd(&sm.cnt[4], co1);
        if (co2) atomicAdd(&sm.cnt[5], co2);
      }
      __syncthreads();  // staged tile, counts and the chunk table complete
      emit_directory();
      if (warp == 0) {
        u8* gout = reinterpret_cast<u8*>(P.out);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const bool live = r ? olive : zlive;
          if (!live) continue;
          const u32 cnt = r ? tile_ones : tile_zeros;
          const u64 dst = r ? odst : zdst;
          const u32 soff = r ? ooff : zoff;
          const u32 bytes = cnt * SZ;
          const u64 db = dst * SZ;
          u32 head = (u32)((16 - (db & 15)) & 15);
          if (head > bytes) head = bytes;
          const u32 body = (bytes - head) & ~15u;
          const u32 tail = bytes - head - body;
          if (lane < (int)head) gout[db + lane] = sm.stage[soff + lane];
          if (lane >= 16 && lane < 16 + (int)tail) {
            const u32 o = head + body + (lane - 16);
            gout[db + o] = sm.stage[soff + o];
          }
          if (lane == 0 && body) bulk_s2g(gout + db + head, sm.stage + soff + head, body);
          if (lane == 1) {
            const u64 tf = dst / NTILE;
            const u32* cc = sm.cnt + 3 * r;
            if (cc[0]) atomicAdd(P.next_counts + tf, cc[0]);
            if (cc[1]) atomicAdd(P.next_counts + tf + 1, cc[1]);
            if (cc[2]) atomicAdd(P.next_counts + tf + 2, cc[2]);
          }
        }
        if (lane == 0) {
          bulk_commit();
          bulk_wait_read();
        }
      }
    } else {
    // ---- general path: several node segments, or the last level -------------
    // ---- 2c. node segments of the tile (only when it spans several nodes) ---
    u32 nseg = 1;
    if (scatter && !single) {
      u32 nb[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const u32 c = (u32)((warp * CPT + k) * 32 + lane);
        const u32 e = c * CH;
        u32 prev = e ? code_at<TIn, TC, kLut>(in, e - 1, sm.lut, P.lut) >> P.shift_key : 0u;
        u32 cnt = 0;
        for (int j = 0; j < CH; ++j) {
          if (e + j >= valid) break;
          const u32 key = code_at<TIn, TC, kLut>(in, e + j, sm.lut, P.lut) >> P.shift_key;
          if (e + j > 0 && key != prev) ++cnt;
          prev = key;
        }
        nb[k] = cnt;
      }
      u32 nbex[CPT];
      {
        u32 run = 0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
          u32 inc = nb[k];
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const u32 y = __shfl_up_sync(FULL, inc, d);
            if (lane >= d) inc += y;
          }
          nbex[k] = run + inc - nb[k];
          run += __shfl_sync(FULL, inc, 31);
        }
        if (lane == 0) sm.warp_nb[warp] = run;
      }
      __syncthreads();
      u32 nbase = 0, nbtot = 0;
#pragma unroll
      for (int w = 0; w < LV_NT / 32; ++w) {
        const u32 t = sm.warp_nb[w];
        nbase += (w < warp) ? t : 0;
        nbtot += t;
      }
      nseg = nbtot + 1;
      if (nseg <= LV_MAXSEG) {
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
          if (!nb[k]) continue;
          const u32 c = (u32)((warp * CPT + k) * 32 + lane);
          const u32 e = c * CH;
          u32 prev = e ? code_at<TIn, TC, kLut>(in, e - 1, sm.lut, P.lut) >> P.shift_key : 0u;
          u32 s = nbase + nbex[k];
          u32 r1 = r1c[k];
          for (int j = 0; j < CH; ++j) {
            if (e + j >= valid) break;
            const u32 key = code_at<TIn, TC, kLut>(in, e + j, sm.lut, P.lut) >> P.shift_key;
            if (e + j > 0 && key != prev) {
              ++s;
              sm.seg_start[s] = (u16)(e + j);
              sm.seg_r1[s] = (u16)r1;
              sm.seg_key[s] = (u16)key;
            }
            prev = key;
            r1 += (msk[k] >> j) & 1u;
          }
        }
      }
    }
    if (scatter && tid == 0) {
      sm.nseg = nseg;
      if (nseg <= LV_MAXSEG) {
        sm.seg_start[0] = 0;
        sm.seg_r1[0] = 0;
        sm.seg_key[0] = (u16)sm.fkey;
        sm.seg_start[nseg] = (u16)valid;
        sm.seg_r1[nseg] = (u16)tile_ones;
      }
    }
    __syncthreads();  // segment table

    // ---- 3. runs: destinations, staging offsets congruent mod 16 ----------
    const bool direct = scatter && nseg > LV_MAXSEG;
    if (scatter && !direct && tid < (int)nseg) {
      const u32 s = tid;
      const u32 ss = sm.seg_start[s], sr = sm.seg_r1[s];
      const u32 ones = sm.seg_r1[s + 1] - sr;
      const u32 zeros = (sm.seg_start[s + 1] - ss) - ones;
      const NodeEnt* ne = P.nodes + sm.seg_key[s];
      const u64 zdst = (u64)__ldg(&ne->zero_base) + (t0 + ss - P1 - sr);
      const u64 odst = (u64)__ldg(&ne->one_base) + P1 + sr;
      const u32 base = ((ss * SZ + LV_SEGPAD * s) + 15) & ~15u;
      const u32 zoff = base + (u32)((zdst * SZ) & 15);
      const u32 ooff = ((zoff + zeros * SZ + 15) & ~15u) + (u32)((odst * SZ) & 15);
      sm.seg_zoff[s] = (u16)zoff;
      sm.seg_ooff[s] = (u16)ooff;
      sm.seg_zdst[s] = zdst;
      sm.seg_odst[s] = odst;
    }
    if (scatter && !direct) __syncthreads();

    // ---- 3b. stage the partitioned tile (or store directly) ------------------
    if (scatter) {
      TC* gout = reinterpret_cast<TC*>(P.out);
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const u32 c = (u32)((warp * CPT + k) * 32 + lane);
        const u32 e = c * CH;
        if (e >= valid) continue;
        u32 cw[WPC];
        load_chunk<TIn, TC, kLut>(in, c, valid, sm.lut, P.lut, cw);
        const u32 m = msk[k];
        if (direct) {
          u32 r1 = r1c[k];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            if (e + j < valid) {
              const u32 v = elem<TC>(cw, j);
              const NodeEnt* ne = P.nodes + (v >> P.shift_key);
              const u32 b = (m >> j) & 1u;
              const u64 dst = b ? (u64)__ldg(&ne->one_base) + P1 + r1
                                : (u64)__ldg(&ne->zero_base) + (t0 + e + j - P1 - r1);
              if (dst < P.m_next) {
                gout[dst] = (TC)v;
                if ((v >> (P.shift_bit - 1)) & 1u) atomicAdd(P.next_counts + dst / NTILE, 1u);
              }
              r1 += b;
            }
          }
        } else if (single) {
          u32 oslot = sm.seg_ooff[0] + r1c[k] * SZ;
          u32 zslot = sm.seg_zoff[0] + (e - r1c[k]) * SZ;
          if (e + CH <= valid) {
#pragma unroll
            for (int j = 0; j < CH; ++j) {
              const u32 v = elem<TC>(cw, j);
              if (m & (1u << j)) {
                *reinterpret_cast<TC*>(sm.stage + oslot) = (TC)v;
                oslot += SZ;
              } else {
                *reinterpret_cast<TC*>(sm.stage + zslot) = (TC)v;
                zslot += SZ;
              }
            }
          } else {
            for (int j = 0; j < CH && e + j < valid; ++j) {
              const u32 v = elem<TC>(cw, j);
              const u32 b = (m >> j) & 1u;
              *reinterpret_cast<TC*>(sm.stage + (b ? oslot : zslot)) = (TC)v;
              oslot += b * SZ;
              zslot += (b ^ 1u) * SZ;
            }
          }
        } else {
          u32 lo = 0, hi = nseg - 1;
          while (lo < hi) {
            const u32 mid = (lo + hi + 1) >> 1;
            if (sm.seg_start[mid] <= e) lo = mid; else hi = mid - 1;
          }
          u32 s = lo;
          u32 r1 = r1c[k];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const u32 ej = e + j;
            if (ej < valid) {
              if (s + 1 < nseg && sm.seg_start[s + 1] == ej) ++s;
              const u32 ss = sm.seg_start[s], sr = sm.seg_r1[s];
              const u32 b = (m >> j) & 1u;
              const u32 slot = b ? sm.seg_ooff[s] + (r1 - sr) * SZ
                                 : sm.seg_zoff[s] + ((ej - ss) - (r1 - sr)) * SZ;
              *reinterpret_cast<TC*>(sm.stage + slot) = (TC)elem<TC>(cw, j);
              r1 += b;
            }
          }
        }
      }
      if (!direct) fence_proxy_async();
    }

    emit_directory();

    // ---- 5. runs leave: bulk body per run, heads / tails by lanes; the next
    //         level's ones are counted per destination tile on the way ------
    if (scatter && !direct) {
      __syncthreads();  // staged tile complete (and proxy-fenced)
      u8* gout = reinterpret_cast<u8*>(P.out);
      bool issued = false;
      for (u32 r = warp; r < 2 * nseg; r += LV_NT / 32) {
        const u32 s = r >> 1;
        const bool one = r & 1;
        const u32 ss = sm.seg_start[s], sr = sm.seg_r1[s];
        const u32 ones = sm.seg_r1[s + 1] - sr;
        const u32 cnt = one ? ones : (sm.seg_start[s + 1] - ss) - ones;
        const u64 dst = one ? sm.seg_odst[s] : sm.seg_zdst[s];
        if (!cnt || dst >= P.m_next) continue;  // empty run or leaf child
        const u32 soff = one ? sm.seg_ooff[s] : sm.seg_zoff[s];
        const u32 bytes = cnt * SZ;
        const u64 db = dst * SZ;
        u32 head = (u32)((16 - (db & 15)) & 15);
        if (head > bytes) head = bytes;
        const u32 body = (bytes - head) & ~15u;
        const u32 tail = bytes - head - body;
        if (lane < (int)head) gout[db + lane] = sm.stage[soff + lane];
        if (lane >= 16 && lane < 16 + (int)tail) {
          const u32 o = head + body + (lane - 16);
          gout[db + o] = sm.stage[soff + o];
        }
        if (lane == 0 && body) {
          bulk_s2g(gout + db + head, sm.stage + soff + head, body);
          issued = true;
        }
        // ones of the next level's bit in the run, split at the next level's
        // tile boundaries (a run of <= one tile spans at most three of them).
        // Aligned 16-byte chunks covering [soff, soff + bytes) of the stage.
        const u64 t_first = dst / NTILE;
        const u32 b1 = (u32)((t_first + 1) * NTILE - dst);  // run index of 1st boundary
        const u32 b2 = b1 + NTILE;
        const u32 a0 = soff & ~15u;
        constexpr int EPC = 16 / (int)SZ;
        const u32 nchunks = (soff + bytes - a0 + 15) >> 4;
        u32 c0 = 0, c1 = 0, c2 = 0;
        const u32 sh1 = P.shift_bit - 1;
        for (u32 q = lane; q < nchunks; q += 32) {
          const uint4 v = *reinterpret_cast<const uint4*>(sm.stage + a0 + q * 16);
          u32 mm = 0;
          constexpr int EPW = 4 / (int)SZ;
          mm |= word_bits<TC>(v.x, sh1);
          mm |= word_bits<TC>(v.y, sh1) << EPW;
          mm |= word_bits<TC>(v.z, sh1) << (2 * EPW);
          mm |= word_bits<TC>(v.w, sh1) << (3 * EPW);
          // run index of chunk element 0 (may be negative for the first chunk)
          const int i0 = (int)(a0 + q * 16 - soff) / (int)SZ;
          // keep elements with run index in [0, cnt)
          const int lo_cut = i0 < 0 ? -i0 : 0;
          const int hi_keep = (int)cnt - i0;  // elements with index < hi_keep
          u32 keep = hi_keep >= EPC ? (EPC == 16 ? 0xffffu : 0xffu) : (1u << hi_keep) - 1u;
          keep &= ~((1u << lo_cut) - 1u);
          mm &= keep;
          // split at b1, b2 (run indices)
          const int k1 = (int)b1 - i0, k2 = (int)b2 - i0;
          const u32 below1 = k1 <= 0 ? 0u : (k1 >= EPC ? 0xffffu : (1u << k1) - 1u);
          const u32 below2 = k2 <= 0 ? 0u : (k2 >= EPC ? 0xffffu : (1u << k2) - 1u);
          c0 += __popc(mm & below1);
          c1 += __popc(mm & below2 & ~below1);
          c2 += __popc(mm & ~below2);
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) {
          c0 += __shfl_xor_sync(FULL, c0, d);
          c1 += __shfl_xor_sync(FULL, c1, d);
          c2 += __shfl_xor_sync(FULL, c2, d);
        }
        if (lane == 0) {
          if (c0) atomicAdd(P.next_counts + t_first, c0);
          if (c1) atomicAdd(P.next_counts + t_first + 1, c1);
          if (c2) atomicAdd(P.next_counts + t_first + 2, c2);
        }
      }
      if (issued) {
        bulk_commit();
        bulk_wait_read();  // staging buffer reusable once the bulk reads are done
      }
    }
    }
    __syncthreads();  // end of tile: input slot and staging buffer free
  }
}

// ---------------------------------------------------------------------------
// level 0: ones per tile of the text's top code bit (streaming pass)
// ---------------------------------------------------------------------------
template <typename TIn, bool kLut>
__global__ void __launch_bounds__(LV_NT) count0_kernel(const TIn* __restrict__ text, u64 n,
                                                      const u16* __restrict__ lut, u32 shift_bit,
                                                      u32* __restrict__ counts) {
  using S = LvShape<TIn>;
  constexpr int CH = S::CH;
  __shared__ u16 slut[kLut && sizeof(TIn) == 1 ? 256 : 1];
  __shared__ u32 wsum[LV_NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (kLut && sizeof(TIn) == 1)
    for (int i = tid; i < 256; i += LV_NT) slut[i] = lut[i];
  __syncthreads();
  const u64 t0 = (u64)blockIdx.x * S::TILE;
  u32 cnt = 0;
#pragma unroll
  for (int k = 0; k < LV_CPT; ++k) {
    const u64 e = t0 + (u64)((warp * LV_CPT + k) * 32 + lane) * CH;
    if (e >= n) continue;
    u32 qw[4] = {0, 0, 0, 0};
    if (e + CH <= n) {
      const uint4 q = ld_stream16(text + e);
      qw[0] = q.x; qw[1] = q.y; qw[2] = q.z; qw[3] = q.w;
    } else {
      for (int j = 0; (u64)j < n - e; ++j) {
        const u32 v = (u32)text[e + j];
        if (sizeof(TIn) == 1) qw[j >> 2] |= v << ((j & 3) * 8);
        else qw[j >> 1] |= v << ((j & 1) * 16);
      }
    }
    if (!kLut) {
#pragma unroll
      for (int i = 0; i < 4; ++i) cnt += __popc(word_bits<TIn>(qw[i], shift_bit));
    } else {
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        if (e + j >= n) break;
        const u32 raw = sizeof(TIn) == 1 ? (qw[j >> 2] >> ((j & 3) * 8)) & 0xffu
                                         : (qw[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
        const u32 code = sizeof(TIn) == 1 ? (u32)slut[raw] : (u32)__ldg(lut + raw);
        cnt += (code >> shift_bit) & 1u;
      }
    }
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) cnt += __shfl_xor_sync(FULL, cnt, d);
  if (lane == 0) wsum[warp] = cnt;
  __syncthreads();
  if (tid == 0) {
    u32 t = 0;
    for (int w = 0; w < LV_NT / 32; ++w) t += wsum[w];
    counts[blockIdx.x] = t;
  }
}

// one CTA: exclusive prefix of the per-tile counts, L1 entries, level total.
// Each thread owns a contiguous run of tiles read as uint4 (counts are
// padded to a multiple of 4 with zeros by the caller's memset).
__global__ void __launch_bounds__(1024) tile_scan_kernel(const u32* __restrict__ counts, u32 tiles,
                                                         int tpl1, u64* __restrict__ prefix,
                                                         u64* __restrict__ l1, u64 n_l1,
                                                         u64* __restrict__ total) {
  __shared__ u64 wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 quads = (tiles + 3) / 4;
  const u32 per = (quads + 1023) / 1024;  // quads per thread
  const u32 a = min(quads, tid * per), b = min(quads, a + per);
  const uint4* c4 = reinterpret_cast<const uint4*>(counts);
  u64 s = 0;
  for (u32 i = a; i < b; ++i) {
    const uint4 v = __ldg(c4 + i);
    s += (u64)v.x + v.y + v.z + v.w;
  }
  u64 inc = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u64 y = __shfl_up_sync(FULL, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    u64 v = wsum[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u64 y = __shfl_up_sync(FULL, v, d);
      if (lane >= d) v += y;
    }
    wsum[lane] = v;  // inclusive per warp
  }
  __syncthreads();
  u64 run = (warp ? wsum[warp - 1] : 0) + inc - s;
  for (u32 i = a; i < b; ++i) {
    const uint4 v = __ldg(c4 + i);
    const u32 t = i * 4;
    ulonglong2 p0, p1;
    p0.x = run; run += v.x;
    p0.y = run; run += v.y;
    p1.x = run; run += v.z;
    p1.y = run; run += v.w;
    if (t + 3 < tiles) {
      reinterpret_cast<ulonglong2*>(prefix + t)[0] = p0;  // prefix is 16-byte aligned
      reinterpret_cast<ulonglong2*>(prefix + t)[1] = p1;
    } else {
      const u64 pv[4] = {p0.x, p0.y, p1.x, p1.y};
      for (u32 j = 0; j < 4 && t + j < tiles; ++j) prefix[t + j] = pv[j];
    }
  }
  if (tid == 1023) {
    prefix[tiles] = wsum[31];
    *total = wsum[31];
  }
  __syncthreads();
  for (u64 j = tid; j < n_l1; j += 1024) l1[j] = prefix[j * tpl1];
}

template <typename TIn, typename TC, bool kLut>
static cudaError_t launch_level_t(const LevelParams& p, cudaStream_t st) {
  using S = LvShape<TIn>;
  const size_t smem = sizeof(LvSmem<TIn, TC>);
  auto kern = level_kernel<TIn, TC, kLut>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LV_NT, smem);
  if (per_sm < 1) per_sm = 1;
  const u64 tiles = (p.m + S::TILE - 1) / S::TILE;
  const u64 cap = (u64)sms * per_sm;
  const u64 grid = tiles < cap ? tiles : cap;
  kern<<<(unsigned)grid, LV_NT, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_level(const LevelParams& p, int in_bytes, int code_bytes, bool lut,
                         cudaStream_t st) {
  if (p.m == 0) return cudaSuccess;
  if (in_bytes == 1 && code_bytes == 1)
    return lut ? launch_level_t<u8, u8, true>(p, st) : launch_level_t<u8, u8, false>(p, st);
  if (in_bytes == 1 && code_bytes == 2) return launch_level_t<u8, u16, true>(p, st);
  if (in_bytes == 2 && code_bytes == 1) return launch_level_t<u16, u8, true>(p, st);
  if (in_bytes == 2 && code_bytes == 2)
    return lut ? launch_level_t<u16, u16, true>(p, st) : launch_level_t<u16, u16, false>(p, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_level0_counts(const void* text, u64 n, int in_bytes, const u16* lut,
                                 u32 shift_bit, u32* counts, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const u32 tiles = level_tiles(n, in_bytes);
  if (in_bytes == 1) {
    if (lut) count0_kernel<u8, true><<<tiles, LV_NT, 0, st>>>((const u8*)text, n, lut, shift_bit, counts);
    else count0_kernel<u8, false><<<tiles, LV_NT, 0, st>>>((const u8*)text, n, lut, shift_bit, counts);
  } else {
    if (lut) count0_kernel<u16, true><<<tiles, LV_NT, 0, st>>>((const u16*)text, n, lut, shift_bit, counts);
    else count0_kernel<u16, false><<<tiles, LV_NT, 0, st>>>((const u16*)text, n, lut, shift_bit, counts);
  }
  return cudaGetLastError();
}

cudaError_t launch_tile_scan(const u32* counts, u32 tiles, int tiles_per_l1, u64* prefix, u64* l1,
                             u64 n_l1, u64* total, cudaStream_t st) {
  tile_scan_kernel<<<1, 1024, 0, st>>>(counts, tiles, tiles_per_l1, prefix, l1, n_l1, total);
  return cudaGetLastError();
}

u32 level_tiles(u64 m, int in_bytes) {
  const u64 t = in_bytes == 1 ? LvShape<u8>::TILE : LvShape<u16>::TILE;
  return (u32)((m + t - 1) / t);
}
int level_tiles_per_l1(int in_bytes) {
  return in_bytes == 1 ? LvShape<u8>::TPL1 : LvShape<u16>::TPL1;
}

}  // namespace wt
