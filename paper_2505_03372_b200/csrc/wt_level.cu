// wt_level.cu -- K2: one fused pass per wavelet-tree level.
//
// Replaces, for level l, the reference's
//   stable_sort_by_prefix  (wtree.py:92-100)   -> one-pass stable per-node partition
//   fill_level / fill_region / _pack_span (wtree.py:103-107, bitvec.py:119-151)
//                                              -> SWAR bit extraction, u16/u8 stores
//   build_index phases 1-2 (rankselect.py:456-504) -> in-tile scan + decoupled look-back
//   build_index samples   (rankselect.py:509-532) -> emitted by the tile holding them
//
// One CTA = one tile of 16384 consecutive elements of the level (a quarter L1
// block).  Data flow per tile:
//   1. 16-byte streaming loads (coalesced: one warp instruction = 512 B),
//      level-0 symbol->code LUT, SWAR extraction of the level bit;
//   2. in-tile exclusive scan of ones (packed warp scans + 8-entry block scan);
//   3. warp 0 publishes the tile aggregate and runs the decoupled look-back
//      for the global ones prefix P1 while the other warps write the packed
//      bit words and stage the partitioned elements in shared memory;
//   4. L1 / L2 / select samples from (P1, in-tile prefix);
//   5. the staged tile leaves as <= 2 runs per node segment (zeros run, ones
//      run) with 16-byte stores (destinations of a node stay in
//      the node's range, and each (node, bit) run is contiguous).
// Destination of an element j with bit b in node `key`:
//   b=1: one_base[key] + R1(j)        b=0: zero_base[key] + R0(j)
#include "wt_common.cuh"
#include "wt_kernels.h"

namespace wt {

constexpr int LV_NT = 256;
constexpr int LV_EPT = 64;
constexpr int LV_TILE = LV_NT * LV_EPT;  // 16384 elements
constexpr int LV_TILES_PER_L1 = kL1Bits / LV_TILE;
constexpr int LV_MAXSEG = 512;
constexpr unsigned FULL = 0xffffffffu;

static_assert(LV_TILE <= 65535, "in-tile offsets are kept in u16");

// code element i of the thread's register file (packed in u32 words)
template <typename TC>
__device__ __forceinline__ u32 elem(const u32* cw, int i) {
  if (sizeof(TC) == 1) return (cw[i >> 2] >> ((i & 3) * 8)) & 0xffu;
  return (cw[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
}

template <typename TC>
__device__ __forceinline__ void set_elem(u32* cw, int i, u32 v) {
  if (sizeof(TC) == 1) {
    const int s = (i & 3) * 8;
    cw[i >> 2] = (cw[i >> 2] & ~(0xffu << s)) | (v << s);
  } else {
    const int s = (i & 1) * 16;
    cw[i >> 1] = (cw[i >> 1] & ~(0xffffu << s)) | (v << s);
  }
}

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

// copy one run of bytes shared -> global with 16-byte aligned stores
__device__ __forceinline__ void copy_run(u8* __restrict__ gout, const u8* __restrict__ s_stage,
                                         u32 sb, u64 db, u32 bytes) {
  if (bytes == 0) return;
  u32 head = (u32)((16 - (db & 15)) & 15);
  if (head > bytes) head = bytes;
  const u32 nvec = (bytes - head) >> 4;
  const u32 tail = bytes - head - nvec * 16;
  const int tid = threadIdx.x;
  if (tid < (int)head) gout[db + tid] = s_stage[sb + tid];
  if (tid >= 32 && tid < 32 + (int)tail) {
    const u32 o = head + nvec * 16 + (tid - 32);
    gout[db + o] = s_stage[sb + o];
  }
  for (u32 v = tid; v < nvec; v += LV_NT) {
    const u32 s = sb + head + v * 16;
    const u32* sw = reinterpret_cast<const u32*>(s_stage + (s & ~3u));
    const u32 sh = (s & 3u) * 8;
    const u32 a0 = sw[0], a1 = sw[1], a2 = sw[2], a3 = sw[3], a4 = sw[4];
    uint4 o;
    o.x = __funnelshift_r(a0, a1, sh);
    o.y = __funnelshift_r(a1, a2, sh);
    o.z = __funnelshift_r(a2, a3, sh);
    o.w = __funnelshift_r(a3, a4, sh);
    *reinterpret_cast<uint4*>(gout + db + head + (u64)v * 16) = o;
  }
}

// first multiple of `rate` strictly above `o` (64-bit)
__device__ __forceinline__ u64 next_multiple(u64 o, u64 rate, int rate_log) {
  if (rate_log >= 0) return ((o >> rate_log) + 1) << rate_log;
  return (o / rate + 1) * rate;
}

// emit select samples of one (warp-row, chunk) : ordinals (o0, o0+cnt]
__device__ __forceinline__ void emit_samples(u64* __restrict__ out, u64 cap, u64 o0, u32 mask,
                                             u64 q_row, u64 rate, int rate_log, u64 pos0) {
  const u32 cnt = __popc(mask);
  if (!cnt || q_row > o0 + cnt) return;
  u64 q = q_row;
  if (q <= o0) {
    const u64 d = o0 + 1 - q;  // < row size, small
    q += ((d + rate - 1) / rate) * rate;
  }
  for (; q <= o0 + cnt; q += rate) {
    const u64 s = (rate_log >= 0 ? (q >> rate_log) : q / rate) - 1;
    if (s < cap) out[s] = pos0 + __fns(mask, 0, (int)(q - o0));
  }
}

template <typename TIn, typename TC, bool kLut>
__global__ void __launch_bounds__(LV_NT) level_kernel(const LevelParams P) {
  constexpr int CH = 16 / (int)sizeof(TIn);    // elements per 16-byte input chunk
  constexpr int CPT = LV_EPT / CH;             // chunks per thread
  constexpr int NCH = LV_TILE / CH;            // chunks per tile
  constexpr int WPC = CH * (int)sizeof(TC) / 4;  // u32 words of codes per chunk
  constexpr int STAGE_BYTES = LV_TILE * (int)sizeof(TC);

  __shared__ __align__(16) u8 s_stage[STAGE_BYTES + 32];
  __shared__ u16 s_lut[kLut && sizeof(TIn) == 1 ? 256 : 1];
  __shared__ u16 s_lastkey[NCH];
  __shared__ u16 s_seg_start[LV_MAXSEG + 1];
  __shared__ u16 s_seg_r1[LV_MAXSEG + 1];
  __shared__ u16 s_seg_key[LV_MAXSEG + 1];
  __shared__ u32 s_warp_tot[LV_NT / 32];
  __shared__ u32 s_warp_nb[LV_NT / 32];
  __shared__ u32 s_tile, s_fkey, s_lkey, s_nseg;
  __shared__ u64 s_P1, s_l1val;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (kLut && sizeof(TIn) == 1) {
    for (int i = tid; i < 256; i += LV_NT) s_lut[i] = P.lut[i];
  }
  if (tid == 0) s_tile = atomicAdd(P.counter, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u64 t0 = (u64)tile * LV_TILE;
  const u32 valid = (u32)min((u64)LV_TILE, P.m - t0);

  // ---- 1. load, map, extract bits ------------------------------------------
  u32 cw[CPT * WPC];
  u32 msk[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const u32 c = (u32)((warp * CPT + k) * 32 + lane);
    const u32 e = c * CH;
    const TIn* src = reinterpret_cast<const TIn*>(P.in) + t0 + e;
    if (e + CH <= valid) {
      const uint4 q = ld_stream16(src);
      const u32 qw[4] = {q.x, q.y, q.z, q.w};
      if (!kLut) {
#pragma unroll
        for (int i = 0; i < 4; ++i) cw[k * WPC + i] = qw[i];
      } else {
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const u32 raw = sizeof(TIn) == 1 ? (qw[j >> 2] >> ((j & 3) * 8)) & 0xffu
                                           : (qw[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
          const u32 code = sizeof(TIn) == 1 ? (u32)s_lut[raw] : (u32)__ldg(P.lut + raw);
          set_elem<TC>(&cw[k * WPC], j, code);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < WPC; ++i) cw[k * WPC + i] = 0;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        if (e + j < valid) {
          const u32 raw = (u32)src[j];
          u32 code = raw;
          if (kLut) code = sizeof(TIn) == 1 ? (u32)s_lut[raw] : (u32)__ldg(P.lut + raw);
          set_elem<TC>(&cw[k * WPC], j, code);
        }
      }
    }
    u32 m = 0;
    constexpr int EPW = 4 / (int)sizeof(TC);  // elements per u32 word
#pragma unroll
    for (int i = 0; i < WPC; ++i) m |= word_bits<TC>(cw[k * WPC + i], P.shift_bit) << (i * EPW);
    msk[k] = m;
  }

  // first / last key of the tile (keys are sorted inside a level)
  if (tid == 0) s_fkey = elem<TC>(cw, 0) >> P.shift_key;
  {
    const u32 lc = (valid - 1) / CH, lj = (valid - 1) % CH;
    const u32 ll = lc & 31, lk = (lc >> 5) % CPT, lw = (lc >> 5) / CPT;
    if ((u32)lane == ll && (u32)warp == lw) {
#pragma unroll
      for (int k = 0; k < CPT; ++k)
        if ((u32)k == lk) {
#pragma unroll
          for (int j = 0; j < CH; ++j)
            if ((u32)j == lj) s_lkey = elem<TC>(&cw[k * WPC], j) >> P.shift_key;
        }
    }
  }

  // ---- 2. in-tile exclusive scan of ones, order (warp, chunk, lane) -------
  u32 r1c[CPT];  // ones in the tile before chunk
  u32 rowtot[CPT];
  {
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
    u32 run = 0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      r1c[k] += run;
      run += rowtot[k];
    }
    if (lane == 0) s_warp_tot[warp] = run;
  }
  __syncthreads();
  u32 tile_ones = 0, wbase = 0;
#pragma unroll
  for (int w = 0; w < LV_NT / 32; ++w) {
    const u32 t = s_warp_tot[w];
    wbase += (w < warp) ? t : 0;
    tile_ones += t;
  }
#pragma unroll
  for (int k = 0; k < CPT; ++k) r1c[k] += wbase;
  const u32 tile_zeros = valid - tile_ones;

  // ---- 3a. warp 0: aggregate + look-back + L1 value ---------------------------
  if (warp == 0) {
    if (lane == 0) st_release32(&P.agg[tile], tile_ones + 1);
    const u64 P1 = lookback_prefix(P.status, tile, tile_ones);
    if (lane == 0) {
      const u32 first = (tile / LV_TILES_PER_L1) * LV_TILES_PER_L1;
      u64 l1v = P1;
      for (u32 u = first; u < tile; ++u) {
        u32 a;
        while ((a = ld_acquire32(&P.agg[u])) == 0) {
        }
        l1v -= a - 1;
      }
      if (tile == first) P.l1[tile / LV_TILES_PER_L1] = P1;
      if (t0 + LV_TILE >= P.m) *P.total_out = P1 + tile_ones;
      s_P1 = P1;
      s_l1val = l1v;
    }
  }

  // ---- 3b. packed bit words (independent of P1) ---------------------------
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

  const bool scatter = P.out != nullptr;
  const bool single = s_fkey == s_lkey;  // written before the first barrier
  bool direct = false;                   // too many segments: unstaged stores

  // ---- 3c. segment table (only when the tile spans several nodes) ---------
  if (scatter && !single) {
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const u32 c = (u32)((warp * CPT + k) * 32 + lane);
      const u32 e = c * CH;
      int jl = (int)min((u32)CH, valid > e ? valid - e : 0u) - 1;
      u32 kk = 0;
#pragma unroll
      for (int j = 0; j < CH; ++j)
        if (j == jl) kk = elem<TC>(&cw[k * WPC], j) >> P.shift_key;
      s_lastkey[c] = (u16)kk;
    }
    __syncthreads();
    u32 nb[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const u32 c = (u32)((warp * CPT + k) * 32 + lane);
      const u32 e = c * CH;
      u32 prev = c ? s_lastkey[c - 1] : 0xffffffffu;
      u32 cnt = 0;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const u32 key = elem<TC>(&cw[k * WPC], j) >> P.shift_key;
        if (e + j < valid && e + j > 0 && key != prev) ++cnt;
        prev = key;
      }
      nb[k] = cnt;
    }
    // exclusive scan of boundary counts in the same (warp, chunk, lane) order
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
      if (lane == 0) s_warp_nb[warp] = run;
    }
    __syncthreads();
    u32 nbase = 0, nbtot = 0;
#pragma unroll
    for (int w = 0; w < LV_NT / 32; ++w) {
      const u32 t = s_warp_nb[w];
      nbase += (w < warp) ? t : 0;
      nbtot += t;
    }
    const u32 nseg = nbtot + 1;
    direct = nseg > LV_MAXSEG;
    if (!direct) {
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const u32 c = (u32)((warp * CPT + k) * 32 + lane);
        const u32 e = c * CH;
        u32 prev = c ? s_lastkey[c - 1] : 0xffffffffu;
        u32 s = nbase + nbex[k];
        u32 r1 = r1c[k];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const u32 key = elem<TC>(&cw[k * WPC], j) >> P.shift_key;
          if (e + j < valid && e + j > 0 && key != prev) {
            ++s;
            s_seg_start[s] = (u16)(e + j);
            s_seg_r1[s] = (u16)r1;
            s_seg_key[s] = (u16)key;
          }
          prev = key;
          r1 += (msk[k] >> j) & 1u;
        }
      }
      if (tid == 0) {
        s_seg_start[0] = 0;
        s_seg_r1[0] = 0;
        s_seg_key[0] = (u16)s_fkey;
        s_nseg = nseg;
      }
    }
    if (tid == LV_NT - 1 && !direct) {
      s_seg_start[nseg] = (u16)min(valid, 65535u);
      s_seg_r1[nseg] = (u16)tile_ones;
    }
    __syncthreads();
  } else if (scatter && tid == 0) {
    s_nseg = 1;
    s_seg_start[0] = 0;
    s_seg_r1[0] = 0;
    s_seg_key[0] = (u16)s_fkey;
    s_seg_start[1] = (u16)min(valid, 65535u);
    s_seg_r1[1] = (u16)tile_ones;
  }

  // ---- 3d. stage the locally partitioned tile in shared memory ------------
  TC* stage = reinterpret_cast<TC*>(s_stage);
  if (scatter && !direct) {
    if (single) {
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const u32 c = (u32)((warp * CPT + k) * 32 + lane);
        const u32 e = c * CH;
        u32 one_slot = tile_zeros + r1c[k];
        u32 zero_slot = e - r1c[k];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const u32 b = (msk[k] >> j) & 1u;
          const u32 slot = b ? one_slot : zero_slot;
          if (e + j < valid) stage[slot] = (TC)elem<TC>(&cw[k * WPC], j);
          one_slot += b;
          zero_slot += b ^ 1u;
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const u32 c = (u32)((warp * CPT + k) * 32 + lane);
        const u32 e = c * CH;
        // segment of the chunk's first element: last seg start <= e
        u32 lo = 0, hi = s_nseg - 1;
        while (lo < hi) {
          const u32 mid = (lo + hi + 1) >> 1;
          if (s_seg_start[mid] <= e) lo = mid; else hi = mid - 1;
        }
        u32 s = lo;
        u32 r1 = r1c[k];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const u32 ej = e + j;
          if (ej < valid) {
            if (s + 1 < s_nseg + 0u && s_seg_start[s + 1] == ej) ++s;
            const u32 ss = s_seg_start[s], sr = s_seg_r1[s];
            const u32 sz = (s_seg_start[s + 1] - ss) - (s_seg_r1[s + 1] - sr);
            const u32 b = (msk[k] >> j) & 1u;
            const u32 slot = b ? ss + sz + (r1 - sr) : ss + (ej - ss) - (r1 - sr);
            stage[slot] = (TC)elem<TC>(&cw[k * WPC], j);
            r1 += b;
          }
        }
      }
    }
  }
  __syncthreads();  // P1, l1 value, staged tile, segment table visible

  const u64 P1 = s_P1;
  const u64 l1v = s_l1val;

  // ---- 4. L2 entries and select samples -----------------------------------
  {
    const u32 l2_mask = (1u << P.l2_log) - 1;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const u32 c = (u32)((warp * CPT + k) * 32 + lane);
      const u64 g = t0 + (u64)c * CH;
      if (g < P.m && (g & l2_mask) == 0) P.l2[g >> P.l2_log] = (u16)(P1 + r1c[k] - l1v);
    }
    // rows of 32 chunks are contiguous in ordinal space
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const u32 c = (u32)((warp * CPT + k) * 32 + lane);
      const u32 e = c * CH;
      const u32 row_e = (u32)((warp * CPT + k) * 32) * CH;
      const u32 row_r1 = __shfl_sync(FULL, r1c[k], 0);
      const u64 o_row = P1 + row_r1;
      const u64 z_row = (t0 + row_e) - o_row;
      const u64 q1 = next_multiple(o_row, P.rate, P.rate_log);
      const u64 q0 = next_multiple(z_row, P.rate, P.rate_log);
      const u32 vmask = e >= valid ? 0u : (valid - e >= (u32)CH ? (CH == 32 ? FULL : (1u << CH) - 1)
                                                                : (1u << (valid - e)) - 1);
      const u64 o0 = P1 + r1c[k];
      const u64 z0 = (t0 + e) - o0;
      emit_samples(P.ones, P.ones_cap, o0, msk[k], q1, P.rate, P.rate_log, t0 + e);
      emit_samples(P.zeros, P.zeros_cap, z0, ~msk[k] & vmask, q0, P.rate, P.rate_log, t0 + e);
    }
  }

  // ---- 5. scatter to the next level ---------------------------------------
  if (!scatter) return;
  u8* gout = reinterpret_cast<u8*>(P.out);
  if (direct) {
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const u32 c = (u32)((warp * CPT + k) * 32 + lane);
      const u32 e = c * CH;
      u32 r1 = r1c[k];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        if (e + j < valid) {
          const u32 v = elem<TC>(&cw[k * WPC], j);
          const NodeEnt ne = P.nodes[v >> P.shift_key];
          const u32 b = (msk[k] >> j) & 1u;
          const u64 dst = b ? (u64)ne.one_base + P1 + r1
                            : (u64)ne.zero_base + (t0 + e + j - P1 - r1);
          if (dst < P.m_next) reinterpret_cast<TC*>(P.out)[dst] = (TC)v;
          r1 += b;
        }
      }
    }
    return;
  }
  const u32 nseg = s_nseg;
  for (u32 s = 0; s < nseg; ++s) {
    const u32 ss = s_seg_start[s], sr = s_seg_r1[s];
    const u32 len = s_seg_start[s + 1] - ss;
    const u32 ones = s_seg_r1[s + 1] - sr;
    const u32 zeros = len - ones;
    const NodeEnt ne = P.nodes[s_seg_key[s]];
    const u64 zdst = (u64)ne.zero_base + (t0 + ss - P1 - sr);
    const u64 odst = (u64)ne.one_base + P1 + sr;
    if (zeros && zdst < P.m_next)
      copy_run(gout, s_stage, ss * (u32)sizeof(TC), zdst * sizeof(TC), zeros * (u32)sizeof(TC));
    if (ones && odst < P.m_next)
      copy_run(gout, s_stage, (ss + zeros) * (u32)sizeof(TC), odst * sizeof(TC),
               ones * (u32)sizeof(TC));
  }
}

// ---------------------------------------------------------------------------
template <typename TIn, typename TC, bool kLut>
static cudaError_t launch_level_t(const LevelParams& p, u32 tiles, cudaStream_t st) {
  level_kernel<TIn, TC, kLut><<<tiles, LV_NT, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_level(const LevelParams& p, int in_bytes, int code_bytes, bool lut,
                         cudaStream_t st) {
  const u32 tiles = (u32)((p.m + LV_TILE - 1) / LV_TILE);
  if (tiles == 0) return cudaSuccess;
  if (in_bytes == 1 && code_bytes == 1)
    return lut ? launch_level_t<u8, u8, true>(p, tiles, st) : launch_level_t<u8, u8, false>(p, tiles, st);
  if (in_bytes == 1 && code_bytes == 2) return launch_level_t<u8, u16, true>(p, tiles, st);
  if (in_bytes == 2 && code_bytes == 1) return launch_level_t<u16, u8, true>(p, tiles, st);
  if (in_bytes == 2 && code_bytes == 2)
    return lut ? launch_level_t<u16, u16, true>(p, tiles, st) : launch_level_t<u16, u16, false>(p, tiles, st);
  return cudaErrorInvalidValue;
}

u32 level_tiles(u64 m) { return (u32)((m + LV_TILE - 1) / LV_TILE); }

}  // namespace wt
