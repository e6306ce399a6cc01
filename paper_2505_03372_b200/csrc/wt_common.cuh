// wt_common.cuh -- layout constants, device-side tree descriptors, PTX helpers.
//
// Layout contract (reference bitvec.py:1-21, rankselect.py:1-37):
//   * bits LSB-first inside u64 words; region l starts at a 1024-bit aligned
//     bit offset; padding bits are zero;
//   * L1 = ones before each 65536-bit block (u64), L2 = ones from the L1
//     block start to each l2_bits block (u16), samples = position of every
//     rate-th one / zero.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define WT_STATUS_FLAG_AGG (1ull << 62)
#define WT_STATUS_FLAG_INC (2ull << 62)
#define WT_STATUS_VALUE(x) ((x) & ((1ull << 62) - 1))

namespace wt {

typedef unsigned long long u64;
typedef long long i64;
typedef unsigned int u32;
typedef unsigned short u16;
typedef unsigned char u8;

constexpr int kWordBits = 64;
constexpr int kAlignBits = 1024;
constexpr int kL1Bits = 65536;
constexpr int kMaxLevels = 16;

// One wavelet-tree node at level l, indexed by its l-bit code prefix (key).
// A position p inside the node maps to the next level as
//   bit 1:  rank1(p) + one_base        bit 0:  rank0(p) + zero_base
// with zero_base = ones before the node and one_base = zeros before the
// node's end.  leaf[b] >= 0 when child b is a single symbol.
struct NodeEnt {
  i64 zero_base;
  i64 one_base;
  int leaf[2];
};
static_assert(sizeof(NodeEnt) == 24, "NodeEnt layout");

struct LevelDev {
  const u64* words;      // region start (word aligned)
  const u64* l1;         // stored as i64 in the reference; values >= 0
  const u16* l2;
  const u64* ones;       // select samples
  const u64* zeros;
  const NodeEnt* nodes;  // 2^l entries
  u64 n_bits, total_ones, n_ones, n_zeros, n_l1, n_l2;
};

// Query-side layout of one level ("rank lines"): 32-byte lines (one sector,
// one LDG.256), word 0 = ones before the line (absolute), words 1..kQW = the
// next 64*kQW bits of the level.  A rank step touches exactly one line;
// select narrows to a few lines through a line index per 2^kQSelLog-th one /
// zero.  (64-byte lines of 448 bits, WT_QW=7, halve the header overhead but
// double the sectors and L1 wavefronts per step.)  Built from the reference layout by
// qlayout_kernel; exports keep the reference layout (wtree.py / bitvec.py).
#ifndef WT_QW
#define WT_QW 3
#endif
constexpr int kQW = WT_QW;                // data words per line (3: 32-byte lines, 7: 64-byte)
constexpr int kQBits = 64 * kQW;          // bits per line
constexpr int kQLineBytes = 8 * (kQW + 1);
constexpr int kQLineU2 = kQLineBytes / 16;  // ulonglong2 per line
#ifndef WT_QSEL_LOG
#define WT_QSEL_LOG 6
#endif
constexpr int kQSelLog = WT_QSEL_LOG;  // one select sample per 2^kQSelLog ones / zeros
struct QLevelDev {
  const ulonglong2* lines;  // kQLineU2 x 16 B per line
  const u32* sel1;          // line holding the (j*128+1)-th one
  const u32* sel0;
  u64 n_lines, n_sel1, n_sel0, n_bits, total_ones;
};

struct TreeDev {
  LevelDev lv[kMaxLevels];
  QLevelDev ql[kMaxLevels];
  const u32* id_code;    // code value | (len << 16), per symbol id
  const i64* cum;        // sigma + 1
  const u16* symbols;    // sigma, original symbol values
  const int* sym2id;     // 65536: original symbol value -> id, -1 if absent
  u64 n;                 // text length
  u32 L, sigma, l2_shift, width;
  u64 rate;
};

// ---------------------------------------------------------------------------
// memory-model helpers for the decoupled look-back
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 ld_acquire(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u32 ld_acquire32(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release32(u32* p, u32 v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Relaxed (gpu-scope, L1-bypassing, no fences): the look-back words carry
// their value in the same 64/32-bit word as the flag, so no ordering with
// other data is needed -- and acquire loads would invalidate L1 (CCTL.IVALL).
__device__ __forceinline__ u64 ld_relaxed(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u32 ld_relaxed32(const u32* p) {
  u32 v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed32(u32* p, u32 v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// streaming 16-byte load that does not allocate in L1 (read-once data)
__device__ __forceinline__ uint4 ld_stream16(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// position (0-based) of the k-th (1-based, k <= popc(w)) set bit of a word.
// Branch-free popcount halving (the reference's select_in_word,
// rankselect.py:59-80, halves the same way).  __fns is NOT one instruction on
// sm_100a (ptxas expands it into a loop that dominated the select kernel).
__device__ __forceinline__ u32 select_in_word32(u32 w, u32 k) {
  u32 pos = 0, c, t;
  c = __popc(w & 0xffffu); t = k > c ? 16u : 0u; k -= t ? c : 0u; w >>= t; pos += t;
  c = __popc(w & 0xffu);   t = k > c ? 8u : 0u;  k -= t ? c : 0u; w >>= t; pos += t;
  c = __popc(w & 0xfu);    t = k > c ? 4u : 0u;  k -= t ? c : 0u; w >>= t; pos += t;
  c = __popc(w & 0x3u);    t = k > c ? 2u : 0u;  k -= t ? c : 0u; w >>= t; pos += t;
  return pos + (k > (w & 1u) ? 1u : 0u);
}
__device__ __forceinline__ u32 select_in_word64(u64 w, u32 k) {
  const u32 lo = (u32)w;
  const u32 c = __popc(lo);
  return k > c ? 32u + select_in_word32((u32)(w >> 32), k - c) : select_in_word32(lo, k);
}

__device__ __forceinline__ u64 warp_sum_u64(u64 v) {
#pragma unroll
  for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Decoupled look-back over per-tile status words (flag in bits 62-63).
// Called by one full warp; returns the exclusive prefix of `tile`.
__device__ __forceinline__ u64 lookback_prefix(u64* status, u32 tile, u64 tile_total) {
  const int lane = threadIdx.x & 31;
  u64 prefix = 0;
  if (tile == 0) {
    if (lane == 0) st_relaxed(&status[0], WT_STATUS_FLAG_INC | tile_total);
    return 0;
  }
  if (lane == 0) st_relaxed(&status[tile], WT_STATUS_FLAG_AGG | tile_total);
  long long pred = (long long)tile - 1;
  while (true) {
    const long long idx = pred - lane;
    u64 s = idx >= 0 ? ld_relaxed(&status[idx]) : WT_STATUS_FLAG_INC;
    while (__any_sync(0xffffffffu, (s >> 62) == 0)) {
      if ((s >> 62) == 0) s = ld_relaxed(&status[idx]);
    }
    const u32 incm = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    u64 val = WT_STATUS_VALUE(s);
    if (incm) {
      const int j = __ffs(incm) - 1;
      if (lane > j) val = 0;
      prefix += warp_sum_u64(val);
      break;
    }
    prefix += warp_sum_u64(val);
    pred -= 32;
  }
  if (lane == 0) st_relaxed(&status[tile], WT_STATUS_FLAG_INC | (prefix + tile_total));
  return prefix;
}

}  // namespace wt
