// wt_bits.cu -- rank/select directory of one stand-alone bit vector.
//
// Replaces rankselect.build_index over a single BitArray region
// (rankselect.py:442-536): phase 1 (per-L2 popcounts + in-block prefix),
// phase 2 (exclusive prefix over L1 totals) and the select samples, fused in
// one pass: one CTA per 65536-bit L1 block, 4 words per thread, decoupled
// look-back for the L1 prefix.
#include "wt_common.cuh"
#include "wt_kernels.h"

namespace wt {

constexpr int B_NT = 256;
constexpr int B_WPT = 4;  // words per thread -> 1024 words = 65536 bits per CTA

__device__ __forceinline__ void bits_emit(u64* out, u64 cap, u64 o0, u64 w, u64 rate, int rate_log,
                                          u64 pos0) {
  const u32 pc = __popcll(w);
  if (!pc) return;
  const u64 hi = o0 + pc;
  u64 q = rate_log >= 0 ? ((o0 >> rate_log) + 1) << rate_log : (o0 / rate + 1) * rate;
  for (; q <= hi; q += rate) {
    const u64 s = (rate_log >= 0 ? q >> rate_log : q / rate) - 1;
    if (s < cap) out[s] = pos0 + select_in_word64(w, (u32)(q - o0));
  }
}

__global__ void __launch_bounds__(B_NT) bits_directory_kernel(const BitsParams P) {
  __shared__ u32 s_warp[B_NT / 32];
  __shared__ u32 s_tile;
  __shared__ u64 s_P1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(P.counter, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u64 nwords = (P.n_bits + 63) >> 6;
  const u64 w0 = (u64)tile * (B_NT * B_WPT) + (u64)tid * B_WPT;
  u64 w[B_WPT];
  u32 pc[B_WPT];
  u32 tsum = 0;
#pragma unroll
  for (int i = 0; i < B_WPT; ++i) {
    w[i] = (w0 + i < nwords) ? P.words[w0 + i] : 0ull;
    const u64 bit0 = (w0 + i) << 6;
    if (bit0 + 64 > P.n_bits && bit0 < P.n_bits) w[i] &= (1ull << (P.n_bits - bit0)) - 1;
    pc[i] = __popcll(w[i]);
    tsum += pc[i];
  }
  u32 inc = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  u32 base = 0, total = 0;
#pragma unroll
  for (int i = 0; i < B_NT / 32; ++i) {
    base += i < warp ? s_warp[i] : 0;
    total += s_warp[i];
  }
  u32 pre = base + inc - tsum;  // ones in the tile before this thread's words
  if (warp == 0) {
    const u64 P1 = lookback_prefix(P.status, tile, total);
    if (lane == 0) {
      P.l1[tile] = P1;
      if ((u64)(tile + 1) * kL1Bits >= P.n_bits) *P.total_out = P1 + total;
      s_P1 = P1;
    }
  }
  __syncthreads();
  const u64 P1 = s_P1;
  const u32 l2_mask = (1u << P.l2_log) - 1;
#pragma unroll
  for (int i = 0; i < B_WPT; ++i) {
    const u64 g = (w0 + i) << 6;  // bit position of the word
    if (g < P.n_bits) {
      if ((g & l2_mask) == 0) P.l2[g >> P.l2_log] = (u16)pre;
      const u64 o0 = P1 + pre;
      const u64 vmask = (g + 64 <= P.n_bits) ? ~0ull : ((1ull << (P.n_bits - g)) - 1);
      bits_emit(P.ones, P.ones_cap, o0, w[i], P.rate, P.rate_log, g);
      bits_emit(P.zeros, P.zeros_cap, g - o0, ~w[i] & vmask, P.rate, P.rate_log, g);
    }
    pre += pc[i];
  }
}

u32 bits_tiles(u64 n_bits) { return (u32)((n_bits + kL1Bits - 1) / kL1Bits); }

cudaError_t launch_bits_directory(const BitsParams& p, cudaStream_t st) {
  const u32 tiles = bits_tiles(p.n_bits);
  if (!tiles) return cudaSuccess;
  bits_directory_kernel<<<tiles, B_NT, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace wt
