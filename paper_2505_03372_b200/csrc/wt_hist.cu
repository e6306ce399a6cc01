// wt_hist.cu -- K1: raw-symbol histogram of the text.
//
// Replaces the O(n) parts of minimal_alphabet (alphabet.py:94-111: bincount /
// np.unique over the text) and the bincount of encode_and_histogram
// (alphabet.py:210-242).  The histogram of raw symbol values gives the
// present set (-> minimal alphabet) and, after the O(sigma) host mapping, the
// per-id histogram (-> cum_hist, level sizes, node tables).
//
// u8 : warp-private shared-memory sub-histograms (8 x 256 counters per CTA),
//      16-byte streaming loads, one merge per CTA.
// u16: warp-aggregated (match_any) global atomics into 65536 u64 bins.
#include "wt_common.cuh"
#include "wt_kernels.h"

namespace wt {

constexpr int H_NT = 256;

__global__ void __launch_bounds__(H_NT) hist8_kernel(const u8* __restrict__ text, u64 n,
                                                     u64* __restrict__ hist) {
  __shared__ u32 sh[H_NT / 32][256];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (H_NT / 32) * 256; i += H_NT) (&sh[0][0])[i] = 0;
  __syncthreads();
  u32* mine = sh[warp];
  const u64 nvec = n >> 4;
  const u64 stride = (u64)gridDim.x * H_NT;
  for (u64 v = (u64)blockIdx.x * H_NT + tid; v < nvec; v += stride) {
    const uint4 q = ld_stream16(text + (v << 4));
    const u32 w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
      for (int b = 0; b < 4; ++b) atomicAdd(&mine[(w[i] >> (8 * b)) & 0xff], 1u);
    }
  }
  if (blockIdx.x == 0) {
    for (u64 i = (nvec << 4) + tid; i < n; i += H_NT) atomicAdd(&mine[text[i]], 1u);
  }
  __syncthreads();
  for (int b = tid; b < 256; b += H_NT) {
    u64 s = 0;
#pragma unroll
    for (int w = 0; w < H_NT / 32; ++w) s += sh[w][b];
    if (s) atomicAdd(&hist[b], s);
  }
}

__global__ void __launch_bounds__(H_NT) hist16_kernel(const u16* __restrict__ text, u64 n,
                                                      u64* __restrict__ hist) {
  const int lane = threadIdx.x & 31;
  const u64 nvec = n >> 3;
  const u64 stride = (u64)gridDim.x * H_NT;
  // every lane of a warp runs the same trip count so match_any sees full warps
  const u64 base0 = (u64)blockIdx.x * H_NT + (threadIdx.x & ~31);
  for (u64 vb = base0; vb < nvec; vb += stride) {
    const u64 v = vb + lane;
    const bool ok = v < nvec;
    uint4 q = make_uint4(0, 0, 0, 0);
    if (ok) q = ld_stream16(text + (v << 3));
    const u32 w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const u32 s = ok ? (w[i >> 1] >> ((i & 1) * 16)) & 0xffffu : 0x10000u + lane;
      const u32 peers = __match_any_sync(0xffffffffu, s);
      if (ok && lane == __ffs(peers) - 1) atomicAdd(&hist[s], (u64)__popc(peers));
    }
  }
  if (blockIdx.x == 0) {
    for (u64 i = (nvec << 3) + threadIdx.x; i < n; i += H_NT) atomicAdd(&hist[text[i]], 1ull);
  }
}

__global__ void __launch_bounds__(H_NT) first_outside_kernel(const void* __restrict__ text, u64 n,
                                                             int sym_bytes,
                                                             const u8* __restrict__ member,
                                                             u64* __restrict__ best) {
  const u64 stride = (u64)gridDim.x * H_NT;
  for (u64 i = (u64)blockIdx.x * H_NT + threadIdx.x; i < n; i += stride) {
    const u32 s = sym_bytes == 1 ? (u32)((const u8*)text)[i] : (u32)((const u16*)text)[i];
    if (!member[s]) atomicMin(best, (unsigned long long)i);
  }
}

cudaError_t launch_histogram(const void* text, u64 n, int sym_bytes, u64* hist, int sms,
                             cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const u64 work = sym_bytes == 1 ? (n >> 4) : (n >> 3);
  u64 blocks = (work + H_NT - 1) / H_NT;
  const u64 cap = (u64)sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  if (sym_bytes == 1)
    hist8_kernel<<<(unsigned)blocks, H_NT, 0, st>>>((const u8*)text, n, hist);
  else
    hist16_kernel<<<(unsigned)blocks, H_NT, 0, st>>>((const u16*)text, n, hist);
  return cudaGetLastError();
}

cudaError_t launch_first_outside(const void* text, u64 n, int sym_bytes, const u8* member,
                                 u64* best, int sms, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  u64 blocks = (n + H_NT - 1) / H_NT;
  const u64 cap = (u64)sms * 8;
  if (blocks > cap) blocks = cap;
  first_outside_kernel<<<(unsigned)blocks, H_NT, 0, st>>>(text, n, sym_bytes, member, best);
  return cudaGetLastError();
}

}  // namespace wt
