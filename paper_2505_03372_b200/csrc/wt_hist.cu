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
// u16: one CTA per SM, packed 16-bit shared counters for all 65536 symbols.
#include <atomic>
#include <mutex>
#include <cstdlib>
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

// u8 with per-block histograms (the level-0 block mode of the level kernel):
// a CTA takes whole 65536-symbol L1 blocks, each warp an 8 KiB slice of the
// block into its shared sub-histogram; thread i then folds bin i of the eight
// sub-histograms, writes it to block_hist[block][i] and keeps a running total
// for the text histogram.
constexpr int HB_BLOCK = 65536;
__global__ void __launch_bounds__(H_NT) hist8_blocks_kernel(const u8* __restrict__ text, u64 n,
                                                            u64* __restrict__ hist,
                                                            u32* __restrict__ block_hist) {
  __shared__ u32 sh[H_NT / 32][256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < (H_NT / 32) * 256; i += H_NT) (&sh[0][0])[i] = 0;
  __syncthreads();
  u32* mine = sh[warp];
  constexpr int SLICE = HB_BLOCK / (H_NT / 32);  // 8192 bytes per warp
  const u64 nblk = (n + HB_BLOCK - 1) / HB_BLOCK;
  u64 total = 0;
  for (u64 c = blockIdx.x; c < nblk; c += gridDim.x) {
    const u64 s0 = c * HB_BLOCK + (u64)warp * SLICE;
    const u8* p = text + s0;
    if (s0 + SLICE <= n) {
#pragma unroll 4
      for (int k = 0; k < SLICE / 512; ++k) {
        const uint4 q = ld_stream16(p + (k * 32 + lane) * 16);
        const u32 w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
#pragma unroll
          for (int b = 0; b < 4; ++b) atomicAdd(&mine[(w[i] >> (8 * b)) & 0xff], 1u);
        }
      }
    } else if (s0 < n) {
      for (u64 i = s0 + lane; i < n; i += 32) atomicAdd(&mine[text[i]], 1u);
    }
    __syncthreads();
    u32 v = 0;
#pragma unroll
    for (int w = 0; w < H_NT / 32; ++w) {
      v += sh[w][tid];
      sh[w][tid] = 0;
    }
    block_hist[c * 256 + tid] = v;
    total += v;
    __syncthreads();
  }
  if (total) atomicAdd(&hist[tid], total);
}

// ones of every L1 block for level 0 (symbols >= thr): a warp per block
__global__ void __launch_bounds__(256) block_l1_kernel(const u32* __restrict__ block_hist, u64 nblk,
                                                       u32 thr, u32* __restrict__ l1_counts) {
  const int lane = threadIdx.x & 31;
  for (u64 c = (u64)blockIdx.x * 8 + (threadIdx.x >> 5); c < nblk; c += (u64)gridDim.x * 8) {
    u32 s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const u32 b = j * 32 + lane;
      if (b >= thr) s += __ldg(block_hist + c * 256 + b);
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
    if (lane == 0) l1_counts[c] = s;
  }
}

constexpr int H16_NT = 1024;
// u16, one pass: each CTA counts ALL 65536 symbols of its chunks into packed
// 16-bit shared counters (two per 32-bit word, 128 KB, one CTA per SM) and
// reads its chunks once.  Counters spill 32768 to the global bin before they
// could carry into their neighbour (see `bump`).  Each CTA writes its counts
// as one row of `part`; hist16_fold_kernel adds the rows.
__global__ void __launch_bounds__(H16_NT, 1) hist16p_kernel(const u16* __restrict__ text, u64 n,
                                                            u64* __restrict__ hist,
                                                            u32* __restrict__ part,
                                                            u32* __restrict__ block_hi) {
  extern __shared__ u32 w2[];  // 32768 words = 65536 packed counters
  const int tid = threadIdx.x;
  for (int i = tid; i < 32768; i += H16_NT) w2[i] = 0;
  __syncthreads();
  // Each 16-bit field counts up to 0x7fff with bit 15 as a guard: the one
  // increment that takes a field from 0x7fff to 0x8000 (seen in the old value)
  // clears the guard again and moves 32768 to the global bin.  Increments
  // landing in between only raise the field above 0x8000, so no carry ever
  // reaches the neighbouring counter.
  auto bump = [&](u32 a) {
    const u32 sh = (a & 1u) * 16u;
    const u32 old = atomicAdd(&w2[a >> 1], 1u << sh);
    if (((old >> sh) & 0xffffu) == 0x7fffu) {
      atomicSub(&w2[a >> 1], 0x8000u << sh);
      atomicAdd(&hist[a], 32768ull);
    }
  };
  const u64 nvec = n >> 3;
  const u64 stride = (u64)gridDim.x * H16_NT;
  // warp-uniform trip count (the per-block reduction below needs every lane);
  // the next iteration's 16 bytes are loaded before this one's counters are
  // bumped (one CTA per SM: without the prefetch each thread had one load in
  // flight, 16 KiB per SM -- far too little to cover HBM latency)
  const uint4* t4 = reinterpret_cast<const uint4*>(text);
  u64 wv = (u64)blockIdx.x * H16_NT + (tid & ~31);
  uint4 qn = make_uint4(0, 0, 0, 0);
  if (wv + (tid & 31) < nvec) qn = __ldg(t4 + wv + (tid & 31));
  for (; wv < nvec; wv += stride) {
    const u64 v = wv + (tid & 31);
    uint4 q = qn;
    qn = wv + stride + (tid & 31) < nvec ? __ldg(t4 + wv + stride + (tid & 31)) : make_uint4(0, 0, 0, 0);
    if (v < nvec) {
      const u32 w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        bump(w[i] & 0xffffu);
        bump(w[i] >> 16);
      }
    }
    if (block_hi) {  // symbols >= 32768 per L1 block: a warp's 256 symbols share one block
      u32 hi = (u32)(__popc(q.x & 0x80008000u) + __popc(q.y & 0x80008000u)) +
               (u32)(__popc(q.z & 0x80008000u) + __popc(q.w & 0x80008000u));
#pragma unroll
      for (int d = 16; d; d >>= 1) hi += __shfl_xor_sync(0xffffffffu, hi, d);
      if ((tid & 31) == 0 && hi) atomicAdd(block_hi + ((wv << 3) >> 16), hi);
    }
  }
  if (blockIdx.x == 0)
    for (u64 i = (nvec << 3) + tid; i < n; i += H16_NT) {
      bump(text[i]);
      if (block_hi && text[i] >= 32768u) atomicAdd(block_hi + (i >> 16), 1u);
    }
  __syncthreads();
  u32* row = part + (u64)blockIdx.x * 65536;
  for (int i = tid; i < 32768; i += H16_NT) {
    const u32 x = w2[i];
    reinterpret_cast<uint2*>(row)[i] = make_uint2(x & 0xffffu, x >> 16);
  }
}
__global__ void hist16_fold_kernel(const u32* __restrict__ part, int rows, u64* __restrict__ hist) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= 65536) return;
  u64 s = 0;
  for (int r = 0; r < rows; ++r) s += part[(u64)r * 65536 + b];
  if (s) hist[b] += s;
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
                             cudaStream_t st, u32* block_hist) {
  if (n == 0) return cudaSuccess;
  if (sym_bytes == 1 && block_hist) {
    const u64 nblk = (n + HB_BLOCK - 1) / HB_BLOCK;
    const u64 blocks = nblk < (u64)sms * 8 ? nblk : (u64)sms * 8;
    hist8_blocks_kernel<<<(unsigned)blocks, H_NT, 0, st>>>((const u8*)text, n, hist, block_hist);
    return cudaGetLastError();
  }
  const u64 work = sym_bytes == 1 ? (n >> 4) : (n >> 3);
  u64 blocks = (work + H_NT - 1) / H_NT;
  const u64 cap = (u64)sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  if (sym_bytes == 1)
    hist8_kernel<<<(unsigned)blocks, H_NT, 0, st>>>((const u8*)text, n, hist);
  else {
    // the shared-memory opt-in is per device context: once per device (a
    // race only repeats the idempotent call)
    static std::atomic<bool> attr[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[dev].load(std::memory_order_acquire)) {
      cudaError_t e = cudaFuncSetAttribute(hist16p_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4);
      if (e != cudaSuccess) return e;
      if (dev >= 0 && dev < 64) attr[dev].store(true, std::memory_order_release);
    }
    u64 rows = (n / 8 + H16_NT - 1) / H16_NT;
    if (rows > (u64)sms) rows = (u64)sms;
    if (rows < 1) rows = 1;
    // the per-CTA count rows (rows x 256 KiB) live in one grow-only buffer per
    // device, reused in stream order through an event: a stream-ordered
    // allocation of it per build measured 10 ms .. 0.66 s host stalls in
    // later builds (C3 series in bench.py)
    struct PartCache {
      std::mutex mu;
      u32* p = nullptr;
      size_t bytes = 0;
      cudaEvent_t ev = nullptr;
    };
    static PartCache cache[64];
    PartCache& C = cache[(dev >= 0 && dev < 64) ? dev : 0];
    std::lock_guard<std::mutex> lk(C.mu);
    const size_t need = rows * 65536 * 4;
    cudaError_t e = cudaSuccess;
    if (!C.ev) e = cudaEventCreateWithFlags(&C.ev, cudaEventDisableTiming);
    if (e == cudaSuccess && C.bytes < need) {
      if (C.p) {
        cudaEventSynchronize(C.ev);
        cudaFree(C.p);
        C.p = nullptr;
        C.bytes = 0;
      }
      e = cudaMalloc(&C.p, need);
      if (e == cudaSuccess) C.bytes = need;
    }
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, C.ev, 0);  // the previous user is done
    if (e != cudaSuccess) return e;
    hist16p_kernel<<<(unsigned)rows, H16_NT, 32768 * 4, st>>>((const u16*)text, n, hist, C.p,
                                                              block_hist);
    hist16_fold_kernel<<<256, 256, 0, st>>>(C.p, (int)rows, hist);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaEventRecord(C.ev, st);
    return e;
  }
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

cudaError_t launch_block_l1(const u32* block_hist, u64 n_blocks, u32 thr, u32* l1_counts,
                            cudaStream_t st) {
  if (n_blocks == 0) return cudaSuccess;
  u64 blocks = (n_blocks + 7) / 8;
  if (blocks > 65535) blocks = 65535;
  block_l1_kernel<<<(unsigned)blocks, 256, 0, st>>>(block_hist, n_blocks, thr, l1_counts);
  return cudaGetLastError();
}

}  // namespace wt
