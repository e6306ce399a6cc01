// wt_ops.cu -- the reference's O(n) building blocks as stand-alone device ops.
//
// wt_construct fuses all of these into its own kernels (K1 histogram, the
// per-level partition + pack); the reference also exports them one by one
// (wtindex/__init__.py:61-73) and its tests call them directly, so the
// drop-in exposes each as a C-ABI entry over host arrays:
//
//   wt_minimal_alphabet  <- alphabet.minimal_alphabet      (alphabet.py:94-111)
//   wt_map_text          <- AlphabetMap.map_text           (alphabet.py:76-84)
//   wt_encode_histogram  <- alphabet.encode_and_histogram  (alphabet.py:210-242)
//   wt_sort_by_prefix    <- wtree.stable_sort_by_prefix    (wtree.py:92-100)
//   wt_fill_level        <- wtree.fill_level / BitArray.fill_region packing
//                           (wtree.py:103-107, bitvec.py:119-151)
//
// All are HBM-streaming kernels; the stable sort is an LSD sequence of
// stable binary splits (one popcount scan per key bit), which needs no
// per-bucket state for the up-to-16-bit prefix keys.
#include <algorithm>
#include <string>
#include <vector>

#include "wt_common.cuh"
#include "wt_host.h"
#include "wt_kernels.h"

using namespace wt;

namespace {

constexpr int OP_NT = 256;
constexpr u32 kLutAbsent = 1u << 16;   // lut entry flag: symbol not in the alphabet
constexpr u64 kNone = ~0ull;

// first index i with flag set, warp-aggregated
__device__ __forceinline__ void first_bad(bool bad, u64 i, u64* best) {
  const unsigned m = __ballot_sync(__activemask(), bad);
  if (m && bad && (threadIdx.x & 31) == __ffs(m) - 1) atomicMin(best, i);
}

template <typename T>
__global__ void __launch_bounds__(OP_NT) map_kernel(const T* __restrict__ text, u64 n,
                                                    const u32* __restrict__ lut,
                                                    u16* __restrict__ out, u64* best) {
  const u64 stride = (u64)gridDim.x * OP_NT;
  for (u64 base = (u64)blockIdx.x * OP_NT; base < n; base += stride) {
    const u64 i = base + threadIdx.x;
    u32 v = 0;
    if (i < n) {
      v = lut[text[i]];
      if (!(v & kLutAbsent)) out[i] = (u16)v;
    }
    first_bad(i < n && (v & kLutAbsent), i, best);
  }
}

__global__ void __launch_bounds__(OP_NT) encode_kernel(const u16* __restrict__ ids, u64 n,
                                                       const u16* __restrict__ values, u32 sigma,
                                                       u16* __restrict__ enc, u64* best) {
  const u64 stride = (u64)gridDim.x * OP_NT;
  for (u64 base = (u64)blockIdx.x * OP_NT; base < n; base += stride) {
    const u64 i = base + threadIdx.x;
    bool bad = false;
    if (i < n) {
      const u32 id = ids[i];
      bad = id >= sigma;
      enc[i] = bad ? 0 : values[id];
    }
    first_bad(bad, i, best);
  }
}

// ---- stable binary split on one bit: tile = OP_NT threads x 16 elements ----
constexpr int SP_PER = 16;
constexpr int SP_TILE = OP_NT * SP_PER;

__device__ __forceinline__ u32 block_exclusive_scan(u32 v, u32* sh, u32* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u32 x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    u32 w = lane < OP_NT / 32 ? sh[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < OP_NT / 32) sh[lane] = w;
  }
  __syncthreads();
  const u32 before = (warp ? sh[warp - 1] : 0) + x - v;
  if (total) *total = sh[OP_NT / 32 - 1];
  __syncthreads();
  return before;
}

__global__ void __launch_bounds__(OP_NT) split_count_kernel(const u16* __restrict__ in, u64 n,
                                                            u32 bit, u32* __restrict__ tile_ones) {
  __shared__ u32 sh[OP_NT / 32];
  const u64 t0 = (u64)blockIdx.x * SP_TILE + (u64)threadIdx.x * SP_PER;
  u32 c = 0;
  for (int j = 0; j < SP_PER; ++j)
    if (t0 + j < n) c += (in[t0 + j] >> bit) & 1;
  u32 tot;
  block_exclusive_scan(c, sh, &tot);
  if (threadIdx.x == 0) tile_ones[blockIdx.x] = tot;
}

// exclusive prefix of the tile counts (one CTA; tiles <= 2^20 at n <= 2^32)
__global__ void __launch_bounds__(1024) split_scan_kernel(const u32* __restrict__ tile_ones,
                                                          u64 n_tiles, u64* __restrict__ prefix) {
  __shared__ u64 sh[1024];
  __shared__ u64 carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (u64 base = 0; base < n_tiles; base += 1024) {
    const u64 i = base + threadIdx.x;
    const u64 v = i < n_tiles ? tile_ones[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {
      const u64 y = threadIdx.x >= (unsigned)d ? sh[threadIdx.x - d] : 0;
      __syncthreads();
      sh[threadIdx.x] += y;
      __syncthreads();
    }
    if (i < n_tiles) prefix[i] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) prefix[n_tiles] = carry;
}

__global__ void __launch_bounds__(OP_NT) split_scatter_kernel(const u16* __restrict__ in, u64 n,
                                                              u32 bit, const u64* __restrict__ prefix,
                                                              u64 n_tiles, u16* __restrict__ out) {
  __shared__ u32 sh[OP_NT / 32];
  const u64 t0 = (u64)blockIdx.x * SP_TILE + (u64)threadIdx.x * SP_PER;
  u16 v[SP_PER];
  u32 c = 0;
#pragma unroll
  for (int j = 0; j < SP_PER; ++j) {
    v[j] = t0 + j < n ? in[t0 + j] : 0;
    c += (v[j] >> bit) & 1;
  }
  const u64 zeros_total = n - prefix[n_tiles];
  u64 ones_before = prefix[blockIdx.x] + block_exclusive_scan(c, sh, nullptr);
#pragma unroll
  for (int j = 0; j < SP_PER; ++j) {
    const u64 i = t0 + j;
    if (i >= n) break;
    if ((v[j] >> bit) & 1) {
      out[zeros_total + ones_before] = v[j];
      ++ones_before;
    } else {
      out[i - ones_before] = v[j];
    }
  }
}

// bit `bit` of each code, LSB-first into u64 words (as two u32 halves)
__global__ void __launch_bounds__(OP_NT) pack_bits_kernel(const u16* __restrict__ in, u64 count,
                                                          u32 bit, u32* __restrict__ out32,
                                                          u64 n32) {
  const u64 stride = (u64)gridDim.x * OP_NT;
  for (u64 i = (u64)blockIdx.x * OP_NT + threadIdx.x; (i >> 5) < n32; i += stride) {
    const bool b = i < count && ((in[i] >> bit) & 1);
    const u32 m = __ballot_sync(0xffffffffu, b);
    if ((threadIdx.x & 31) == 0) out32[i >> 5] = m;
  }
}

unsigned grid_for(u64 n, int device) {
  const u64 blocks = (n + OP_NT - 1) / OP_NT;
  const u64 cap = (u64)sm_count(device) * 8;
  return (unsigned)std::max<u64>(1, std::min(blocks, cap));
}

// device buffers of one call, freed (stream-ordered) on every exit path
struct Bufs {
  cudaStream_t st = nullptr;
  std::vector<void*> ptrs;
  ~Bufs() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  }
  template <typename T>
  int get(T** p, u64 count) {
    CU(cudaMallocAsync((void**)p, std::max<u64>(count, 1) * sizeof(T), st));
    ptrs.push_back(*p);
    return WT_OK;
  }
};

int open_call(Bufs& B, int device) {
  TRY(setup_device(device));
  CU(cudaStreamCreateWithFlags(&B.st, cudaStreamNonBlocking));
  return WT_OK;
}

// raw text -> minimal ids through a lut of nb entries
int map_through(Bufs& B, const void* text, u64 n, int sym_bytes, const std::vector<u32>& lut,
                uint16_t* ids_out, u64* bad_out, int device) {
  u8* dt;
  u32* dl;
  u16* di;
  u64* dbad;
  TRY(B.get(&dt, n * sym_bytes));
  TRY(B.get(&dl, lut.size()));
  TRY(B.get(&di, n));
  TRY(B.get(&dbad, 1));
  CU(cudaMemcpyAsync(dt, text, n * sym_bytes, cudaMemcpyHostToDevice, B.st));
  CU(cudaMemcpyAsync(dl, lut.data(), lut.size() * 4, cudaMemcpyHostToDevice, B.st));
  CU(cudaMemsetAsync(dbad, 0xff, 8, B.st));
  if (sym_bytes == 1)
    map_kernel<u8><<<grid_for(n, device), OP_NT, 0, B.st>>>(dt, n, dl, di, dbad);
  else
    map_kernel<u16><<<grid_for(n, device), OP_NT, 0, B.st>>>((const u16*)dt, n, dl, di, dbad);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(ids_out, di, n * 2, cudaMemcpyDeviceToHost, B.st));
  CU(cudaMemcpyAsync(bad_out, dbad, 8, cudaMemcpyDeviceToHost, B.st));
  CU(cudaStreamSynchronize(B.st));
  return WT_OK;
}

u32 sym_at(const void* text, int sym_bytes, u64 i) {
  return sym_bytes == 1 ? ((const u8*)text)[i] : ((const u16*)text)[i];
}

}  // namespace

extern "C" int wt_minimal_alphabet(const void* text, uint64_t n, int sym_bytes, int device,
                                   uint16_t* ids_out, uint16_t* symbols_out,
                                   uint32_t* sigma_out) {
  if (n == 0) return fail(WT_ERR_BUILD, "text must be non-empty");
  if (sym_bytes != 1 && sym_bytes != 2) return fail(WT_ERR_ARG, "sym_bytes must be 1 or 2");
  if (!text || !ids_out || !symbols_out || !sigma_out) return fail(WT_ERR_ARG, "NULL pointer");
  Bufs B;
  TRY(open_call(B, device));
  const int nb = sym_bytes == 1 ? 256 : 65536;
  u8* dt;
  u64* dh;
  TRY(B.get(&dt, n * sym_bytes));
  TRY(B.get(&dh, nb));
  CU(cudaMemcpyAsync(dt, text, n * sym_bytes, cudaMemcpyHostToDevice, B.st));
  CU(cudaMemsetAsync(dh, 0, nb * 8, B.st));
  CU(launch_histogram(dt, n, sym_bytes, dh, sm_count(device), B.st));
  std::vector<uint64_t> hist(nb);
  CU(cudaMemcpyAsync(hist.data(), dh, nb * 8, cudaMemcpyDeviceToHost, B.st));
  CU(cudaStreamSynchronize(B.st));
  std::vector<u32> lut(nb, kLutAbsent);
  uint32_t sigma = 0;
  for (int s = 0; s < nb; ++s)
    if (hist[s]) {
      symbols_out[sigma] = (uint16_t)s;
      lut[s] = sigma++;
    }
  *sigma_out = sigma;
  u64 bad = kNone;
  TRY(map_through(B, text, n, sym_bytes, lut, ids_out, &bad, device));
  if (bad != kNone) return fail(WT_ERR_CUDA, "minimal alphabet: histogram and map disagree");
  return WT_OK;
}

extern "C" int wt_map_text(const void* text, uint64_t n, int sym_bytes, const uint16_t* symbols,
                           uint32_t sigma, int device, uint16_t* ids_out) {
  g_err_index = -1;
  if (sym_bytes != 1 && sym_bytes != 2) return fail(WT_ERR_ARG, "sym_bytes must be 1 or 2");
  if (sigma > 65536) return fail(WT_ERR_BUILD, "alphabet larger than 2^16");
  if (n == 0) return WT_OK;
  if (!text || !ids_out || (sigma && !symbols)) return fail(WT_ERR_ARG, "NULL pointer");
  const int nb = sym_bytes == 1 ? 256 : 65536;
  std::vector<u32> lut(nb, kLutAbsent);
  for (uint32_t i = 0; i < sigma; ++i)
    if (symbols[i] < nb) lut[symbols[i]] = i;
  Bufs B;
  TRY(open_call(B, device));
  u64 bad = kNone;
  TRY(map_through(B, text, n, sym_bytes, lut, ids_out, &bad, device));
  if (bad != kNone) {
    g_err_index = (int64_t)bad;
    return fail(WT_ERR_SYMBOL, "symbol " + std::to_string(sym_at(text, sym_bytes, bad)) +
                                   " at position " + std::to_string(bad) +
                                   " is not in the alphabet");
  }
  return WT_OK;
}

extern "C" int wt_encode_histogram(const uint16_t* ids, uint64_t n, const uint16_t* code_values,
                                   uint32_t sigma, int device, uint16_t* encoded_out,
                                   int64_t* hist_out) {
  g_err_index = -1;
  if (sigma == 0 || sigma > 65536) return fail(WT_ERR_ARG, "sigma must lie in [1, 2^16]");
  if (!code_values || !hist_out || (n && (!ids || !encoded_out)))
    return fail(WT_ERR_ARG, "NULL pointer");
  if (n == 0) {
    std::fill(hist_out, hist_out + sigma, 0);
    return WT_OK;
  }
  Bufs B;
  TRY(open_call(B, device));
  u16 *di, *dv, *de;
  u64 *dh, *dbad;
  TRY(B.get(&di, n));
  TRY(B.get(&dv, sigma));
  TRY(B.get(&de, n));
  TRY(B.get(&dh, 65536));
  TRY(B.get(&dbad, 1));
  CU(cudaMemcpyAsync(di, ids, n * 2, cudaMemcpyHostToDevice, B.st));
  CU(cudaMemcpyAsync(dv, code_values, sigma * 2, cudaMemcpyHostToDevice, B.st));
  CU(cudaMemsetAsync(dh, 0, 65536 * 8, B.st));
  CU(cudaMemsetAsync(dbad, 0xff, 8, B.st));
  encode_kernel<<<grid_for(n, device), OP_NT, 0, B.st>>>(di, n, dv, sigma, de, dbad);
  CU(cudaGetLastError());
  CU(launch_histogram(di, n, 2, dh, sm_count(device), B.st));  // ids as 16-bit symbols
  std::vector<uint64_t> hist(65536);
  u64 bad = kNone;
  CU(cudaMemcpyAsync(hist.data(), dh, 65536 * 8, cudaMemcpyDeviceToHost, B.st));
  CU(cudaMemcpyAsync(&bad, dbad, 8, cudaMemcpyDeviceToHost, B.st));
  CU(cudaMemcpyAsync(encoded_out, de, n * 2, cudaMemcpyDeviceToHost, B.st));
  CU(cudaStreamSynchronize(B.st));
  if (bad != kNone) {
    g_err_index = (int64_t)bad;
    return fail(WT_ERR_SYMBOL, "symbol id " + std::to_string(ids[bad]) + " outside [0, " +
                                   std::to_string(sigma) + ")");
  }
  for (uint32_t s = 0; s < sigma; ++s) hist_out[s] = (int64_t)hist[s];
  return WT_OK;
}

extern "C" int wt_sort_by_prefix(const uint16_t* codes, uint64_t n, uint32_t shift, int device,
                                 uint16_t* out) {
  if (n == 0) return WT_OK;
  if (!codes || !out) return fail(WT_ERR_ARG, "NULL pointer");
  Bufs B;
  TRY(open_call(B, device));
  const u64 n_tiles = (n + SP_TILE - 1) / SP_TILE;
  if (n_tiles > (1ull << 22)) return fail(WT_ERR_ARG, "sequence too long for wt_sort_by_prefix");
  u16 *a, *b;
  u32* cnt;
  u64* pre;
  TRY(B.get(&a, n));
  TRY(B.get(&b, n));
  TRY(B.get(&cnt, n_tiles));
  TRY(B.get(&pre, n_tiles + 1));
  CU(cudaMemcpyAsync(a, codes, n * 2, cudaMemcpyHostToDevice, B.st));
  // key = code >> shift: an LSD pass per key bit, each a stable split
  for (uint32_t bit = shift; bit < 16; ++bit) {
    split_count_kernel<<<(unsigned)n_tiles, OP_NT, 0, B.st>>>(a, n, bit, cnt);
    split_scan_kernel<<<1, 1024, 0, B.st>>>(cnt, n_tiles, pre);
    split_scatter_kernel<<<(unsigned)n_tiles, OP_NT, 0, B.st>>>(a, n, bit, pre, n_tiles, b);
    CU(cudaGetLastError());
    std::swap(a, b);
  }
  CU(cudaMemcpyAsync(out, a, n * 2, cudaMemcpyDeviceToHost, B.st));
  CU(cudaStreamSynchronize(B.st));
  return WT_OK;
}

extern "C" int wt_fill_level(const uint16_t* codes, uint64_t count, uint32_t bit, int device,
                             uint64_t* words_out) {
  if (bit >= 16) return fail(WT_ERR_ARG, "bit must lie in [0, 16)");
  if (count == 0) return WT_OK;
  if (!codes || !words_out) return fail(WT_ERR_ARG, "NULL pointer");
  Bufs B;
  TRY(open_call(B, device));
  const u64 n_words = (count + 63) / 64, n32 = 2 * n_words;
  u16* dc;
  u32* dw;
  TRY(B.get(&dc, count));
  TRY(B.get(&dw, n32));
  CU(cudaMemcpyAsync(dc, codes, count * 2, cudaMemcpyHostToDevice, B.st));
  pack_bits_kernel<<<grid_for(n32 * 32, device), OP_NT, 0, B.st>>>(dc, count, bit, dw, n32);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(words_out, dw, n_words * 8, cudaMemcpyDeviceToHost, B.st));
  CU(cudaStreamSynchronize(B.st));
  return WT_OK;
}
