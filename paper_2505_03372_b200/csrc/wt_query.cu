// wt_query.cu -- Q kernels: batched access / rank / select, one thread per query.
//
// The reference walks node intervals [start, end) with cum_hist offsets and
// node_rank0 lookups (wtree.py:200-279 scalar, :283-375 bulk).  Here a node is
// addressed by its code prefix (key) and one NodeEnt holds both position
// offsets, so each level is exactly one rank (or select) plus one 24-byte
// table read (verified equal to _access_id/_rank_id/_select_id):
//   access: p' = bit ? rank1(p) + one_base : rank0(p) + zero_base,
//           stop when child `bit` of the node is a leaf (width-1 interval);
//   rank:   the same walk along the code of c, result p_len - cum_hist[c];
//   select: bottom-up, p = select_bit(p' - base + 1), from cum_hist[c]+k-1.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include "wt_common.cuh"
#include "wt_kernels.h"
#include "wt_rs.cuh"

namespace wt {

#ifndef WT_Q_NT
#define WT_Q_NT 128  // 128 vs 256 vs 512 threads: select -1.3 %, others flat
#endif
constexpr int Q_NT = WT_Q_NT;
#ifndef WT_QS_QPT
#define WT_QS_QPT 1  // A/B on B200: 2 / 4 / 8 measured 0.2-1.5 % slower
#endif
constexpr int QS_QPT = WT_QS_QPT;  // queries per thread in the sort's key / scatter kernels
#ifndef WT_QS_RANK
#define WT_QS_RANK 0  // A/B on B200: 1 measured slower (C2 sorted batches +3.5 % time)
#endif
constexpr bool QS_RANK = WT_QS_RANK != 0;  // ranks in bucket from the count pass

// a sorted batch (WT_F_SORT) carries (argument | id << 48) per query
// unpack the sorted batch (rank / select): id and argument
__device__ __forceinline__ void qsort_unpack(i64 packed, u32& c, u64& a) {
  c = (u32)((u64)packed >> 48);
  a = (u64)packed & ((1ull << 48) - 1);
}


// Query batch contract (BatchRunner.run, batch.py:112-148 + :152-239):
//   kValidate: `ids` holds ORIGINAL symbol values; each thread maps its symbol
//   through sym2id and checks its argument range; an invalid query records
//   its index with atomicMin(bad) and produces no result.  The host raises
//   BatchError(first bad index) and discards the batch, exactly as the
//   reference validates before processing.
//   kOut (access): 1 / 2 = decoded original symbol (batch._decode),
//                  8 = minimal id as int64 (access_ids_bulk).
template <int kOut, bool kValidate>
__global__ void __launch_bounds__(Q_NT) access_kernel(const __grid_constant__ TreeDev T,
                                                      const i64* __restrict__ pos,
                                                      void* __restrict__ out, u64 m, u64 base,
                                                      u64* __restrict__ bad,
                                                      bool packed,
                                                      const u32* __restrict__ pos32 = nullptr) {
  const u64 q = (u64)blockIdx.x * Q_NT + threadIdx.x;
  if (q >= m) return;
  const u64 i = q;
  u64 p = pos32 ? (u64)__ldg(pos32 + q) : (u64)ld_stream_i64(pos + q, l2_evict_first_policy());
  if (packed) p = min(p & ((1ull << 48) - 1), T.n - 1);  // sorted batch: clamped in range
  if (kValidate && p >= T.n) {  // negative positions wrap to huge values
    atomicMin(bad, base + i);
    return;
  }
  u32 key = 0;
  int id = 0;
  for (u32 l = 0; l < T.L; ++l) {
    const NodeEnt* ne = T.lv[l].nodes + key;
    u32 bit;
    const u64 r1 = qrank1_bit(T.ql[l], p, bit);  // one 64-byte line per level
    const int leaf = __ldg(&ne->leaf[bit]);
    if (leaf >= 0) {
      id = leaf;
      break;
    }
    p = bit ? r1 + (u64)__ldg(&ne->one_base) : (p - r1) + (u64)__ldg(&ne->zero_base);
    key = (key << 1) | bit;
  }
  if (kOut == 8) {
    reinterpret_cast<i64*>(out)[i] = id;
  } else {
    const u16 sym = __ldg(T.symbols + id);
    if (kOut == 1)
      reinterpret_cast<u8*>(out)[i] = (u8)sym;
    else
      reinterpret_cast<u16*>(out)[i] = sym;
  }
}

template <bool kValidate>
__device__ __forceinline__ bool symbol_id(const TreeDev& T, i64 raw, u32& c) {
  if (!kValidate) {
    c = (u32)raw;
    return true;
  }
  if (raw < 0 || raw > 65535) return false;
  const int id = __ldg(T.sym2id + raw);
  if (id < 0) return false;
  c = (u32)id;
  return true;
}

template <bool kValidate>
__global__ void __launch_bounds__(Q_NT) rank_kernel(const __grid_constant__ TreeDev T,
                                                    const i64* __restrict__ ids,
                                                    const i64* __restrict__ pos,
                                                    i64* __restrict__ out, u64 m, u64 base,
                                                    u64* __restrict__ bad,
                                                    bool packed, u32* __restrict__ out32 = nullptr) {
  const u64 q = (u64)blockIdx.x * Q_NT + threadIdx.x;
  if (q >= m) return;
  const u64 i = q;
  u32 c;
  u64 p;
  const u64 pol = l2_evict_first_policy();
  if (packed) {  // sorted batch: packed (position | id << 48), clamped in range
    qsort_unpack(ld_stream_i64(pos + q, pol), c, p);
    p = min(p, T.n);
  } else {
    p = (u64)pos[q];
    if (!symbol_id<kValidate>(T, ids[q], c) || (kValidate && p > T.n)) {
      atomicMin(bad, base + i);
      return;
    }
  }
  const u32 cd = __ldg(T.id_code + c);
  const u32 code = cd & 0xffffu, len = cd >> 16;
  for (u32 l = 0; l < len; ++l) {
    const u32 bit = (code >> (T.L - 1 - l)) & 1u;
    const u32 key = code >> (T.L - l);
    const NodeEnt* ne = T.lv[l].nodes + key;
    const u64 base = bit ? (u64)__ldg(&ne->one_base) : (u64)__ldg(&ne->zero_base);
    const u64 r1 = qrank1(T.ql[l], p);
    p = (bit ? r1 : p - r1) + base;
  }
  const u64 r = p - (u64)__ldg(T.cum + c);
  if (out32)  // sorted-order results of a text below 2^32: 4 bytes (half the gather's working set)
    out32[i] = (u32)r;
  else
    st_stream_i64(out + i, (i64)r, pol);
}

template <bool kValidate>
__global__ void __launch_bounds__(Q_NT) select_kernel(const __grid_constant__ TreeDev T,
                                                      const i64* __restrict__ ids,
                                                      const i64* __restrict__ ks,
                                                      i64* __restrict__ out, u64 m, int rate_log,
                                                      u64 base, u64* __restrict__ bad,
                                                      bool packed,
                                                      const u32* __restrict__ ks32 = nullptr,
                                                      u32 kbits = 0, u32* __restrict__ out32 = nullptr) {
  const u64 q = (u64)blockIdx.x * Q_NT + threadIdx.x;
  if (q >= m) return;
  const u64 i = q;
  u32 c;
  i64 k;
  const u64 pol = l2_evict_first_policy();
  if (packed) {  // sorted batch: packed (ordinal | id << 48 or << kbits), clamped in range
    u64 a;
    if (ks32) {
      const u32 v = __ldg(ks32 + q);
      c = v >> kbits;
      a = v & ((1u << kbits) - 1u);
    } else {
      qsort_unpack(ld_stream_i64(ks + q, pol), c, a);
    }
    const i64 occ = __ldg(T.cum + c + 1) - __ldg(T.cum + c);
    k = min(max((i64)a, (i64)1), max(occ, (i64)1));
  } else if (k = ks[q], !symbol_id<kValidate>(T, ids[q], c) ||
      (kValidate && (k < 1 || k > __ldg(T.cum + c + 1) - __ldg(T.cum + c)))) {
    atomicMin(bad, base + i);
    return;
  }
  const u32 cd = __ldg(T.id_code + c);
  const u32 code = cd & 0xffffu, len = cd >> 16;
  u64 p = (u64)__ldg(T.cum + c) + (u64)k - 1;
  for (int l = (int)len - 1; l >= 0; --l) {
    const u32 bit = (code >> (T.L - 1 - l)) & 1u;
    const u32 key = code >> (T.L - l);
    const NodeEnt* ne = T.lv[l].nodes + key;
    if (bit)
      p = qselect<true>(T.ql[l], p - (u64)__ldg(&ne->one_base) + 1);
    else
      p = qselect<false>(T.ql[l], p - (u64)__ldg(&ne->zero_base) + 1);
  }
  if (out32)
    out32[i] = (u32)p;
  else
    st_stream_i64(out + i, (i64)p, pol);
}

template <bool V>
static void launch_q(const TreeDev& T, int kind, int out_kind, const i64* ids, const i64* args,
                     void* out, u64 m, int rate_log, u64 base, u64* bad, bool packed,
                     unsigned blocks, cudaStream_t st) {
  switch (kind) {
    case 0:
      if (out_kind == 8)
        access_kernel<8, V><<<blocks, Q_NT, 0, st>>>(T, args, out, m, base, bad, packed);
      else if (out_kind == 1)
        access_kernel<1, V><<<blocks, Q_NT, 0, st>>>(T, args, out, m, base, bad, packed);
      else
        access_kernel<2, V><<<blocks, Q_NT, 0, st>>>(T, args, out, m, base, bad, packed);
      break;
    case 1:
      rank_kernel<V><<<blocks, Q_NT, 0, st>>>(T, ids, args, (i64*)out, m, base, bad, packed);
      break;
    default:
      select_kernel<V><<<blocks, Q_NT, 0, st>>>(T, ids, args, (i64*)out, m, rate_log, base, bad, packed);
      break;
  }
}

cudaError_t launch_query(const TreeDev& T, int kind, int out_kind, bool validate, const i64* ids,
                         const i64* args, void* out, u64 m, int rate_log, u64 base, u64* bad,
                         cudaStream_t st, bool packed) {
  if (m == 0) return cudaSuccess;
  if (kind < 0 || kind > 2) return cudaErrorInvalidValue;
  const u64 blocks = (m + Q_NT - 1) / Q_NT;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidValue;
  if (validate)
    launch_q<true>(T, kind, out_kind, ids, args, out, m, rate_log, base, bad, packed, (unsigned)blocks, st);
  else
    launch_q<false>(T, kind, out_kind, ids, args, out, m, rate_log, base, bad, packed, (unsigned)blocks, st);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// sort_queries_by_symbol on the device (batch.py:61-75):
// a counting sort into 2^10 .. 2^20 buckets (about 128 queries each) --
// (coarse text position, symbol id) for rank, (coarse estimated position
// k * n / occ, symbol id) for select, coarse position for access -- so
// queries that walk the same nodes and nearby lines run side by side.
// The query kernel writes results in sorted order; qunsort_kernel gathers
// them back into query order through each query's slot.  Validation happens
// here, before anything runs (batch.py:112-148).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(Q_NT) qsort_key_kernel(const __grid_constant__ TreeDev T, int kind,
                                                         const i64* __restrict__ ids,
                                                         const i64* __restrict__ args, u64 m,
                                                         bool validate, u32 sym_bits,
                                                         u32 arg_shift, u32 nb, u32* __restrict__ bucket_of,
                                                         u32* __restrict__ hist, u64 base,
                                                         u64* __restrict__ bad,
                                                         u32* __restrict__ rank_of) {
  // QS_QPT queries per thread, Q_NT apart: every load is issued before the
  // first query's dependent table reads
  const u64 i0 = (u64)blockIdx.x * QS_QPT * Q_NT + threadIdx.x;
  u64 aq[QS_QPT];
  i64 rq[QS_QPT];
#pragma unroll
  for (int j = 0; j < QS_QPT; ++j) {
    const u64 i = i0 + (u64)j * Q_NT;
    aq[j] = i < m ? (u64)__ldg(args + i) : 0ull;
    rq[j] = i < m && kind != 0 ? __ldg(ids + i) : 0ll;
  }
#pragma unroll
  for (int j = 0; j < QS_QPT; ++j) {
  const u64 i = i0 + (u64)j * Q_NT;
  if (i >= m) return;
  const u64 a = aq[j];
  u32 bucket = 0;
  bool ok = true;
  if (kind == 0) {
    ok = !validate || a < T.n;
    bucket = ok ? (u32)(a >> arg_shift) : 0u;
  } else {
    u32 c = 0;
    if (validate) {
      const i64 raw = rq[j];
      const int id = (raw < 0 || raw > 65535) ? -1 : __ldg(T.sym2id + raw);
      ok = id >= 0;
      c = ok ? (u32)id : 0u;
    } else {
      const i64 raw = rq[j];
      c = raw < 0 ? 0u : (u32)min(raw, (i64)T.sigma - 1);  // memory safety only
    }
    if (ok && validate) {
      if (kind == 1) ok = a <= T.n;
      else ok = a >= 1 && (i64)a <= __ldg(T.cum + c + 1) - __ldg(T.cum + c);
    }
    // Position-block major, symbol minor: consecutive buckets walk the same
    // stretch of the text -- and so of every level's nodes -- for all
    // symbols, which keeps each level's lines in L2 while the stretch runs
    // (symbol-major buckets re-read the upper levels once per symbol).
    // select orders by the estimated text position k * n / occ(c).  The low
    // bits are the minimal id: the scatter recovers it.
    if (ok) {
      u64 est = a;
      if (kind == 2) {
        const i64 occ = __ldg(T.cum + c + 1) - __ldg(T.cum + c);
        const float f = (float)(a - 1) * ((float)T.n / (float)(occ > 0 ? occ : 1));
        est = min((u64)f, T.n);
      }
      bucket = ((u32)(est >> arg_shift) << sym_bits) | c;
    }
  }
  if (!ok) atomicMin(bad, base + i);
  // unvalidated callers promise ids < sigma and in-range arguments; clamp
  // anyway so a broken promise cannot index past the bucket table
  bucket = min(bucket, nb - 1u);
  bucket_of[i] = bucket;
  // WT_QS_RANK: the count's returning atomic hands each query its rank in
  // the bucket, so the scatter needs no atomics of its own (one returning
  // atomic per query instead of a reduction plus a returning atomic)
  if (QS_RANK)
    rank_of[i] = atomicAdd(hist + bucket, 1u);
  else
    atomicAdd(hist + bucket, 1u);
  }
}

// exclusive scan of the bucket counts in place, 4096 buckets per CTA (1024
// threads x uint4): pass 1 writes each CTA's total, pass 2 adds the totals of
// the CTAs before it (<= 256 of them) and scans its own buckets
constexpr int QS_PER_CTA = 4096;
__device__ __forceinline__ u32 qs_block_sum(u32 v, u32* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  __syncthreads();
  if (lane == 0) wsum[warp] = v;
  __syncthreads();
  u32 t = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0u;
#pragma unroll
  for (int d = 16; d; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
  return t;
}
__device__ __forceinline__ uint4 qs_load(const u32* hist, u32 nb, u32 i4) {
  if ((i4 + 1) * 4 <= nb) return reinterpret_cast<const uint4*>(hist)[i4];
  uint4 v = make_uint4(0, 0, 0, 0);
  if (i4 * 4 + 0 < nb) v.x = hist[i4 * 4 + 0];
  if (i4 * 4 + 1 < nb) v.y = hist[i4 * 4 + 1];
  if (i4 * 4 + 2 < nb) v.z = hist[i4 * 4 + 2];
  return v;
}
__global__ void __launch_bounds__(1024) qsort_scan_partial_kernel(const u32* __restrict__ hist, u32 nb,
                                                                  u32* __restrict__ partial) {
  __shared__ u32 wsum[32];
  const uint4 v = qs_load(hist, nb, blockIdx.x * (QS_PER_CTA / 4) + threadIdx.x);
  const u32 t = qs_block_sum(v.x + v.y + v.z + v.w, wsum);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}
__global__ void __launch_bounds__(1024) qsort_scan_final_kernel(u32* __restrict__ hist, u32 nb,
                                                                const u32* __restrict__ partial) {
  __shared__ u32 wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 off = qs_block_sum(tid < (int)blockIdx.x ? partial[tid] : 0u, wsum);
  const u32 i4 = blockIdx.x * (QS_PER_CTA / 4) + tid;
  const uint4 v = qs_load(hist, nb, i4);
  const u32 sum = v.x + v.y + v.z + v.w;
  u32 inc = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  __syncthreads();
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    u32 t = wsum[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, t, d);
      if (lane >= d) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  u32 run = off + (warp ? wsum[warp - 1] : 0u) + inc - sum;
  const u32 e[4] = {v.x, v.y, v.z, v.w};
  if ((i4 + 1) * 4 <= nb) {  // one 16-byte store per thread (coalesced)
    const u32 o0 = run, o1 = o0 + v.x, o2 = o1 + v.y, o3 = o2 + v.z;
    reinterpret_cast<uint4*>(hist)[i4] = make_uint4(o0, o1, o2, o3);
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (i4 * 4 + j < nb) hist[i4 * 4 + j] = run;
    run += e[j];
  }
}

// the sorted batch: (argument | id << 48) -- 8 bytes of scattered writes per
// query (ids ride in the argument's top bits: positions / ordinals stay below
// 2^48; the id is the bucket's top bits) -- and, in query order, the slot each
// query went to (a coalesced write: the results come back by a gather)
__global__ void __launch_bounds__(Q_NT) qsort_scatter_kernel(const u32* __restrict__ bucket_of,
                                                             bool with_id, u32 sym_bits,
                                                             const i64* __restrict__ args, u64 m,
                                                             u32* __restrict__ cursor,
                                                             i64* __restrict__ sargs,
                                                             u32* __restrict__ sargs32, u32 kbits,
                                                             u32* __restrict__ slot_of) {
  // L2 policy: the streams (bucket_of, args in; slot_of out) evict first, the
  // scattered sorted-batch stores evict last -- a bucket's 32-byte sectors
  // fill up over the whole kernel and a partial sector written back costs a
  // DRAM read-modify-write (-10 % kernel time, -11 % DRAM writes)
  u64 pf, pl;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  // QS_QPT queries per thread, Q_NT apart: their returning cursor atomics are
  // independent, so a thread keeps QS_QPT of them in flight
  const u64 i0 = (u64)blockIdx.x * QS_QPT * Q_NT + threadIdx.x;
  u32 bq[QS_QPT], sq[QS_QPT];
  u64 aq[QS_QPT];
#pragma unroll
  for (int j = 0; j < QS_QPT; ++j) {
    const u64 i = i0 + (u64)j * Q_NT;
    bq[j] = 0; aq[j] = 0;
    if (i < m) {
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                   : "=r"(bq[j]) : "l"(bucket_of + i), "l"(pf));
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
                   : "=l"(aq[j]) : "l"(args + i), "l"(pf));
    }
  }
#pragma unroll
  for (int j = 0; j < QS_QPT; ++j)
    if (i0 + (u64)j * Q_NT < m)
      sq[j] = QS_RANK ? __ldg(cursor + bq[j]) + slot_of[i0 + (u64)j * Q_NT]
                      : atomicAdd(cursor + bq[j], 1u);
#pragma unroll
  for (int j = 0; j < QS_QPT; ++j) {
  const u64 i = i0 + (u64)j * Q_NT;
  if (i >= m) return;
  const u32 b = bq[j], slot = sq[j];
  const u64 a = aq[j] & ((1ull << 48) - 1);
  const u64 v = with_id ? a | ((u64)(b & ((1u << sym_bits) - 1u)) << 48) : a;
  if (sargs32) {  // 4-byte records: access position, or select (ordinal | id << kbits)
    // (invalid queries -- the batch raises -- keep a masked ordinal and id 0)
    const u32 v32 = with_id ? ((u32)a & ((1u << kbits) - 1u)) | ((b & ((1u << sym_bits) - 1u)) << kbits)
                            : (u32)a;
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(sargs32 + slot), "r"(v32),
                 "l"(pl) : "memory");
  }
  else
    asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(sargs + slot), "l"(v), "l"(pl)
                 : "memory");
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(slot_of + i),
               "r"(slot), "l"(pf) : "memory");
  }
}

// results back in query order: out[i] = res[slot_of[i]] -- random 8-byte
// READS (whole sectors, no write-allocate of partial sectors) and coalesced
// writes, where writing through the permutation from the query kernel cost
// as much as the queries' own walk
template <typename TR, typename T>
__global__ void __launch_bounds__(Q_NT) qunsort_kernel(const TR* __restrict__ res,
                                                       const u32* __restrict__ slot_of,
                                                       T* __restrict__ out, u64 m, bool o16) {
  const u64 i0 = ((u64)blockIdx.x * Q_NT + threadIdx.x) * 4;
  if (i0 + 4 <= m) {
    const uint4 s = *reinterpret_cast<const uint4*>(slot_of + i0);
    const T a = __ldg(res + s.x), b = __ldg(res + s.y), c = __ldg(res + s.z), d = __ldg(res + s.w);
    if (o16) {  // the four results as one vector store (16-byte aligned output)
      if (sizeof(T) == 8) {
        reinterpret_cast<ulonglong2*>(out + i0)[0] = make_ulonglong2((u64)a, (u64)b);
        reinterpret_cast<ulonglong2*>(out + i0)[1] = make_ulonglong2((u64)c, (u64)d);
      } else if (sizeof(T) == 2) {
        *reinterpret_cast<uint2*>(out + i0) =
            make_uint2((u32)a | ((u32)b << 16), (u32)c | ((u32)d << 16));
      } else {
        *reinterpret_cast<u32*>(out + i0) = (u32)a | ((u32)b << 8) | ((u32)c << 16) | ((u32)d << 24);
      }
    } else {
      out[i0] = a; out[i0 + 1] = b; out[i0 + 2] = c; out[i0 + 3] = d;
    }
  } else {
    for (u64 i = i0; i < m; ++i) out[i] = (T)res[slot_of[i]];
  }
}

cudaError_t launch_query_sorted(const TreeDev& T, int kind, int out_kind, bool validate,
                                const i64* ids, const i64* args, void* out, u64 m, int rate_log,
                                u64 base, u64* bad, const QuerySortScratch& S, cudaStream_t st,
                                cudaEvent_t* phase) {
  if (m == 0) return cudaSuccess;
  if (m > 0xffffffffull) return cudaErrorInvalidValue;
  const u64 blocks = (m + Q_NT - 1) / Q_NT;
  // buckets: about 128 queries each (2^10 .. 2^20 of them) -- a warp's
  // queries then share nodes and lines at every level; bucket = argument
  // bits over symbol id bits
  u32 qb = 10;
  u32 qmax = kQSortMaxBits, qlog = 7;  // <= 2^20 buckets of ~2^7 queries (swept: 2^5..2^7
                                       // per bucket within 2 %, 2^16 buckets -10 %)
  if (const char* e = getenv(kind == 0 ? "WT_QSORT_A" : kind == 1 ? "WT_QSORT_R" : "WT_QSORT_S")) {
    int a = 0, b = 0;  // tuning override "maxbits,log2 queries per bucket"
    if (sscanf(e, "%d,%d", &a, &b) == 2 && a >= 10 && a <= (int)kQSortMaxBits && b >= 0 && b < 16) {
      qmax = (u32)a;
      qlog = (u32)b;
    }
  }
  while (qb < qmax && (1ull << (qb + qlog)) < m) ++qb;
  u32 sym_bits = 0;
  if (kind != 0)
    while ((1u << sym_bits) < T.sigma) ++sym_bits;
  if (qb < sym_bits) qb = sym_bits;
  const u32 pos_bits = qb - sym_bits;
  u32 arg_shift = 0;  // positions [0, n] must fit in pos_bits bits
  while ((T.n >> arg_shift) >= (1ull << pos_bits)) ++arg_shift;
  const u32 nb = 1u << qb;
  cudaError_t e = cudaMemsetAsync(S.hist, 0, nb * 4, st);
  if (e != cudaSuccess) return e;
  const unsigned kblocks = (unsigned)((m + (u64)QS_QPT * Q_NT - 1) / ((u64)QS_QPT * Q_NT));
  qsort_key_kernel<<<kblocks, Q_NT, 0, st>>>(T, kind, ids, args, m, validate, sym_bits,
                                                      arg_shift, nb, S.bucket_of, S.hist,
                                                      base, bad, S.slot_of);
  const unsigned sb = (nb + QS_PER_CTA - 1) / QS_PER_CTA;
  u32* partial = S.hist + (1u << kQSortMaxBits);
  qsort_scan_partial_kernel<<<sb, 1024, 0, st>>>(S.hist, nb, partial);
  qsort_scan_final_kernel<<<sb, 1024, 0, st>>>(S.hist, nb, partial);
  // access on texts below 2^32: the sorted positions as 4-byte records (half
  // the scattered bytes; the sorted_args buffer holds them)
  // select when ordinal and id fit 32 bits together: (ordinal | id << kbits)
  const bool sel32 = kind == 2 && S.sel_kbits && S.sel_kbits + sym_bits <= 32;
  u32* s32 = (kind == 0 && T.n <= 0xffffffffull) || sel32 ? reinterpret_cast<u32*>(S.sorted_args)
                                                          : nullptr;
  qsort_scatter_kernel<<<kblocks, Q_NT, 0, st>>>(S.bucket_of, kind != 0, sym_bits,
                                                          args, m, S.hist, S.sorted_args, s32,
                                                          sel32 ? S.sel_kbits : 0u, S.slot_of);
  e = cudaGetLastError();
  if (e == cudaSuccess && phase) e = cudaEventRecord(phase[0], st);
  if (e != cudaSuccess) return e;
  // ids are mapped minimal ids now (packed into the arguments): run
  // unvalidated -- validation happened above; invalid queries are clamped
  // into range by the walk and the batch raises anyway.  Results land in
  // sorted order (coalesced), then one gather puts them in query order.
  // rank / select results of a text below 2^32 go to the sorted-order buffer
  // as 4 bytes: the gather back reads half the bytes and mostly hits L2
  u32* r32 = kind != 0 && T.n <= 0xffffffffull ? reinterpret_cast<u32*>(S.res) : nullptr;
  const unsigned wb = (unsigned)((m + Q_NT - 1) / Q_NT);
  if (kind == 2) {
    select_kernel<false><<<wb, Q_NT, 0, st>>>(T, nullptr, S.sorted_args, (i64*)S.res, m, rate_log,
                                              base, bad, true, sel32 ? s32 : nullptr,
                                              sel32 ? S.sel_kbits : 0u, r32);
    e = cudaGetLastError();
  } else if (kind == 1) {
    rank_kernel<false><<<wb, Q_NT, 0, st>>>(T, nullptr, S.sorted_args, (i64*)S.res, m, base, bad,
                                            true, r32);
    e = cudaGetLastError();
  } else if (s32) {
    const unsigned qb2 = (unsigned)((m + Q_NT - 1) / Q_NT);
    if (out_kind == 8)
      access_kernel<8, false><<<qb2, Q_NT, 0, st>>>(T, nullptr, S.res, m, base, bad, true, s32);
    else if (out_kind == 1)
      access_kernel<1, false><<<qb2, Q_NT, 0, st>>>(T, nullptr, S.res, m, base, bad, true, s32);
    else
      access_kernel<2, false><<<qb2, Q_NT, 0, st>>>(T, nullptr, S.res, m, base, bad, true, s32);
    e = cudaGetLastError();
  } else {
    e = launch_query(T, kind, out_kind, false, nullptr, S.sorted_args, S.res, m, rate_log, base,
                     bad, st, true);
  }
  if (e == cudaSuccess && phase) e = cudaEventRecord(phase[1], st);
  if (e != cudaSuccess) return e;
  const unsigned ub = (unsigned)((m + 4 * Q_NT - 1) / (4 * Q_NT));
  const bool o16 = ((uintptr_t)out & 15) == 0;
  const int ob = kind == 0 ? out_kind : 8;
  if (r32)
    qunsort_kernel<u32, u64><<<ub, Q_NT, 0, st>>>(r32, S.slot_of, (u64*)out, m, o16);
  else if (ob == 1)
    qunsort_kernel<u8, u8><<<ub, Q_NT, 0, st>>>((const u8*)S.res, S.slot_of, (u8*)out, m, o16);
  else if (ob == 2)
    qunsort_kernel<u16, u16><<<ub, Q_NT, 0, st>>>((const u16*)S.res, S.slot_of, (u16*)out, m, o16);
  else
    qunsort_kernel<u64, u64><<<ub, Q_NT, 0, st>>>((const u64*)S.res, S.slot_of, (u64*)out, m, o16);
  e = cudaGetLastError();
  if (e == cudaSuccess && phase) e = cudaEventRecord(phase[2], st);
  return e;
}

// ---------------------------------------------------------------------------
// narrow wire format (wt_capi.cu host pipeline): 6 bytes per rank / select
// query and 4 per access query cross PCIe instead of 16 / 8; the widening is
// a streaming pass (22 B per query of HBM traffic, ~0.1 ms per 2^22 chunk)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) widen_kernel(const u16* __restrict__ w16,
                                                    const u32* __restrict__ w32,
                                                    i64* __restrict__ ids, i64* __restrict__ args,
                                                    u64 m) {
  const u64 stride = (u64)gridDim.x * 256;
  for (u64 i = (u64)blockIdx.x * 256 + threadIdx.x; i < m; i += stride) {
    args[i] = (i64)__ldg(w32 + i);
    if (w16) ids[i] = (i64)__ldg(w16 + i);
  }
}

cudaError_t launch_widen(const u16* w16, const u32* w32, i64* ids, i64* args, u64 m,
                         cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  const u64 want = (m + 255) / 256;
  const unsigned blocks = (unsigned)std::min<u64>(want, 148ull * 16);
  widen_kernel<<<blocks, 256, 0, st>>>(w16, w32, ids, args, m);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// single bit-vector queries (RankSelectIndex.*_bulk, rankselect.py:145-373)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(Q_NT) bits_query_kernel(const LevelDev L, u32 l2_shift, u64 rate,
                                                          int rate_log, int kind,
                                                          const i64* __restrict__ args,
                                                          i64* __restrict__ out, u64 m) {
  const u64 i = (u64)blockIdx.x * Q_NT + threadIdx.x;
  if (i >= m) return;
  const u64 a = (u64)args[i];
  i64 r;
  switch (kind) {
    case 0: r = (i64)rank1_dev(L, a, l2_shift); break;
    case 1: r = (i64)(a - rank1_dev(L, a, l2_shift)); break;
    case 2: r = (i64)select_dev<true>(L, a, l2_shift, rate, rate_log); break;
    case 3: r = (i64)select_dev<false>(L, a, l2_shift, rate, rate_log); break;
    default: r = (i64)((__ldg(L.words + (a >> 6)) >> (a & 63)) & 1ull); break;
  }
  out[i] = r;
}

cudaError_t launch_bits_query(const LevelDev& L, u32 l2_shift, u64 rate, int rate_log, int kind,
                              const i64* args, i64* out, u64 m, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  const u64 blocks = (m + Q_NT - 1) / Q_NT;
  bits_query_kernel<<<(unsigned)blocks, Q_NT, 0, st>>>(L, l2_shift, rate, rate_log, kind, args,
                                                       out, m);
  return cudaGetLastError();
}

}  // namespace wt
