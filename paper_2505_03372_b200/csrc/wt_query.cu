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
#include "wt_common.cuh"
#include "wt_kernels.h"
#include "wt_rs.cuh"

namespace wt {

constexpr int Q_NT = 256;

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
                                                      u64* __restrict__ bad) {
  const u64 i = (u64)blockIdx.x * Q_NT + threadIdx.x;
  if (i >= m) return;
  u64 p = (u64)pos[i];
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
                                                    u64* __restrict__ bad) {
  const u64 i = (u64)blockIdx.x * Q_NT + threadIdx.x;
  if (i >= m) return;
  u32 c;
  u64 p = (u64)pos[i];
  if (!symbol_id<kValidate>(T, ids[i], c) || (kValidate && p > T.n)) {
    atomicMin(bad, base + i);
    return;
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
  out[i] = (i64)(p - (u64)__ldg(T.cum + c));
}

template <bool kValidate>
__global__ void __launch_bounds__(Q_NT) select_kernel(const __grid_constant__ TreeDev T,
                                                      const i64* __restrict__ ids,
                                                      const i64* __restrict__ ks,
                                                      i64* __restrict__ out, u64 m, int rate_log,
                                                      u64 base, u64* __restrict__ bad) {
  const u64 i = (u64)blockIdx.x * Q_NT + threadIdx.x;
  if (i >= m) return;
  u32 c;
  const i64 k = ks[i];
  if (!symbol_id<kValidate>(T, ids[i], c) ||
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
  out[i] = (i64)p;
}

template <bool V>
static void launch_q(const TreeDev& T, int kind, int out_kind, const i64* ids, const i64* args,
                     void* out, u64 m, int rate_log, u64 base, u64* bad, unsigned blocks,
                     cudaStream_t st) {
  switch (kind) {
    case 0:
      if (out_kind == 8)
        access_kernel<8, V><<<blocks, Q_NT, 0, st>>>(T, args, out, m, base, bad);
      else if (out_kind == 1)
        access_kernel<1, V><<<blocks, Q_NT, 0, st>>>(T, args, out, m, base, bad);
      else
        access_kernel<2, V><<<blocks, Q_NT, 0, st>>>(T, args, out, m, base, bad);
      break;
    case 1:
      rank_kernel<V><<<blocks, Q_NT, 0, st>>>(T, ids, args, (i64*)out, m, base, bad);
      break;
    default:
      select_kernel<V><<<blocks, Q_NT, 0, st>>>(T, ids, args, (i64*)out, m, rate_log, base, bad);
      break;
  }
}

cudaError_t launch_query(const TreeDev& T, int kind, int out_kind, bool validate, const i64* ids,
                         const i64* args, void* out, u64 m, int rate_log, u64 base, u64* bad,
                         cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  if (kind < 0 || kind > 2) return cudaErrorInvalidValue;
  const u64 blocks = (m + Q_NT - 1) / Q_NT;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidValue;
  if (validate)
    launch_q<true>(T, kind, out_kind, ids, args, out, m, rate_log, base, bad, (unsigned)blocks, st);
  else
    launch_q<false>(T, kind, out_kind, ids, args, out, m, rate_log, base, bad, (unsigned)blocks, st);
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
