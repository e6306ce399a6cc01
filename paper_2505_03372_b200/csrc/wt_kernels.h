// wt_kernels.h -- host-visible launch wrappers of the CUDA kernels.
#pragma once
#include "wt_common.cuh"

namespace wt {

// K2w parameters (wt_wlevel.cu): warp-granular tiles of 2 KB of input
struct WLevelParams {
  const void* in;          // level input: text (level 0) or the partitioned codes
  void* out;               // next level's codes (nullptr at the last level)
  u64 m, m_next;           // level_sizes[l], level_sizes[l+1]
  u64* words;              // region start
  u16* l2;
  u64* ones;
  u64* zeros;
  u64 ones_cap, zeros_cap;
  const NodeEnt* nodes;    // 2^l entries keyed by the l-bit code prefix
  const u16* lut;          // level 0: raw symbol -> code (nullptr: identity)
  const u64* l1;           // this level's L1 directory (ones before each 65536-bit block)
  const u32* tile_counts;  // ones per warp tile of this level (nullptr: block mode, level 0)
  u32* next_tile_counts;   // ones of level l+1 per warp tile of level l+1 (atomics)
  u32* next_l1_counts;     // ones of level l+1 per L1 block (atomics)
  // pair mode (out == nullptr, next_words != nullptr): level l+1 is the last
  // level; its bits are written straight from the staged runs (region start,
  // zeroed by the caller) instead of partitioning the codes into `out`
  u64* next_words;
  // block mode for this AND the next level (tile_counts == nullptr,
  // next_tile_counts unused): next-level ones per L1 block only, counted in
  // the first pass; nthr = the three raw-symbol thresholds of the code's top
  // two bits at a LUT level 0 (bit l+1 = parity of symbol >= nthr[i])
  int next_block;
  int skip_dir;            // L2 entries / samples left to dir_kernel (fast tiles)
  // small alphabets at a u8 LUT level: code = byte plut_lo|hi[(sym >> plut_shift)
  // & 7] -- one PRMT per 4 symbols instead of 4 table loads (0xff: unused)
  u32 plut_shift, plut_lo, plut_hi;
  u32 nthr[3];
  u32 thr;                 // level 0 with a LUT: smallest symbol whose code has the top bit
  u32 shift_bit;           // L-1-l
  u32 shift_key;           // L-l
  u32 l2_log;
  int rate_log;            // log2(rate) when rate is a power of two, else -1
  u64 rate;
};
cudaError_t launch_wlevel(const WLevelParams& p, int in_bytes, int code_bytes, bool lut, int sms,
                          cudaStream_t st);
u32 wlevel_tiles(u64 m, int in_bytes);
// resident warps of the u8 level kernel on the device (block-mode threshold)
u64 wlevel_warp_slots(int sms);
// level 0 of a u8 text in block mode (WLevelParams::tile_counts == nullptr):
// per-L1-block ones (symbols >= thr) from the per-block histograms K1 wrote
cudaError_t launch_block_l1(const u32* block_hist, u64 n_blocks, u32 thr, u32* l1_counts,
                            cudaStream_t st);
// ones per warp tile of level 0: text symbols >= thr (the top code bit)
cudaError_t launch_wcount0(const void* text, u64 n, int in_bytes, u32 thr, u32* tile_counts,
                           u32* l1_counts, int sms, cudaStream_t st);
// exclusive scan of per-L1-block counts -> l1[0..n_l1) and the level total
cudaError_t launch_l1_scan(const u32* counts, u64 n_l1, u64* l1, u64* total, cudaStream_t st);
// L2 entries and select samples of a level whose bits and L1 directory exist
// (the level a pair-mode launch wrote): one warp per L1 block
struct DirParams {
  const u64* words;  // region start
  u64 m;             // bits
  const u64* l1;
  u16* l2;
  u64* ones;
  u64* zeros;
  u64 ones_cap, zeros_cap;
  u32 l2_log;
  int rate_log;
  u64 rate;
};
cudaError_t launch_dir(const DirParams& p, int sms, cudaStream_t st);

// K1: raw-symbol histogram (wt_hist.cu); hist must be zeroed (u64[256|65536])
// block_hist (may be null): per 65536-symbol L1 block, u8: its 256-bin
// histogram, u32[n_blocks][256]; u16: its count of symbols >= 32768,
// u32[n_blocks] (zeroed by the caller)
cudaError_t launch_histogram(const void* text, u64 n, int sym_bytes, u64* hist, int sms,
                             cudaStream_t st, u32* block_hist = nullptr);
// first text position whose raw symbol has member[sym] == 0; *best preset to ~0
cudaError_t launch_first_outside(const void* text, u64 n, int sym_bytes, const u8* member,
                                 u64* best, int sms, cudaStream_t st);

// Q kernels (wt_query.cu)
// kind 0/1/2 = access/rank/select; out_kind (access): 1|2 = symbol bytes, 8 = int64 id;
// validate: ids are original symbols, invalid queries -> atomicMin(bad, base + i)
// packed: arguments are the device sort's (argument | id << 48), clamped, unvalidated
cudaError_t launch_query(const TreeDev& T, int kind, int out_kind, bool validate, const i64* ids,
                         const i64* args, void* out, u64 m, int rate_log, u64 base, u64* bad,
                         cudaStream_t st, bool packed = false);

// device sort_queries_by_symbol: counting sort into <= 2^20 buckets, then the
// query kernel on the sorted batch writing results back in query order
constexpr u32 kQSortMaxBits = 20;  // at most 2^20 sort buckets
struct QuerySortScratch {
  u32* hist;        // (1 << kQSortMaxBits) bucket counts / cursors + 256 scan partials
  u32* bucket_of;   // m (the minimal id is the bucket's top bits)
  i64* sorted_args; // m: argument | id << 48
  u32* slot_of;     // m: sorted slot of each query (query order)
  void* res;        // m results in sorted order (out_kind bytes each)
  u32 sel_kbits = 0; // bits of the largest select ordinal (0: 8-byte records only)
};
// phase (optional): 3 events recorded after the sort (key + scan + scatter),
// after the walk and after the gather back to query order
// host-buffer batches on the narrow wire format: u16 symbols / u32 arguments
// (packed on the host) widened into the i64 chunk buffers the query kernels read
cudaError_t launch_widen(const u16* w16, const u32* w32, i64* ids, i64* args, u64 m,
                         cudaStream_t st);
cudaError_t launch_query_sorted(const TreeDev& T, int kind, int out_kind, bool validate,
                                const i64* ids, const i64* args, void* out, u64 m, int rate_log,
                                u64 base, u64* bad, const QuerySortScratch& S, cudaStream_t st,
                                cudaEvent_t* phase = nullptr);

// query-side rank-line layout (wt_qlayout.cu)
u64 qlayout_lines(u64 n_bits);
// one streaming pass over a level whose bits and L1 directory exist: its L2
// entries and select samples (the reference directory) AND its query lines
// with their line samples (wt_qlayout.cu); replaces dir_kernel + qlayout
struct DirQParams {
  DirParams d;
  const u64* total;  // the level's ones (device)
  ulonglong2* lines;
  u64 n_lines;
  u32* sel1;
  u32* sel0;
  u64 cap1, cap0;
};
// pdl: launched as a programmatic dependent of the preceding kernel on `st`
// (an l1_scan_kernel, which releases it at its start): the two overlap.  The
// directory pass reads nothing that kernel writes.
cudaError_t launch_dirq(const DirQParams& p, int sms, cudaStream_t st, bool pdl = false);
cudaError_t launch_qlayout(const LevelDev& L, const u64* total, u32 l2_shift, ulonglong2* lines,
                           u64 n_lines, u32* sel1, u64 cap1, u32* sel0, u64 cap0, cudaStream_t st);

// single bit-vector index (wt_bits.cu)
struct BitsParams {
  const u64* words;
  u64 n_bits;
  u64* l1;
  u16* l2;
  u64* ones;
  u64* zeros;
  u64 ones_cap, zeros_cap;
  u64* status;
  u32* agg;
  u32* counter;
  u64* total_out;
  u32 l2_log;
  int rate_log;
  u64 rate;
};
cudaError_t launch_bits_directory(const BitsParams& p, cudaStream_t st);
u32 bits_tiles(u64 n_bits);
cudaError_t launch_bits_query(const LevelDev& L, u32 l2_shift, u64 rate, int rate_log, int kind,
                              const i64* args, i64* out, u64 m, cudaStream_t st);

}  // namespace wt
