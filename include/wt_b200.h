/*
 * wt_b200.h -- C-ABI of the B200-native wavelet-tree engine (libwt_b200.so).
 *
 * Plain pointers and sizes only; no torch / CUDA types cross this boundary
 * (streams are passed as void*).  Every function returns WT_OK (0) or a
 * nonzero status; wt_last_error() returns the thread's last message.
 *
 * Each entry point replaces one reference interface of wtindex 0.1.0
 * (paths relative to /root/reference/pkg/src/wtindex):
 *
 *   wt_construct          <- wtree.construct / construct_with_alphabet
 *                            (wtree.py:438-466) = _coerce_text'd array in,
 *                            minimal_alphabet / map_text (alphabet.py:76-111),
 *                            encode_and_histogram (alphabet.py:210-242),
 *                            _build (wtree.py:406-435) incl. build_index per
 *                            level (rankselect.py:442-536) and node_rank0.
 *   wt_tree_meta/_get     <- the attributes WaveletTree exposes
 *                            (wtree.py:113-133, bits/rs/node tables).
 *   wt_tree_query         <- WaveletTree.access_ids_bulk (wtree.py:283-315),
 *                            rank_ids_bulk (:317-341), select_ids_bulk (:343-375)
 *                            driven by BatchRunner.run (batch.py:152-239); access
 *                            also applies batch._decode (batch.py:241-244)
 *   wt_tree_from_arrays   <- wtree.load (wtree.py:500-577): device tree from
 *                            validated host arrays.
 *   wt_bits_build         <- rankselect.build_index over one BitArray region
 *                            (rankselect.py:442-536)
 *   wt_bits_query         <- RankSelectIndex.rank1_bulk / rank0_bulk /
 *                            select1_bulk / select0_bulk / get_bits_bulk
 *                            (rankselect.py:145-222, :293-373)
 *   wt_tree_level_query   <- RankSelectIndex rank/select/get_bit on tree.rs[l]
 *   wt_tree_replicate     <- (no reference counterpart; the north star's NCCL
 *                            broadcast of a built tree to the other GPUs)
 *   wt_bits_from_arrays   <- RankSelectIndex.read / rebind (rankselect.py:397-411,
 *                            :135-136): a deserialized directory, uploaded as is
 *   wt_minimal_alphabet   <- alphabet.minimal_alphabet (alphabet.py:94-111)
 *   wt_map_text           <- AlphabetMap.map_text (alphabet.py:76-84)
 *   wt_encode_histogram   <- alphabet.encode_and_histogram (alphabet.py:210-242)
 *   wt_sort_by_prefix     <- wtree.stable_sort_by_prefix (wtree.py:92-100)
 *   wt_fill_level         <- wtree.fill_level (wtree.py:103-107) ->
 *                            BitArray.fill_region packing (bitvec.py:119-151)
 */
#ifndef WT_B200_H
#define WT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WT_ABI_VERSION 1

/* status codes */
#define WT_OK           0
#define WT_ERR_CUDA     1   /* CUDA runtime/driver failure            */
#define WT_ERR_ARG      2   /* invalid argument (caller bug)          */
#define WT_ERR_OOM      3   /* device allocation failed               */
#define WT_ERR_SYMBOL   4   /* text symbol outside declared alphabet; */
                            /* wt_last_error_index() = first position */
#define WT_ERR_NCCL     5   /* NCCL load/communication failure        */
#define WT_ERR_BUILD    6   /* alphabet larger than 2^16 etc.         */

/* query kinds */
#define WT_Q_ACCESS 0
#define WT_Q_RANK   1
#define WT_Q_SELECT 2

/* bit-vector query kinds (wt_bits_query) */
#define WT_B_RANK1   0
#define WT_B_RANK0   1
#define WT_B_SELECT1 2
#define WT_B_SELECT0 3
#define WT_B_BIT     4

/* flags for the query entry points */
#define WT_F_DEVICE_PTRS 1  /* ids/args/out are device pointers (no copies) */
#define WT_F_SYMBOLS     2  /* ids hold ORIGINAL symbols: mapped and range-checked
                               on the device (BatchRunner._validate, batch.py:112-148);
                               *bad_index = first invalid query or -1           */
#define WT_F_ACCESS_IDS  4  /* access returns int64 minimal ids (access_ids_bulk)
                               instead of decoded symbols (batch._decode)        */
#define WT_F_SORT        8  /* sort the batch on the device before the walk, for
                               locality -- the device counterpart of
                               batch.sort_queries_by_symbol (batch.py:61-75;
                               PAPER.md:928, :988): buckets of (coarse text
                               position, symbol); results stay in query order,
                               errors report the first bad index as unsorted  */
#define WT_F_PHASES     16  /* with WT_F_SORT | WT_F_DEVICE_PTRS and ms_out: ms_out
                               is float[4] = {total, sort, walk, gather} device
                               times (CUDA events on the query stream)        */

/* array selectors for wt_tree_get */
#define WT_A_SYMBOLS      0   /* u16[sigma]   sorted alphabet symbols        */
#define WT_A_CODE_VALUES  1   /* u16[sigma]   left-aligned path words        */
#define WT_A_CODE_LENS    2   /* u8[sigma]                                  */
#define WT_A_CUM_HIST     3   /* i64[sigma+1]                               */
#define WT_A_LEVEL_SIZES  4   /* i64[levels]                                */
#define WT_A_REGION_OFFS  5   /* i64[levels]  bit offsets (1024-aligned)     */
#define WT_A_WORDS        6   /* u64[n_words] whole bit array                */
#define WT_A_L1           7   /* i64[n_l1]    per level                      */
#define WT_A_L2           8   /* u16[n_l2]    per level                      */
#define WT_A_ONES         9   /* i64[n_ones]  per level (select samples)     */
#define WT_A_ZEROS       10   /* i64[n_zeros] per level                      */
#define WT_A_NODE_STARTS 11   /* i64[n_nodes] per level                      */
#define WT_A_NODE_RANK0  12   /* i64[n_nodes] per level                      */
/* query-side layout (this engine's own, not part of the index format):     */
#define WT_A_QLINES      13   /* u64[4 * n_lines] per level: [ones before | 3 words] */
#define WT_A_QSEL1       14   /* u32 per level: line of every 64-th one           */
#define WT_A_QSEL0       15   /* u32 per level: line of every 64-th zero          */

typedef struct wt_tree wt_tree;
typedef struct wt_bits wt_bits;

typedef struct {
    uint64_t n;            /* text length                                     */
    uint32_t sigma;        /* alphabet size                                   */
    uint32_t levels;       /* ceil(lg sigma)                                  */
    uint32_t symbol_width; /* 1 | 2 bytes                                     */
    uint32_t l2_bits;
    uint64_t sample_rate;
    uint32_t first_coded;  /* first symbol id with an explicit (short) code   */
    uint32_t device;
    uint64_t n_words;      /* length of the whole bit array in u64 words      */
    uint64_t device_bytes; /* device memory held by the tree                  */
} wt_meta;

typedef struct {
    uint64_t n_bits, total_ones, n_l1, n_l2, n_ones, n_zeros, n_nodes;
} wt_level_meta;

/* -- errors / device -------------------------------------------------------- */
const char* wt_last_error(void);
int64_t     wt_last_error_index(void);
int         wt_abi_version(void);
int         wt_device_count(int* count);

/* -- construction ------------------------------------------------------------
 * text: n symbols of sym_bytes (1|2) bytes, host pointer (copied) or device
 * pointer (text_on_device=1; borrowed for the call).
 * alphabet: NULL -> infer the minimal alphabet (construct); else alphabet_len
 * strictly increasing symbols (construct_with_alphabet), and every text
 * symbol must be in it (else WT_ERR_SYMBOL, wt_last_error_index() = first
 * offending position).  symbol_width is the reported width (1|2).
 * stream: cudaStream_t or NULL (library stream).  ms_out (may be NULL):
 * device time of the build measured with CUDA events on that stream.      */
int wt_construct(const void* text, uint64_t n, int sym_bytes, int text_on_device,
                 const uint16_t* alphabet, uint32_t alphabet_len, int symbol_width,
                 uint32_t l2_bits, uint64_t sample_rate, int device, void* stream,
                 wt_tree** out, float* ms_out);

/* Device tree from host arrays (index-file load).  All arrays as wt_tree_get
 * returns them; per-level arrays concatenated level after level.          */
int wt_tree_from_arrays(const wt_meta* meta, const uint16_t* symbols,
                        const int64_t* cum_hist, const uint64_t* words,
                        const wt_level_meta* levels, const int64_t* l1_cat,
                        const uint16_t* l2_cat, const int64_t* ones_cat,
                        const int64_t* zeros_cat, int device, wt_tree** out);

int wt_tree_meta(const wt_tree* t, wt_meta* out);
int wt_tree_level_meta(const wt_tree* t, uint32_t level, wt_level_meta* out);
/* copy array `what` (WT_A_*) of `level` into host memory dst (cap bytes) */
int wt_tree_get(const wt_tree* t, int what, uint32_t level, void* dst, uint64_t cap);
/* device time of the last build, CUDA events on the build stream:
 * ms[0] = text upload + histogram + O(sigma) plan, ms[1+l] = level-l kernel  */
int wt_tree_build_profile(const wt_tree* t, float* ms, uint32_t cap);
int wt_tree_destroy(wt_tree* t);

/* -- queries (minimal-id domain, validated by the caller) --------------------
 * access: args = positions in [0,n); out = original symbols (u8 if
 *         symbol_width==1 else u16) or int64 ids (WT_F_ACCESS_IDS) -- ids ignored
 * rank:   ids = symbol ids, args = positions in [0,n]; out = int64
 * select: ids = symbol ids, args = ordinals in [1,occ]; out = int64
 * Host pointers are streamed through pinned double buffers in chunks of
 * `chunk` queries (0 = default); WT_F_DEVICE_PTRS runs in place.
 * ms_out (may be NULL): device time of the kernels (CUDA events).          */
int wt_tree_query(wt_tree* t, int kind, const int64_t* ids, const int64_t* args,
                  void* out, uint64_t m, uint64_t chunk, int flags, void* stream,
                  int64_t* bad_index, float* ms_out);

/* Pipeline accounting of one host-buffer query (device times from CUDA
 * events on the three pipeline streams; BatchRunner.stage_seconds /
 * process_seconds / staging_peak_records, batch.py:93-108, :192-224).      */
typedef struct {
    uint64_t chunks;         /* chunks the batch was split into             */
    uint64_t slots;          /* device staging slots used (<= 2)            */
    uint64_t chunk_records;  /* queries per chunk                           */
    uint64_t peak_records;   /* most queries staged in device slots at once:
                                a chunk is staged from its copy-in start to
                                its kernel's end (CUDA events per chunk)     */
    float h2d_ms;            /* sum of copy-in durations                    */
    float kernel_ms;         /* sum of kernel durations                     */
    float d2h_ms;            /* last kernel end -> last copy-out end         */
    float total_ms;          /* first copy-in start -> last copy-out end     */
    uint64_t h2d_bytes;      /* bytes copied host->device (narrow wire: 6 per
                                rank / select query, 4 per access query;
                                16 / 8 for chunks that crossed wide)         */
    uint64_t narrow_chunks;  /* chunks that crossed on the narrow wire       */
} wt_query_stats;
/* wt_tree_query plus the pipeline accounting (stats may be NULL).          */
int wt_tree_query_ex(wt_tree* t, int kind, const int64_t* ids, const int64_t* args,
                     void* out, uint64_t m, uint64_t chunk, int flags, void* stream,
                     int64_t* bad_index, float* ms_out, wt_query_stats* stats);

/* Pinned host memory (cudaHostAlloc) for result arrays: device->host copies
 * into it are asynchronous and overlap the next chunk's kernel.           */
int wt_host_alloc(uint64_t bytes, void** out);
int wt_host_free(void* p);
/* Page-lock / release an existing host range (cudaHostRegister): the
 * multi-GPU runner's shared result array, whose disjoint slices the ranks
 * of a node fill straight from their devices.                              */
int wt_host_register(void* p, uint64_t bytes);
int wt_host_unregister(void* p);

/* Bit-vector query (WT_B_*) against one level of a built tree: the
 * RankSelectIndex methods of tree.rs[l] (rankselect.py:140-373).  Host
 * int64 arrays; callers validate ranges first.                             */
int wt_tree_level_query(wt_tree* t, uint32_t level, int kind, const int64_t* args,
                        int64_t* out, uint64_t m);

/* -- replication over NCCL (one process per GPU) -----------------------------
 * wt_nccl_unique_id fills 128 bytes on the root; every rank calls
 * wt_tree_replicate with the same id: the root passes its tree, the others
 * NULL and receive a device-resident copy in *out.                         */
int wt_nccl_unique_id(uint8_t id[128]);
int wt_tree_replicate(wt_tree* root_tree, const uint8_t id[128], int rank, int world,
                      int device, wt_tree** out, float* ms_out);

/* -- single bit-vector rank/select index -----------------------------------*/
int wt_bits_build(const uint64_t* words, uint64_t n_bits, int words_on_device,
                  uint32_t l2_bits, uint64_t sample_rate, int device, wt_bits** out);
int wt_bits_level_meta(const wt_bits* b, wt_level_meta* out);
int wt_bits_get(const wt_bits* b, int what, void* dst, uint64_t cap);
int wt_bits_query(wt_bits* b, int kind, const int64_t* args, int64_t* out, uint64_t m,
                  int flags);
int wt_bits_destroy(wt_bits* b);
/* RankSelectIndex.read: a validated, deserialized directory over host words,
 * uploaded unchanged (queries answer from the stored arrays).              */
int wt_bits_from_arrays(const uint64_t* words, uint64_t n_bits, uint32_t l2_bits,
                        uint64_t sample_rate, uint64_t total_ones, const int64_t* l1,
                        uint64_t n_l1, const uint16_t* l2, uint64_t n_l2,
                        const int64_t* ones, uint64_t n_ones, const int64_t* zeros,
                        uint64_t n_zeros, int device, wt_bits** out);

/* -- the reference's O(n) building blocks, one call each (host arrays in and
 * out; the device does the O(n) work).  wt_construct fuses all of them.     */
/* ids_out[n] = minimal id of each symbol; symbols_out (256 | 65536 entries
 * of room) = the sorted present symbols; *sigma_out = their count.          */
int wt_minimal_alphabet(const void* text, uint64_t n, int sym_bytes, int device,
                        uint16_t* ids_out, uint16_t* symbols_out, uint32_t* sigma_out);
/* ids_out[n] = index of text[i] in the sorted `symbols`; an undeclared symbol
 * -> WT_ERR_SYMBOL, wt_last_error_index() = its first position.            */
int wt_map_text(const void* text, uint64_t n, int sym_bytes, const uint16_t* symbols,
                uint32_t sigma, int device, uint16_t* ids_out);
/* encoded_out[i] = code_values[ids[i]], hist_out[sigma] = counts of each id;
 * an id >= sigma -> WT_ERR_SYMBOL, wt_last_error_index() = first one.      */
int wt_encode_histogram(const uint16_t* ids, uint64_t n, const uint16_t* code_values,
                        uint32_t sigma, int device, uint16_t* encoded_out, int64_t* hist_out);
/* out = codes stably sorted by (code >> shift).                             */
int wt_sort_by_prefix(const uint16_t* codes, uint64_t n, uint32_t shift, int device,
                      uint16_t* out);
/* words_out[ceil(count/64)] = bit `bit` of codes[0..count), LSB-first, zero
 * padded.                                                                    */
int wt_fill_level(const uint16_t* codes, uint64_t count, uint32_t bit, int device,
                  uint64_t* words_out);

#ifdef __cplusplus
}
#endif
#endif /* WT_B200_H */
