// wt_capi.cu -- the extern "C" boundary (include/wt_b200.h) and the native
// host runtime around the kernels: O(sigma) planning (codes, level sizes,
// region layout, node tables), device memory, streams, the chunked host
// query pipeline and NCCL replication.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <type_traits>
#include <dlfcn.h>
#include <unistd.h>
#include <atomic>
#include <immintrin.h>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "../../include/wt_b200.h"
#include "wt_common.cuh"
#include "wt_kernels.h"
#include "wt_host.h"

using namespace wt;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
#include <chrono>
thread_local std::string g_err;
thread_local int64_t g_err_index = -1;
// WT_TRACE=1: host-side phase timestamps of wt_construct on stderr
static bool trace_on() {
  static int v = -1;
  if (v < 0) v = getenv("WT_TRACE") && getenv("WT_TRACE")[0] == '1';
  return v == 1;
}
struct Tracer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!trace_on()) return;
    auto d = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[wt] %8.3f ms  %s\n", d, what);
  }
};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

extern "C" const char* wt_last_error(void) { return g_err.c_str(); }
extern "C" int64_t wt_last_error_index(void) { return g_err_index; }
extern "C" int wt_abi_version(void) { return WT_ABI_VERSION; }
extern "C" int wt_device_count(int* count) {
  CU(cudaGetDeviceCount(count));
  return WT_OK;
}

// ---------------------------------------------------------------------------
// device memory: stream-ordered pool, kept warm across builds
// ---------------------------------------------------------------------------
static std::once_flag g_pool_once[64];
int setup_device(int device) {
  CU(cudaSetDevice(device));
  if (device >= 0 && device < 64) {
    std::call_once(g_pool_once[device], [device]() {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    });
  }
  return WT_OK;
}

int sm_count(int device) {
  int v = 148;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v;
}

template <typename T>
static int dalloc(T** p, size_t count, cudaStream_t st) {
  size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  CU(cudaMallocAsync((void**)p, bytes, st));
  return WT_OK;
}

// ---------------------------------------------------------------------------
// O(sigma) planning (host): the reference's alphabet.py / wtree.py shape logic
// ---------------------------------------------------------------------------
static inline uint32_t ceil_log2_u(uint64_t s) {
  return s <= 1 ? 0u : 64u - (uint32_t)__builtin_clzll(s - 1);
}
static inline uint64_t prev_pow_two_u(uint64_t x) {  // alphabet.py:28-32: largest 2^k < x
  if (x <= 2) return 1;
  return 1ull << (63 - __builtin_clzll(x - 1));
}

struct Plan {
  uint32_t sigma = 0, L = 0, first_coded = 0;
  std::vector<uint16_t> symbols, values;
  std::vector<uint8_t> lens;
  std::vector<int64_t> hist, cum, sizes, offsets;
  uint64_t n_words = 0;
  std::vector<NodeEnt> nodes;
  std::vector<uint64_t> node_off;  // start of level l in `nodes`
  std::vector<uint64_t> n_nodes;                           // per level
  std::vector<std::vector<int64_t>> node_starts, node_rank0;  // filled on export
  int code_bytes = 1;
};

// Reduced-tree codes (alphabet.py:160-207): the left/right path of every leaf
// of the shape in which node [a,b) splits at a + prev_pow_two(b-a)
// (wtree.py:388-403), left-aligned in an L-bit field.
static void plan_codes(Plan& P) {
  const uint32_t s = P.sigma, L = P.L;
  P.values.resize(s);
  P.lens.assign(s, (uint8_t)L);
  for (uint32_t i = 0; i < s; ++i) P.values[i] = (uint16_t)i;
  if ((s & (s - 1)) == 0) {
    P.first_coded = s;
    return;
  }
  P.first_coded = (uint32_t)prev_pow_two_u(s);
  struct Item { uint32_t a, b, depth, path; };
  std::vector<Item> todo{{P.first_coded, s, 1, 1}};
  while (!todo.empty()) {
    Item it = todo.back();
    todo.pop_back();
    const uint32_t w = it.b - it.a;
    if ((w & (w - 1)) == 0) {  // complete subtree: path + plain offsets
      uint32_t k = 0;
      while ((1u << k) < w) ++k;
      for (uint32_t o = 0; o < w; ++o) {
        P.values[it.a + o] = (uint16_t)((((uint32_t)it.path << k) + o) << (L - it.depth - k));
        P.lens[it.a + o] = (uint8_t)(it.depth + k);
      }
      continue;
    }
    const uint32_t p = (uint32_t)prev_pow_two_u(w);
    todo.push_back({it.a, it.a + p, it.depth + 1, it.path << 1});
    todo.push_back({it.a + p, it.b, it.depth + 1, (it.path << 1) | 1});
  }
}

// hist (per id) known: cum_hist, level sizes, region layout, node tables.
static std::vector<NodeEnt>& node_cache() {
  static thread_local std::vector<NodeEnt> v;
  return v;
}
// The node traversal (wtree.py:388-433): device node entries and per-level
// node counts at build time; the reference's node_starts / node_rank0 arrays
// only when exported (wt_tree_get), so a 2^16-symbol build does not allocate
// them.
static void plan_walk(Plan& P, bool tables, uint32_t levels = ~0u) {
  const uint32_t s = P.sigma, L = std::min(P.L, levels);
  static thread_local std::vector<std::pair<uint32_t, uint32_t>> cur, nxt;
  cur.clear();
  P.n_nodes.assign(P.L, 0);
  if (tables) {
    P.node_starts.assign(L, {});
    P.node_rank0.assign(L, {});
  }
  if (L) cur.push_back({0, s});
  for (uint32_t l = 0; l < L; ++l) {
    int64_t zeros_before = 0;
    nxt.clear();
    P.n_nodes[l] = cur.size();
    if (tables) {
      P.node_starts[l].reserve(cur.size());
      P.node_rank0[l].reserve(cur.size());
    }
    for (auto [a, b] : cur) {
      const uint32_t p = (uint32_t)prev_pow_two_u(b - a);
      const int64_t Z = P.cum[a + p] - P.cum[a];
      if (tables) {
        P.node_starts[l].push_back(a);
        P.node_rank0[l].push_back(zeros_before);
      } else {
        const uint32_t key = (uint32_t)P.values[a] >> (P.L - l);
        NodeEnt& ne = P.nodes[P.node_off[l] + key];
        ne.zero_base = P.cum[a] - zeros_before;
        ne.one_base = Z + zeros_before;
        ne.leaf[0] = p == 1 ? (int)a : -1;
        ne.leaf[1] = (b - a - p) == 1 ? (int)(a + p) : -1;
      }
      zeros_before += Z;
      if (p >= 2) nxt.push_back({a, a + p});
      if (b - a - p >= 2) nxt.push_back({a + p, b});
    }
    cur.swap(nxt);
  }
}

// walk_levels: node levels filled now (the construct path fills level 0 only
// and the rest while level 0 runs on the device)
static void plan_shape(Plan& P, uint32_t l2_bits, uint32_t walk_levels = ~0u) {
  (void)l2_bits;
  const uint32_t s = P.sigma, L = P.L;
  P.cum.assign(s + 1, 0);
  for (uint32_t i = 0; i < s; ++i) P.cum[i + 1] = P.cum[i] + P.hist[i];
  // sizes[l] = symbols whose code is longer than l: by code length, O(sigma + L)
  P.sizes.assign(L, 0);
  std::vector<int64_t> by_len(L + 1, 0);
  for (uint32_t i = 0; i < s; ++i) by_len[P.lens[i]] += P.hist[i];
  int64_t longer = 0;
  for (uint32_t l = L; l-- > 0;) {
    longer += by_len[l + 1];
    P.sizes[l] = longer;
  }
  P.offsets.assign(L, 0);
  uint64_t cursor = 0;
  for (uint32_t l = 0; l < L; ++l) {
    P.offsets[l] = (int64_t)cursor;
    cursor = (cursor + (uint64_t)P.sizes[l] + kAlignBits - 1) / kAlignBits * kAlignBits;
  }
  P.n_words = L ? ((uint64_t)P.offsets[L - 1] + (uint64_t)P.sizes[L - 1] + 63) / 64 : 0;
  // node tables, level by level (wtree.py:388-433); keys are code prefixes
  P.node_off.assign(L + 1, 0);
  for (uint32_t l = 0; l < L; ++l) P.node_off[l + 1] = P.node_off[l] + (1ull << l);
  P.nodes.swap(node_cache());  // reuse the last build's pages (given back after the upload)
  P.nodes.assign(P.node_off[L], NodeEnt{0, 0, {-1, -1}});
  plan_walk(P, false, walk_levels);
  P.code_bytes = L <= 8 ? 1 : 2;
}

// ---------------------------------------------------------------------------
// the tree handle
// ---------------------------------------------------------------------------
struct LevelHost {
  wt_level_meta meta;
  u64* l1 = nullptr;
  u16* l2 = nullptr;
  u64* ones = nullptr;
  u64* zeros = nullptr;
  // query-side rank-line layout (wt_qlayout.cu)
  ulonglong2* lines = nullptr;
  u32* sel1 = nullptr;
  u32* sel0 = nullptr;
  u64 n_lines = 0, sel_cap = 0;
};

struct wt_tree {
  int device = 0;
  wt_meta meta{};
  Plan plan;
  std::vector<LevelHost> lv;
  u64* words = nullptr;
  NodeEnt* nodes = nullptr;
  u32* id_code = nullptr;
  i64* cum = nullptr;
  u16* symbols = nullptr;
  int* sym2id = nullptr;
  u64* bad = nullptr;  // first invalid query index (device scalar)
  u8* arena = nullptr;  // every level's directory / line arrays (one allocation)
  TreeDev dev{};
  int rate_log = -1;
  cudaStream_t stream = nullptr;
  // query staging (reused across calls)
  void* qbuf[2] = {nullptr, nullptr};
  size_t qbuf_bytes = 0;
  cudaStream_t qstream[3] = {nullptr, nullptr, nullptr};  // copy-in, compute, copy-out
  cudaEvent_t qev[3][2] = {};                              // per stage and slot
  std::vector<cudaEvent_t> tev;                            // pipeline timing events (stats)
  // narrow wire format: pinned host staging per slot (u32 args, u16 symbols)
  // and "the copy-in of the slot's last packed chunk has finished" events
  void* hst[2] = {nullptr, nullptr};
  size_t hst_bytes = 0;
  cudaEvent_t hev[2] = {nullptr, nullptr};
  std::mutex qmutex;
  std::mutex tables_mutex;
  u32 sel_kbits = 0;        // select_kbits() cache  // lazy node_starts / node_rank0 (wt_tree_get)
  // build profile: [0] text upload + histogram + plan, [1 + l] level-l kernel (ms)
  std::vector<float> build_ms;
};

static int rate_log_of(uint64_t rate) {
  if (rate && (rate & (rate - 1)) == 0) {
    int r = 0;
    while ((1ull << r) < rate) ++r;
    return r;
  }
  return -1;
}

static void fill_treedev(wt_tree* t) {
  TreeDev& D = t->dev;
  memset(&D, 0, sizeof(D));
  const Plan& P = t->plan;
  for (uint32_t l = 0; l < P.L; ++l) {
    LevelDev& d = D.lv[l];
    const LevelHost& h = t->lv[l];
    d.words = t->words + (P.offsets[l] >> 6);
    d.l1 = h.l1;
    d.l2 = h.l2;
    d.ones = h.ones;
    d.zeros = h.zeros;
    d.nodes = t->nodes + P.node_off[l];
    d.n_bits = h.meta.n_bits;
    d.total_ones = h.meta.total_ones;
    d.n_ones = h.meta.n_ones;
    d.n_zeros = h.meta.n_zeros;
    d.n_l1 = h.meta.n_l1;
    d.n_l2 = h.meta.n_l2;
    QLevelDev& q = D.ql[l];
    q.lines = h.lines;
    q.sel1 = h.sel1;
    q.sel0 = h.sel0;
    q.n_lines = h.n_lines;
    q.n_bits = h.meta.n_bits;
    q.total_ones = h.meta.total_ones;
    q.n_sel1 = h.meta.total_ones ? ((h.meta.total_ones - 1) >> kQSelLog) + 1 : 0;
    const u64 z = h.meta.n_bits - h.meta.total_ones;
    q.n_sel0 = z ? ((z - 1) >> kQSelLog) + 1 : 0;
  }
  D.id_code = t->id_code;
  D.cum = t->cum;
  D.symbols = t->symbols;
  D.sym2id = t->sym2id;
  D.n = t->meta.n;
  D.L = P.L;
  D.sigma = P.sigma;
  uint32_t sh = 0;
  while ((1u << sh) < t->meta.l2_bits) ++sh;
  D.l2_shift = sh;
  D.width = t->meta.symbol_width;
  D.rate = t->meta.sample_rate;
  t->rate_log = rate_log_of(t->meta.sample_rate);
}

// allocate the per-level directories and upload the O(sigma) tables
// Device arrays of a tree.  The build path splits this so the GPU never waits
// on the host: alloc_tree_core (bit array, node table) before level 0,
// alloc_level(l) inside the level loop (stream-ordered allocations the host
// makes while earlier levels run), alloc_query_tables after the last launch
// (its uploads run on a side stream from pinned staging, overlapping the
// levels).  alloc_tree does all three synchronously (load / replicate).
static int alloc_tree_core(wt_tree* t, cudaStream_t st, uint64_t node_upload = ~0ull) {
  const Plan& P = t->plan;
  t->lv.assign(P.L, LevelHost{});
  for (uint32_t l = 0; l < P.L; ++l) {
    LevelHost& h = t->lv[l];
    const uint64_t m = (uint64_t)P.sizes[l];
    h.meta.n_bits = m;
    h.meta.n_l1 = (m + kL1Bits - 1) / kL1Bits;
    h.meta.n_l2 = (m + t->meta.l2_bits - 1) / t->meta.l2_bits;
    h.meta.n_nodes = P.n_nodes[l];
    h.n_lines = qlayout_lines(m);
    h.sel_cap = (m >> kQSelLog) + 2;
  }
  TRY(dalloc(&t->words, P.n_words, st));
  // every level's directory / line arrays carved from ONE allocation: one
  // stream-ordered allocation call instead of seven per level, and the same
  // pool footprint build after build
  {
    auto al = [](uint64_t b) { return (b + 255) & ~255ull; };
    uint64_t need = 0;
    for (auto& h : t->lv) {
      const uint64_t m = h.meta.n_bits, ns = m / t->meta.sample_rate;
      need += al(h.meta.n_l1 * 8) + al(h.meta.n_l2 * 2) + 2 * al(std::max<uint64_t>(ns, 1) * 8) +
              al(h.n_lines * kQLineBytes) + 2 * al(h.sel_cap * 4);
    }
    TRY(dalloc(&t->arena, std::max<uint64_t>(need, 1), st));
    uint64_t o = 0;
    auto take = [&](auto*& p, uint64_t bytes) {
      p = reinterpret_cast<std::remove_reference_t<decltype(p)>>(t->arena + o);
      o += al(bytes);
    };
    for (auto& h : t->lv) {
      const uint64_t m = h.meta.n_bits, ns = m / t->meta.sample_rate;
      take(h.l1, h.meta.n_l1 * 8);
      take(h.l2, h.meta.n_l2 * 2);
      take(h.ones, std::max<uint64_t>(ns, 1) * 8);
      take(h.zeros, std::max<uint64_t>(ns, 1) * 8);
      take(h.lines, h.n_lines * kQLineBytes);
      take(h.sel1, h.sel_cap * 4);
      take(h.sel0, h.sel_cap * 4);
    }
  }
  TRY(dalloc(&t->nodes, P.nodes.size(), st));
  // (pageable source: the call returns once the bytes are staged)
  const uint64_t nup = std::min<uint64_t>(P.nodes.size(), node_upload);
  if (nup)
    CU(cudaMemcpyAsync(t->nodes, P.nodes.data(), nup * sizeof(NodeEnt), cudaMemcpyHostToDevice, st));
  uint64_t bytes = P.n_words * 8 + P.nodes.size() * sizeof(NodeEnt) + P.sigma * 14 + 8;
  for (auto& h : t->lv)
    bytes += h.meta.n_l1 * 8 + h.meta.n_l2 * 2 + 2 * (h.meta.n_bits / t->meta.sample_rate) * 8 +
             h.n_lines * kQLineBytes + 2 * h.sel_cap * 4;
  t->meta.device_bytes = bytes;
  return WT_OK;
}

static int alloc_level(wt_tree* t, uint32_t l, cudaStream_t st) {
  LevelHost& h = t->lv[l];
  if (h.l1) return WT_OK;
  const uint64_t m = h.meta.n_bits;
  TRY(dalloc(&h.l1, h.meta.n_l1, st));
  TRY(dalloc(&h.l2, h.meta.n_l2, st));
  TRY(dalloc(&h.ones, m / t->meta.sample_rate, st));
  TRY(dalloc(&h.zeros, m / t->meta.sample_rate, st));
  TRY(dalloc(&h.lines, h.n_lines * kQLineU2, st));
  TRY(dalloc(&h.sel1, h.sel_cap, st));
  TRY(dalloc(&h.sel0, h.sel_cap, st));
  return WT_OK;
}

// pinned host staging for the query-table uploads (thread-local, grows)
static void* pinned_staging(size_t bytes) {
  static thread_local void* p = nullptr;
  static thread_local size_t cap = 0;
  if (bytes > cap) {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    cap = bytes;
  }
  return p;
}

// query-side tables (symbol -> id, id -> code, cum_hist, symbols); with a
// side stream the uploads run there (from pinned staging) and `st` waits for
// them at its current end (or, given `join`, wherever the caller waits on the
// returned event); without one they run on `st` and the call syncs.
static int alloc_query_tables(wt_tree* t, cudaStream_t st, cudaStream_t side,
                              cudaEvent_t* join = nullptr) {
  const Plan& P = t->plan;
  TRY(dalloc(&t->id_code, P.sigma, st));
  TRY(dalloc(&t->cum, P.sigma + 1, st));
  TRY(dalloc(&t->symbols, P.sigma, st));
  TRY(dalloc(&t->sym2id, 65536, st));
  TRY(dalloc(&t->bad, 1, st));
  const size_t b_s2i = 65536 * 4, b_idc = (size_t)P.sigma * 4, b_cum = P.cum.size() * 8,
               b_sym = P.symbols.size() * 2;
  u8* stage = side ? (u8*)pinned_staging(b_s2i + b_idc + b_cum + b_sym) : nullptr;
  static thread_local std::vector<u8> pageable;
  if (!stage) {
    side = nullptr;
    pageable.resize(b_s2i + b_idc + b_cum + b_sym);
    stage = pageable.data();
  }
  int* s2i = reinterpret_cast<int*>(stage);
  for (uint32_t s = 0; s < 65536; ++s) s2i[s] = -1;
  for (uint32_t i = 0; i < P.sigma; ++i) s2i[P.symbols[i]] = (int)i;
  u32* idc = reinterpret_cast<u32*>(stage + b_s2i);
  for (uint32_t i = 0; i < P.sigma; ++i) idc[i] = P.values[i] | ((u32)P.lens[i] << 16);
  memcpy(stage + b_s2i + b_idc, P.cum.data(), b_cum);
  memcpy(stage + b_s2i + b_idc + b_cum, P.symbols.data(), b_sym);
  cudaStream_t cs = side ? side : st;
  cudaEvent_t ready = nullptr, done = nullptr;
  if (side) {  // the side stream may touch the allocations once `st` reaches them
    CU(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    CU(cudaEventRecord(ready, st));
    CU(cudaStreamWaitEvent(side, ready, 0));
  }
  CU(cudaMemcpyAsync(t->sym2id, s2i, b_s2i, cudaMemcpyHostToDevice, cs));
  CU(cudaMemcpyAsync(t->id_code, idc, b_idc, cudaMemcpyHostToDevice, cs));
  CU(cudaMemcpyAsync(t->cum, stage + b_s2i + b_idc, b_cum, cudaMemcpyHostToDevice, cs));
  CU(cudaMemcpyAsync(t->symbols, stage + b_s2i + b_idc + b_cum, b_sym, cudaMemcpyHostToDevice, cs));
  if (side) {
    CU(cudaEventRecord(done, side));
    cudaEventDestroy(ready);
    if (join) {  // the caller joins `st` to the uploads later
      *join = done;
    } else {
      CU(cudaStreamWaitEvent(st, done, 0));
      cudaEventDestroy(done);
    }
  } else {
    CU(cudaStreamSynchronize(st));  // pageable staging is reused by the next call
  }
  return WT_OK;
}

static int finish_tables(wt_tree* t) {
  node_cache().swap(t->plan.nodes);  // the device holds the node table now
  t->plan.nodes.clear();
  return WT_OK;
}

static int alloc_tree(wt_tree* t, cudaStream_t st) {
  TRY(alloc_tree_core(t, st));
  for (uint32_t l = 0; l < t->plan.L; ++l) TRY(alloc_level(t, l, st));
  TRY(alloc_query_tables(t, st, nullptr));
  return finish_tables(t);
}

// query-side layout of every level; totals_dev[l] = ones of level l (device)
static int launch_qlayouts(wt_tree* t, const u64* totals_dev, cudaStream_t st,
                           const std::vector<char>* done = nullptr) {
  const Plan& P = t->plan;
  uint32_t sh = 0;
  while ((1u << sh) < t->meta.l2_bits) ++sh;
  for (uint32_t l = 0; l < P.L; ++l) {
    if (done && l < done->size() && (*done)[l]) continue;  // written by dirq_kernel
    LevelHost& h = t->lv[l];
    LevelDev d{};
    d.words = t->words + (P.offsets[l] >> 6);
    d.l1 = h.l1;
    d.l2 = h.l2;
    d.n_bits = h.meta.n_bits;
    d.n_l1 = h.meta.n_l1;
    d.n_l2 = h.meta.n_l2;
    CU(launch_qlayout(d, totals_dev + l, sh, h.lines, h.n_lines, h.sel1, h.sel_cap, h.sel0,
                      h.sel_cap, st));
  }
  return WT_OK;
}

// host-known totals -> device, then the query layout (load / replicate paths)
static int qlayouts_from_host_totals(wt_tree* t, cudaStream_t st) {
  const Plan& P = t->plan;
  if (!P.L) return WT_OK;
  std::vector<u64> tot(P.L);
  for (uint32_t l = 0; l < P.L; ++l) tot[l] = t->lv[l].meta.total_ones;
  u64* d;
  CU(cudaMalloc(&d, P.L * 8));
  cudaError_t e = cudaMemcpyAsync(d, tot.data(), P.L * 8, cudaMemcpyHostToDevice, st);
  int rc = e == cudaSuccess ? launch_qlayouts(t, d, st) : fail(WT_ERR_CUDA, cudaGetErrorString(e));
  if (rc == WT_OK) {
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(WT_ERR_CUDA, cudaGetErrorString(e));
  }
  cudaFree(d);
  return rc;
}

static void free_tree_arrays(wt_tree* t) {
  cudaSetDevice(t->device);
  // the tree's arrays come from the stream-ordered pool (cudaMallocAsync):
  // once the device is idle they go back to the pool with cudaFreeAsync, so
  // the pool stays mapped for the next build (freeing them with cudaFree
  // measured 10 ms .. 1.4 s pre-phase stalls in later builds, the pool
  // re-growing); the query slots (cudaMalloc) keep cudaFree
  const bool idle = cudaDeviceSynchronize() == cudaSuccess;
  auto F = [idle](void* p) {
    if (!p) return;
    if (idle && cudaFreeAsync(p, 0) == cudaSuccess) return;
    cudaGetLastError();  // (not pool memory: clear the error, free it plainly)
    cudaFree(p);
  };
  auto Fsync = [](void* p) {
    if (p) cudaFree(p);
  };
  F(t->words);
  for (auto& h : t->lv) {
    if (!t->arena) {  // (carved from the arena otherwise)
      F(h.l1);
      F(h.l2);
      F(h.ones);
      F(h.zeros);
      F(h.lines);
      F(h.sel1);
      F(h.sel0);
    }
  }
  F(t->nodes);
  F(t->id_code);
  F(t->cum);
  F(t->symbols);
  F(t->sym2id);
  F(t->bad);
  F(t->arena);
  Fsync(t->qbuf[0]);
  Fsync(t->qbuf[1]);
  for (auto& s : t->qstream)
    if (s) cudaStreamDestroy(s);
  for (auto& a : t->qev)
    for (auto& e : a)
      if (e) cudaEventDestroy(e);
  for (auto& e : t->tev) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (t->hev[i]) cudaEventDestroy(t->hev[i]);
    if (t->hst[i]) cudaFreeHost(t->hst[i]);
  }
  if (t->stream) cudaStreamDestroy(t->stream);
}

static int check_params(uint32_t l2_bits, uint64_t rate) {
  if (l2_bits < 64 || (l2_bits & (l2_bits - 1)) || l2_bits > (uint32_t)kL1Bits)
    return fail(WT_ERR_ARG, "l2_bits must be a power of two in [64, 65536]");
  if (rate < 1) return fail(WT_ERR_ARG, "sample_rate must be positive");
  return WT_OK;
}

// ---------------------------------------------------------------------------
// construction
// ---------------------------------------------------------------------------
struct Scratch {
  std::vector<void*> ptrs;
  cudaStream_t st;
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  template <typename T>
  int get(T** p, size_t count) {
    int s = dalloc(p, count, st);
    if (s == WT_OK) ptrs.push_back(*p);
    return s;
  }
};

extern "C" int wt_construct(const void* text, uint64_t n, int sym_bytes, int text_on_device,
                            const uint16_t* alphabet, uint32_t alphabet_len, int symbol_width,
                            uint32_t l2_bits, uint64_t sample_rate, int device, void* stream,
                            wt_tree** out, float* ms_out) {
  g_err_index = -1;
  if (!out) return fail(WT_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (n == 0) return fail(WT_ERR_BUILD, "cannot build an index over an empty text");
  if (sym_bytes != 1 && sym_bytes != 2) return fail(WT_ERR_ARG, "sym_bytes must be 1 or 2");
  if (symbol_width != 1 && symbol_width != 2) return fail(WT_ERR_ARG, "symbol_width must be 1 or 2");
  TRY(check_params(l2_bits, sample_rate));
  if (alphabet && alphabet_len == 0) return fail(WT_ERR_BUILD, "declared alphabet is empty");
  if (text_on_device && ((uintptr_t)text & 15))
    return fail(WT_ERR_ARG, "device text must be 16-byte aligned");
  TRY(setup_device(device));
  wt_tree* t = new wt_tree();
  t->device = device;
  int rc = WT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (!st) {
    if (cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete t;
      return fail(WT_ERR_CUDA, "stream create failed");
    }
    st = t->stream;
  }
  auto body = [&]() -> int {
    Scratch S{{}, st};
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    struct EvGuard { cudaEvent_t a, b; ~EvGuard() { cudaEventDestroy(a); cudaEventDestroy(b); } } eg{e0, e1};
    Tracer tr;
    CU(cudaEventRecord(e0, st));
    const void* dtext = text;
    if (!text_on_device) {
      u8* p;
      TRY(S.get(&p, n * sym_bytes));
      CU(cudaMemcpyAsync(p, text, n * sym_bytes, cudaMemcpyHostToDevice, st));
      dtext = p;
    }
    const int nb = sym_bytes == 1 ? 256 : 65536;
    u64* dhist;
    TRY(S.get(&dhist, nb));
    CU(cudaMemsetAsync(dhist, 0, nb * 8, st));
    // Large u8 texts: K1 also keeps the histogram of every L1 block, from
    // which level 0's L1 counts follow once the plan fixes the top-bit
    // threshold, and level 0 runs in block mode (no counting pass over the
    // text).  Enough blocks to keep every resident warp of the level kernel
    // busy are required: a warp walks whole blocks.
    const uint64_t n_blk = (n + 65535) >> 16;
    u32* dbh = nullptr;
    // (WT_BLOCK_MODE=0|1 forces it off / on: the parity tests run both)
    const char* bm = getenv("WT_BLOCK_MODE");
    const bool want_blocks = bm ? bm[0] == '1' : n_blk >= 2 * wlevel_warp_slots(sm_count(device));
    if (want_blocks && sym_bytes == 1) TRY(S.get(&dbh, n_blk * 256));
    if (want_blocks && sym_bytes == 2) {  // level 0 in block mode when its threshold is 32768
      TRY(S.get(&dbh, n_blk + 4));
      CU(cudaMemsetAsync(dbh, 0, (n_blk + 4) * 4, st));
    }
    tr.mark("histogram inputs allocated");
    CU(launch_histogram(dtext, n, sym_bytes, dhist, sm_count(device), st, dbh));
    tr.mark("histogram kernels queued");
    static thread_local std::vector<uint64_t> hraw;
    hraw.assign(nb, 0);
    CU(cudaMemcpyAsync(hraw.data(), dhist, nb * 8, cudaMemcpyDeviceToHost, st));
    tr.mark("histogram launched");
    CU(cudaStreamSynchronize(st));
    tr.mark("histogram done");

    Plan& P = t->plan;
    if (alphabet) {
      P.symbols.assign(alphabet, alphabet + alphabet_len);
      // every present symbol must be declared (alphabet.py:76-84)
      std::vector<u8> member(nb, 0);
      bool ok = true;
      for (uint32_t i = 0; i < alphabet_len; ++i)
        if (alphabet[i] < nb) member[alphabet[i]] = 1;
      for (int s = 0; s < nb; ++s)
        if (hraw[s] && !member[s]) ok = false;
      if (!ok) {
        u8* dm;
        u64* dbest;
        TRY(S.get(&dm, nb));
        TRY(S.get(&dbest, 1));
        CU(cudaMemcpyAsync(dm, member.data(), nb, cudaMemcpyHostToDevice, st));
        CU(cudaMemsetAsync(dbest, 0xff, 8, st));
        CU(launch_first_outside(dtext, n, sym_bytes, dm, dbest, sm_count(device), st));
        uint64_t best = 0;
        CU(cudaMemcpyAsync(&best, dbest, 8, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        uint32_t bad_sym = 0;
        CU(cudaMemcpy(&bad_sym, (const u8*)dtext + best * sym_bytes, sym_bytes,
                      cudaMemcpyDeviceToHost));
        g_err_index = (int64_t)best;
        char buf[160];
        snprintf(buf, sizeof buf, "symbol %u at position %llu is not in the alphabet", bad_sym,
                 (unsigned long long)best);
        return fail(WT_ERR_SYMBOL, buf);
      }
    } else {
      for (int s = 0; s < nb; ++s)
        if (hraw[s]) P.symbols.push_back((uint16_t)s);
    }
    P.sigma = (uint32_t)P.symbols.size();
    if (P.sigma > 65536) return fail(WT_ERR_BUILD, "alphabet size exceeds 65536");
    P.L = ceil_log2_u(P.sigma);
    P.hist.assign(P.sigma, 0);
    for (uint32_t i = 0; i < P.sigma; ++i)
      if (P.symbols[i] < nb) P.hist[i] = (int64_t)hraw[P.symbols[i]];
    tr.mark("alphabet done");
    plan_codes(P);
    tr.mark("codes done");
    // Levels >= 1 of the node table (O(sigma), ~0.6 ms at sigma = 2^16) are
    // walked on the host while level 0 runs: level 0 reads only the root.
    // (L <= 2: level 0 is part of the pair pass, which reads level 1 too.)
    const bool defer_walk = P.L >= 3 && !(getenv("WT_DEFER_WALK") && getenv("WT_DEFER_WALK")[0] == '0');
    plan_shape(P, l2_bits, defer_walk ? 1u : ~0u);
    tr.mark("plan done");

    t->meta.n = n;
    t->meta.sigma = P.sigma;
    t->meta.levels = P.L;
    t->meta.symbol_width = (uint32_t)symbol_width;
    t->meta.l2_bits = l2_bits;
    t->meta.sample_rate = sample_rate;
    t->meta.first_coded = P.first_coded;
    t->meta.device = (uint32_t)device;
    t->meta.n_words = P.n_words;
    {
      // grow the stream-ordered pool once for the whole build (tree + scratch)
      // instead of in many small steps; a no-op once the pool is warm
      uint64_t est = P.n_words * 8 + 64ull * 1024 * 1024;
      for (uint32_t l = 0; l < P.L; ++l) {
        const uint64_t m = (uint64_t)P.sizes[l];
        est += m * kQLineBytes / kQBits + m / 32 + m / 256 + 2 * (m / sample_rate) * 8 + (m >> kQSelLog) * 8;
        if (l == 1 || l == 2) est += m * P.code_bytes;
      }
      void* probe = nullptr;
      if (cudaMallocAsync(&probe, est, st) == cudaSuccess) cudaFreeAsync(probe, st);
      else cudaGetLastError();
      tr.mark("pool probe");
    }
    TRY(alloc_tree_core(t, st, defer_walk ? 1ull : ~0ull));
    tr.mark("tree allocated");
    // query tables: uploads on a side stream (pinned staging) once level 0 is
    // queued, so they overlap the levels; `st` joins them at its end
    bool tables_done = false;
    cudaEvent_t tables_join = nullptr;
    struct JoinGuard { cudaEvent_t& e; ~JoinGuard() { if (e) cudaEventDestroy(e); } } jg{tables_join};
    auto query_tables = [&]() -> int {
      cudaStream_t side = nullptr;
      if (cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        side = nullptr;
      }
      const int qrc = alloc_query_tables(t, st, side, &tables_join);
      if (side) cudaStreamDestroy(side);  // (released once its work is done)
      tables_done = true;
      return qrc;
    };

    // raw symbol -> code LUT for level 0, unless the map is the identity
    static thread_local std::vector<u16> lut;
    lut.assign(nb, 0);
    bool identity = true;
    for (uint32_t i = 0; i < P.sigma; ++i) {
      if (P.symbols[i] >= nb) continue;
      lut[P.symbols[i]] = P.values[i];
      if (P.hist[i] && P.values[i] != P.symbols[i]) identity = false;
    }
    if (P.code_bytes != sym_bytes) identity = false;
    u16* dlut = nullptr;
    if (!identity && P.L) {
      TRY(S.get(&dlut, nb));
      CU(cudaMemcpyAsync(dlut, lut.data(), nb * 2, cudaMemcpyHostToDevice, st));
    }

    // zero the alignment gaps between regions (regions themselves are fully written)
    for (uint32_t l = 0; l < P.L; ++l) {
      const uint64_t end_w = ((uint64_t)P.offsets[l] + (uint64_t)P.sizes[l] + 63) / 64;
      const uint64_t next_w = l + 1 < P.L ? (uint64_t)P.offsets[l + 1] / 64 : P.n_words;
      if (next_w > end_w) CU(cudaMemsetAsync(t->words + end_w, 0, (next_w - end_w) * 8, st));
    }

    uint32_t l2_log = 0;
    while ((1u << l2_log) < l2_bits) ++l2_log;
    std::vector<cudaEvent_t> lev(P.L + 1);
    for (auto& e : lev) CU(cudaEventCreate(&e));
    struct EvVec { std::vector<cudaEvent_t>& v; ~EvVec() { for (auto e : v) cudaEventDestroy(e); } } evg{lev};
    u64* totals;
    TRY(S.get(&totals, std::max<uint32_t>(P.L, 1)));
    CU(cudaMemsetAsync(totals, 0, std::max<uint32_t>(P.L, 1) * 8, st));
    void* cur[2] = {nullptr, nullptr};
    if (P.L >= 2) {
      u8* p;
      TRY(S.get(&p, (uint64_t)P.sizes[1] * P.code_bytes + 16));
      cur[0] = p;
    }
    if (P.L >= 3) {
      u8* p;
      TRY(S.get(&p, (uint64_t)P.sizes[2] * P.code_bytes + 16));
      cur[1] = p;
    }
    std::vector<char> q_done(P.L, 0);  // levels whose query layout dirq_kernel wrote
    {
      // K2w: warp tiles; per-tile and per-L1-block ones counts of each level
      // come from the previous level's scatter (level 0: a counting pass)
      uint64_t max_tiles = 1, max_l1 = 1;
      for (uint32_t l = 0; l < P.L; ++l) {
        max_tiles = std::max<uint64_t>(
            max_tiles, wlevel_tiles((uint64_t)P.sizes[l], l == 0 ? sym_bytes : P.code_bytes));
        max_l1 = std::max<uint64_t>(max_l1, t->lv[l].meta.n_l1);
      }
      u32 *tcnt[2], *l1cnt[2];
      for (int i = 0; i < 2; ++i) {
        TRY(S.get(&tcnt[i], max_tiles + 64));
        TRY(S.get(&l1cnt[i], max_l1 + 4));
      }
      // level-0 bit = top code bit = (symbol >= thr): codes are monotone in the symbol
      uint32_t thr = 0x10000u;
      for (uint32_t i = 0; i < P.sigma; ++i)
        if ((P.values[i] >> (P.L - 1)) & 1u) {
          thr = P.symbols[i];
          break;
        }
      const bool block_mode = dbh && P.L >= 2 && (sym_bytes == 1 || thr == 32768u);
      // Levels >= 1 stay in block mode while every resident warp still gets
      // two L1 blocks (one warp walks a whole block: P1 is the block's L1 entry
      // plus a running count); a level whose successor is also in block mode
      // counts the successor's ones per L1 block only, in its first pass.
      // The last level (wlast) reads per-tile counts.
      std::vector<char> blk(P.L, 0);
      {
        const uint64_t slots2 = 2 * wlevel_warp_slots(sm_count(device));
        const char* bl = getenv("WT_BLK_LEVELS");  // "0": levels >= 1 in tile mode (A/B)
        for (uint32_t l = 0; l < P.L; ++l) {
          const bool big = (bm ? bm[0] == '1' : t->lv[l].meta.n_l1 >= slots2) && !(bl && bl[0] == '0');
          blk[l] = l == 0 ? block_mode : (blk[l - 1] && big && l + 1 < P.L);
        }
      }
      // next level's bit at a LUT level 0: parity of (symbol >= nthr[i]) over
      // the first symbols whose code's top two bits reach 1, 2, 3
      uint32_t nthr[3] = {0x10000u, 0x10000u, 0x10000u};
      if (P.L >= 2)
        for (uint32_t i = P.sigma; i-- > 0;) {
          const uint32_t cls = (P.values[i] >> (P.L - 2)) & 3u;
          for (uint32_t k = 1; k <= cls; ++k) nthr[k - 1] = P.symbols[i];
        }
      if (P.L && P.sizes[0]) {
        CU(cudaMemsetAsync(l1cnt[0], 0, (t->lv[0].meta.n_l1 + 4) * 4, st));
        if (block_mode && sym_bytes == 1)
          CU(launch_block_l1(dbh, n_blk, thr, l1cnt[0], st));
        else if (block_mode)  // u16: K1 counted the symbols >= 32768 per block
          CU(cudaMemcpyAsync(l1cnt[0], dbh, n_blk * 4, cudaMemcpyDeviceToDevice, st));
        else
          CU(launch_wcount0(dtext, n, sym_bytes, thr, tcnt[0], l1cnt[0], sm_count(device), st));
      }
      // Pair mode for the last two levels (every code reaches the last level):
      // one pass over level L-2 writes its bits and, from the staged runs,
      // the last level's bits -- no partitioned sequence, no last-level pass.
      // (WT_PAIR=0 turns it off: the parity tests run both.)
      const char* pe = getenv("WT_PAIR");
      const bool pair_ok = !(pe && pe[0] == '0');
      const char* de = getenv("WT_DIR");
      const char* qe = getenv("WT_DIRQ");
      // After each level's kernel, dirq_kernel writes its L2 entries + select
      // samples together with its query lines (one streaming pass over the
      // level's bits).  WT_DIRQ=0: dir_kernel for the directory (WT_DIR=0:
      // inside the level kernel) and qlayout_kernel for the lines (A/B)
      const bool dirq_on = !(qe && qe[0] == '0');
      const bool dir_after = dirq_on || !(de && de[0] == '0');
      auto level_dir = [&](uint32_t lv, const u64* words, bool pdl) -> int {
        LevelHost& hl = t->lv[lv];
        const uint64_t mm = hl.meta.n_bits;
        DirParams dp{};
        dp.words = words;
        dp.m = mm;
        dp.l1 = hl.l1;
        dp.l2 = hl.l2;
        dp.ones = hl.ones;
        dp.zeros = hl.zeros;
        dp.ones_cap = mm / sample_rate;
        dp.zeros_cap = mm / sample_rate;
        dp.l2_log = l2_log;
        dp.rate_log = rate_log_of(sample_rate);
        dp.rate = sample_rate;
        if (!dirq_on) {
          CU(launch_dir(dp, sm_count(device), st));
          return WT_OK;
        }
        DirQParams q{};
        q.d = dp;
        q.total = totals + lv;
        q.lines = hl.lines;
        q.n_lines = hl.n_lines;
        q.sel1 = hl.sel1;
        q.sel0 = hl.sel0;
        q.cap1 = hl.sel_cap;
        q.cap0 = hl.sel_cap;
        CU(launch_dirq(q, sm_count(device), st, pdl));
        q_done[lv] = 1;
        return WT_OK;
      };
      // L1 directory of level lv from its per-L1-block counts (l1cnt[cidx])
      std::vector<char> scanned(P.L + 1, 0);
      auto scan_level = [&](uint32_t lv, int cidx) -> int {
        TRY(alloc_level(t, lv, st));
        LevelHost& hs = t->lv[lv];
        CU(launch_l1_scan(l1cnt[cidx], hs.meta.n_l1, hs.l1, totals + lv, st));
        scanned[lv] = 1;
        return WT_OK;
      };
      int ci = 0;
      for (uint32_t l = 0; l < P.L; ++l) {
        if (l == 1 && defer_walk) {  // level 0 is queued: the rest of the node table
          plan_walk(P, false);
          for (uint32_t k = 0; k < P.L; ++k) t->lv[k].meta.n_nodes = P.n_nodes[k];
          // (pageable source: staged before the call returns; stream order
          // puts the copy ahead of level 1)
          CU(cudaMemcpyAsync(t->nodes, P.nodes.data(), P.nodes.size() * sizeof(NodeEnt),
                             cudaMemcpyHostToDevice, st));
          tr.mark("node table walked");
        }
        if (l == 1 && !tables_done) TRY(query_tables());  // level 0 is queued: overlap it
        const uint64_t m = (uint64_t)P.sizes[l];
        CU(cudaEventRecord(lev[l], st));
        if (m == 0) continue;
        const int in_bytes = l == 0 ? sym_bytes : P.code_bytes;
        LevelHost& h = t->lv[l];
        TRY(alloc_level(t, l, st));
        if (!scanned[l]) TRY(scan_level(l, ci));
        const bool pair = pair_ok && l + 2 == P.L && (uint64_t)P.sizes[l + 1] == m;
        const bool next_blk = !pair && l + 1 < P.L && blk[l] && blk[l + 1];
        WLevelParams wp{};
        wp.in = l == 0 ? dtext : cur[(l - 1) & 1];
        wp.out = l + 1 < P.L && !pair ? cur[l & 1] : nullptr;
        wp.m = m;
        wp.m_next = l + 1 < P.L ? (uint64_t)P.sizes[l + 1] : 0;
        if (wp.out && wp.m_next == 0) wp.out = nullptr;
        if (pair) {
          const uint64_t w0 = (uint64_t)P.offsets[l + 1] / 64;
          const uint64_t w1 = ((uint64_t)P.offsets[l + 1] + wp.m_next + 63) / 64;
          CU(cudaMemsetAsync(t->words + w0, 0, (w1 - w0) * 8, st));
          CU(cudaMemsetAsync(l1cnt[ci ^ 1], 0, (t->lv[l + 1].meta.n_l1 + 4) * 4, st));
          wp.next_words = t->words + w0;
        }
        if (wp.out) {
          const uint64_t nt = wlevel_tiles(wp.m_next, P.code_bytes);
          if (!next_blk) CU(cudaMemsetAsync(tcnt[ci ^ 1], 0, (nt + 64) * 4, st));
          CU(cudaMemsetAsync(l1cnt[ci ^ 1], 0, (t->lv[l + 1].meta.n_l1 + 4) * 4, st));
        }
        wp.words = t->words + (P.offsets[l] >> 6);
        wp.l2 = h.l2;
        wp.ones = h.ones;
        wp.zeros = h.zeros;
        wp.ones_cap = m / sample_rate;
        wp.zeros_cap = m / sample_rate;
        wp.nodes = t->nodes + P.node_off[l];
        wp.lut = l == 0 ? dlut : nullptr;
        wp.l1 = h.l1;
        wp.tile_counts = blk[l] ? nullptr : tcnt[ci];
        wp.next_block = next_blk && wp.out ? 1 : 0;
        for (int i = 0; i < 3; ++i) wp.nthr[i] = nthr[i];
        wp.next_tile_counts = tcnt[ci ^ 1];
        wp.next_l1_counts = l1cnt[ci ^ 1];
        wp.thr = thr;
        wp.shift_bit = P.L - 1 - l;
        wp.shift_key = P.L - l;
        wp.l2_log = l2_log;
        wp.rate_log = rate_log_of(sample_rate);
        wp.rate = sample_rate;
        // L2 entries / samples of a partitioning level by dir_kernel after the
        // launch (a streaming pass over its bits) instead of inside the level
        // kernel (WT_DIR=0: inside)
        wp.skip_dir = dir_after && wp.out ? 1 : 0;
        wp.plut_shift = 0xffu;
        if (l == 0 && dlut && sym_bytes == 1 && P.sigma <= 8) {
          // a shift making (symbol >> s) & 7 distinct over the alphabet: the
          // codes then come from an 8-byte register table (pair kernel)
          for (uint32_t sh = 0; sh <= 5 && wp.plut_shift == 0xffu; ++sh) {
            uint32_t seen = 0, lo = 0, hi = 0;
            bool ok = true;
            for (uint32_t i = 0; i < P.sigma && ok; ++i) {
              const uint32_t ix = (P.symbols[i] >> sh) & 7u;
              ok = !((seen >> ix) & 1u);
              seen |= 1u << ix;
              const uint32_t code = P.values[i] & 0xffu;
              if (ix < 4) lo |= code << (8 * ix); else hi |= code << (8 * (ix - 4));
            }
            if (ok) {
              wp.plut_shift = sh;
              wp.plut_lo = lo;
              wp.plut_hi = hi;
            }
          }
        }
        CU(launch_wlevel(wp, in_bytes, P.code_bytes, l == 0 && dlut != nullptr, sm_count(device), st));
        ci ^= 1;
        // The next level's L1 scan (its counts came from this level's kernel)
        // goes ahead of this level's directory pass, which is launched as its
        // programmatic dependent: the one-CTA scan overlaps the streaming pass.
        bool pdl = false;
        if (dirq_on && l + 1 < P.L && P.sizes[l + 1] && (wp.out || pair)) {
          TRY(scan_level(l + 1, ci));
          pdl = true;
        }
        if (wp.skip_dir || (dirq_on && wp.m)) TRY(level_dir(l, wp.words, pdl));
        if (pair) {  // the last level: L1 from the pair pass's counts, then L2 + samples
          CU(cudaEventRecord(lev[l + 1], st));
          if (!scanned[l + 1]) TRY(scan_level(l + 1, ci));
          TRY(level_dir(l + 1, wp.next_words, false));
          break;
        }
      }
      // (the query-side layouts run after the last level: overlapping them
      // with the next level's kernel on a side stream measured slower)
    }
    for (uint32_t l = 0; l < P.L; ++l) TRY(alloc_level(t, l, st));  // (levels with no bits)
    TRY(launch_qlayouts(t, totals, st, &q_done));
    if (!tables_done) TRY(query_tables());
    if (tables_join) CU(cudaStreamWaitEvent(st, tables_join, 0));
    TRY(finish_tables(t));
    tr.mark("levels launched");
    if (P.L) CU(cudaEventRecord(lev[P.L], st));
    CU(cudaEventRecord(e1, st));
    std::vector<uint64_t> tot(std::max<uint32_t>(P.L, 1));
    CU(cudaMemcpyAsync(tot.data(), totals, tot.size() * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    tr.mark("build done");
    for (uint32_t l = 0; l < P.L; ++l) {
      wt_level_meta& m = t->lv[l].meta;
      m.total_ones = tot[l];
      m.n_ones = tot[l] / sample_rate;
      m.n_zeros = (m.n_bits - tot[l]) / sample_rate;
    }
    fill_treedev(t);
    if (ms_out) CU(cudaEventElapsedTime(ms_out, e0, e1));
    t->build_ms.assign(P.L + 1, 0.f);
    if (P.L) {
      CU(cudaEventElapsedTime(&t->build_ms[0], e0, lev[0]));
      for (uint32_t l = 0; l < P.L; ++l)
        CU(cudaEventElapsedTime(&t->build_ms[1 + l], lev[l], lev[l + 1]));
    }
    return WT_OK;
  };
  rc = body();
  if (rc == WT_OK) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(WT_ERR_CUDA, std::string("build: ") + cudaGetErrorString(e));
  }
  if (rc != WT_OK) {
    cudaStreamSynchronize(st);
    free_tree_arrays(t);
    delete t;
    return rc;
  }
  *out = t;
  return WT_OK;
}

extern "C" int wt_tree_from_arrays(const wt_meta* meta, const uint16_t* symbols,
                                   const int64_t* cum_hist, const uint64_t* words,
                                   const wt_level_meta* levels, const int64_t* l1_cat,
                                   const uint16_t* l2_cat, const int64_t* ones_cat,
                                   const int64_t* zeros_cat, int device, wt_tree** out) {
  if (!meta || !out) return fail(WT_ERR_ARG, "NULL argument");
  TRY(check_params(meta->l2_bits, meta->sample_rate));
  if (meta->sigma < 1 || meta->sigma > 65536) return fail(WT_ERR_ARG, "bad sigma");
  TRY(setup_device(device));
  wt_tree* t = new wt_tree();
  t->device = device;
  if (cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete t;
    return fail(WT_ERR_CUDA, "stream create failed");
  }
  cudaStream_t st = t->stream;
  auto body = [&]() -> int {
    Plan& P = t->plan;
    P.sigma = meta->sigma;
    P.L = ceil_log2_u(P.sigma);
    if (P.L != meta->levels) return fail(WT_ERR_ARG, "levels do not match sigma");
    P.symbols.assign(symbols, symbols + P.sigma);
    P.hist.resize(P.sigma);
    for (uint32_t i = 0; i < P.sigma; ++i) P.hist[i] = cum_hist[i + 1] - cum_hist[i];
    plan_codes(P);
    plan_shape(P, meta->l2_bits);
    t->meta = *meta;
    t->meta.levels = P.L;
    t->meta.first_coded = P.first_coded;
    t->meta.device = (uint32_t)device;
    if (t->meta.n_words != P.n_words) return fail(WT_ERR_ARG, "word count mismatch");
    TRY(alloc_tree(t, st));
    CU(cudaMemcpyAsync(t->words, words, P.n_words * 8, cudaMemcpyHostToDevice, st));
    uint64_t o1 = 0, o2 = 0, o3 = 0, o4 = 0;
    for (uint32_t l = 0; l < P.L; ++l) {
      LevelHost& h = t->lv[l];
      const wt_level_meta& m = levels[l];
      if (m.n_bits != h.meta.n_bits || m.n_l1 != h.meta.n_l1 || m.n_l2 != h.meta.n_l2)
        return fail(WT_ERR_ARG, "level directory shape mismatch");
      h.meta.total_ones = m.total_ones;
      h.meta.n_ones = m.n_ones;
      h.meta.n_zeros = m.n_zeros;
      if (m.n_l1) CU(cudaMemcpyAsync(h.l1, l1_cat + o1, m.n_l1 * 8, cudaMemcpyHostToDevice, st));
      if (m.n_l2) CU(cudaMemcpyAsync(h.l2, l2_cat + o2, m.n_l2 * 2, cudaMemcpyHostToDevice, st));
      if (m.n_ones)
        CU(cudaMemcpyAsync(h.ones, ones_cat + o3, m.n_ones * 8, cudaMemcpyHostToDevice, st));
      if (m.n_zeros)
        CU(cudaMemcpyAsync(h.zeros, zeros_cat + o4, m.n_zeros * 8, cudaMemcpyHostToDevice, st));
      o1 += m.n_l1;
      o2 += m.n_l2;
      o3 += m.n_ones;
      o4 += m.n_zeros;
    }
    CU(cudaStreamSynchronize(st));
    TRY(qlayouts_from_host_totals(t, st));
    fill_treedev(t);
    return WT_OK;
  };
  int rc = body();
  if (rc != WT_OK) {
    cudaStreamSynchronize(st);
    free_tree_arrays(t);
    delete t;
    return rc;
  }
  *out = t;
  return WT_OK;
}

extern "C" int wt_tree_meta(const wt_tree* t, wt_meta* out) {
  if (!t || !out) return fail(WT_ERR_ARG, "NULL argument");
  *out = t->meta;
  return WT_OK;
}

extern "C" int wt_tree_level_meta(const wt_tree* t, uint32_t level, wt_level_meta* out) {
  if (!t || !out || level >= t->plan.L) return fail(WT_ERR_ARG, "bad level");
  *out = t->lv[level].meta;
  return WT_OK;
}

static int copy_out(void* dst, const void* src, uint64_t bytes, uint64_t cap, bool device) {
  if (bytes > cap) return fail(WT_ERR_ARG, "destination too small");
  if (!bytes) return WT_OK;
  if (device)
    CU(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
  else
    memcpy(dst, src, bytes);
  return WT_OK;
}

extern "C" int wt_tree_get(const wt_tree* t, int what, uint32_t level, void* dst, uint64_t cap) {
  if (!t) return fail(WT_ERR_ARG, "NULL tree");
  const Plan& P = t->plan;
  CU(cudaSetDevice(t->device));
  const bool per_level = what >= WT_A_L1;
  if (per_level && level >= P.L) return fail(WT_ERR_ARG, "bad level");
  switch (what) {
    case WT_A_SYMBOLS: return copy_out(dst, P.symbols.data(), P.sigma * 2ull, cap, false);
    case WT_A_CODE_VALUES: return copy_out(dst, P.values.data(), P.sigma * 2ull, cap, false);
    case WT_A_CODE_LENS: return copy_out(dst, P.lens.data(), P.sigma, cap, false);
    case WT_A_CUM_HIST: return copy_out(dst, P.cum.data(), (P.sigma + 1ull) * 8, cap, false);
    case WT_A_LEVEL_SIZES: return copy_out(dst, P.sizes.data(), P.L * 8ull, cap, false);
    case WT_A_REGION_OFFS: return copy_out(dst, P.offsets.data(), P.L * 8ull, cap, false);
    case WT_A_WORDS: return copy_out(dst, t->words, P.n_words * 8, cap, true);
    case WT_A_L1: return copy_out(dst, t->lv[level].l1, t->lv[level].meta.n_l1 * 8, cap, true);
    case WT_A_L2: return copy_out(dst, t->lv[level].l2, t->lv[level].meta.n_l2 * 2, cap, true);
    case WT_A_ONES: return copy_out(dst, t->lv[level].ones, t->lv[level].meta.n_ones * 8, cap, true);
    case WT_A_ZEROS:
      return copy_out(dst, t->lv[level].zeros, t->lv[level].meta.n_zeros * 8, cap, true);
    case WT_A_QLINES:
      return copy_out(dst, t->lv[level].lines, t->lv[level].n_lines * kQLineBytes, cap, true);
    case WT_A_QSEL1:
    case WT_A_QSEL0: {
      // the filled prefix: one entry per 2^kQSelLog ones / zeros
      const wt_level_meta& m = t->lv[level].meta;
      const u64 k = what == WT_A_QSEL1 ? m.total_ones : m.n_bits - m.total_ones;
      const u64 cnt = std::min<u64>((k + (1u << kQSelLog) - 1) >> kQSelLog, t->lv[level].sel_cap);
      return copy_out(dst, what == WT_A_QSEL1 ? t->lv[level].sel1 : t->lv[level].sel0, cnt * 4, cap,
                      true);
    }
    case WT_A_NODE_STARTS:
    case WT_A_NODE_RANK0: {
      std::lock_guard<std::mutex> lk(const_cast<wt_tree*>(t)->tables_mutex);
      if (P.node_starts.size() != P.L) plan_walk(const_cast<Plan&>(P), true);
      const auto& v = what == WT_A_NODE_STARTS ? P.node_starts[level] : P.node_rank0[level];
      return copy_out(dst, v.data(), v.size() * 8, cap, false);
    }
    default: return fail(WT_ERR_ARG, "unknown array selector");
  }
}

extern "C" int wt_tree_build_profile(const wt_tree* t, float* ms, uint32_t cap) {
  if (!t || !ms) return fail(WT_ERR_ARG, "NULL argument");
  for (uint32_t i = 0; i < cap; ++i) ms[i] = i < t->build_ms.size() ? t->build_ms[i] : 0.f;
  return WT_OK;
}

extern "C" int wt_tree_destroy(wt_tree* t) {
  if (!t) return WT_OK;
  free_tree_arrays(t);
  delete t;
  return WT_OK;
}

// ---------------------------------------------------------------------------
// queries
// ---------------------------------------------------------------------------
// bits of the largest select ordinal (k <= max occurrences), cached per tree
static u32 select_kbits(wt_tree* t) {
  if (!t->sel_kbits) {
    u64 mx = 1;
    for (uint32_t i = 0; i < t->plan.sigma; ++i)
      mx = std::max<u64>(mx, (u64)(t->plan.cum[i + 1] - t->plan.cum[i]));
    t->sel_kbits = ceil_log2_u(mx + 1);
  }
  return t->sel_kbits;
}

// ---------------------------------------------------------------------------
// narrow wire format for host-buffer batches.  PCIe, not the device, bounds a
// batch that starts and ends in host memory (16 B per rank / select query in,
// 8 B out).  The host packs each chunk's i64 symbols / arguments into u16 /
// u32 pinned staging (6 B per query, 4 for access) on a persistent thread
// pool while the previous chunk is on the wire; a widen kernel restores the
// i64 chunk buffers on the device.  A chunk holding any value that does not
// fit (a negative or >= 2^16 symbol, a negative or >= 2^32 argument) crosses
// wide, unchanged -- validation (and the first bad index) stays on the device
// either way.  WT_WIRE=0 turns it off (A/B).
// ---------------------------------------------------------------------------
namespace {
class HostPool {
 public:
  // never destroyed: the workers sleep until process exit (no join at exit,
  // where a forked child would wait on threads it does not have)
  static HostPool& get() {
    static HostPool* p = new HostPool;
    return *p;
  }
  int threads() const { return (int)th_.size() + 1; }
  // f(worker, workers) on every pool thread and the caller; returns when all
  // did.  In a child forked after the pool started, the caller does it alone.
  void run(const std::function<void(int, int)>& f) {
    if (th_.empty() || getpid() != pid_) {
      f(0, 1);
      return;
    }
    std::lock_guard<std::mutex> serial(run_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      pending_ = (int)th_.size();
      ++gen_;
    }
    cv_.notify_all();
    f(0, threads());
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }
 private:
  HostPool() : pid_(getpid()) {
    int n = (int)std::thread::hardware_concurrency();
    if (const char* e = getenv("WT_HOST_THREADS")) n = atoi(e);
    n = std::max(1, std::min(n, 64));
    for (int i = 1; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  void loop(int id) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int, int)>* f;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        f = job_;
      }
      (*f)(id, threads());
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int, int)>* job_ = nullptr;
  uint64_t gen_ = 0;
  int pending_ = 0;
  const pid_t pid_;
};

// [a, b) of one pack slice with AVX2: 8 queries per step, staging written
// with non-temporal stores (no read-for-ownership of the staging lines: the
// host's memory bandwidth, shared with the DMA engines, is what bounds the
// pack).  a is a multiple of 64, the staging 256-byte aligned.
__attribute__((target("avx2"))) uint64_t pack_avx2(const int64_t* ids, const int64_t* args,
                                                  uint64_t a, uint64_t b, u16* w16, u32* w32) {
  const __m256i lo32 = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
  __m256i over = _mm256_setzero_si256();
  uint64_t i = a;
  for (; i + 8 <= b; i += 8) {
    const __m256i p0 = _mm256_loadu_si256((const __m256i*)(args + i));
    const __m256i p1 = _mm256_loadu_si256((const __m256i*)(args + i + 4));
    over = _mm256_or_si256(over, _mm256_or_si256(_mm256_srli_epi64(p0, 32), _mm256_srli_epi64(p1, 32)));
    const __m256i q0 = _mm256_permutevar8x32_epi32(p0, lo32), q1 = _mm256_permutevar8x32_epi32(p1, lo32);
    _mm256_stream_si256((__m256i*)(w32 + i), _mm256_permute2x128_si256(q0, q1, 0x20));
    if (ids) {
      const __m256i c0 = _mm256_loadu_si256((const __m256i*)(ids + i));
      const __m256i c1 = _mm256_loadu_si256((const __m256i*)(ids + i + 4));
      over = _mm256_or_si256(over, _mm256_or_si256(_mm256_srli_epi64(c0, 16), _mm256_srli_epi64(c1, 16)));
      const __m256i d = _mm256_permute2x128_si256(_mm256_permutevar8x32_epi32(c0, lo32),
                                                  _mm256_permutevar8x32_epi32(c1, lo32), 0x20);
      // u32 -> u16 (values above 2^16 are caught by `over`; the chunk then crosses wide)
      const __m256i pk = _mm256_permute4x64_epi64(_mm256_packus_epi32(d, d), 0x08);
      _mm_stream_si128((__m128i*)(w16 + i), _mm256_castsi256_si128(pk));
    }
  }
  uint64_t o = (uint64_t)_mm256_testz_si256(over, over) ? 0 : 1;
  for (; i < b; ++i) {
    const uint64_t p = (uint64_t)args[i];
    o |= p >> 32;
    w32[i] = (u32)p;
    if (ids) {
      const uint64_t c = (uint64_t)ids[i];
      o |= c >> 16;
      w16[i] = (u16)c;
    }
  }
  _mm_sfence();
  return o;
}

// pack cnt queries; false if any value does not fit the narrow format
bool pack_wire(const int64_t* ids, const int64_t* args, uint64_t cnt, u16* w16, u32* w32) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  std::atomic<uint64_t> over{0};
  // about 2^15 queries per worker at least: a small chunk (the API's default
  // is 65,536 queries) is packed by fewer threads, or by the caller alone
  const uint64_t want = std::max<uint64_t>(1, cnt >> 15);
  const auto job = [&](int w, int nw_pool) {
    const int nw = (int)std::min<uint64_t>((uint64_t)nw_pool, want);
    if (w >= nw) return;
    // 64-query-aligned slices: whole cache lines of every array per thread
    const uint64_t blocks = (cnt + 63) / 64;
    const uint64_t a = std::min(cnt, blocks * w / nw * 64);
    const uint64_t b = std::min(cnt, blocks * (w + 1) / nw * 64);
    uint64_t o = 0;
    if (avx2 && ((uintptr_t)w32 & 31) == 0 && ((uintptr_t)w16 & 15) == 0) {
      o = pack_avx2(ids, args, a, b, w16, w32);
    } else if (ids) {
      for (uint64_t i = a; i < b; ++i) {
        const uint64_t c = (uint64_t)ids[i], p = (uint64_t)args[i];
        o |= (c >> 16) | (p >> 32);
        w16[i] = (u16)c;
        w32[i] = (u32)p;
      }
    } else {
      for (uint64_t i = a; i < b; ++i) {
        const uint64_t p = (uint64_t)args[i];
        o |= p >> 32;
        w32[i] = (u32)p;
      }
    }
    if (o) over.fetch_or(o, std::memory_order_relaxed);
  };
  if (want == 1)
    job(0, 1);
  else
    HostPool::get().run(job);
  return over.load() == 0;
}

// smallest chunk that crosses narrow (WT_WIRE_MIN_CHUNK overrides; read per
// call so the tests can drive small chunks through the narrow path)
uint64_t wire_min_chunk() {
  const char* e = getenv("WT_WIRE_MIN_CHUNK");
  const unsigned long long v = e ? strtoull(e, nullptr, 10) : 0;
  return v ? (uint64_t)v : (1ull << 20);
}

bool wire_enabled() {
  static const bool on = [] {
    const char* e = getenv("WT_WIRE");
    return !(e && e[0] == '0');
  }();
  return on;
}
}  // namespace

extern "C" int wt_tree_query(wt_tree* t, int kind, const int64_t* ids, const int64_t* args,
                             void* out, uint64_t m, uint64_t chunk, int flags, void* stream,
                             int64_t* bad_index, float* ms_out) {
  return wt_tree_query_ex(t, kind, ids, args, out, m, chunk, flags, stream, bad_index, ms_out,
                          nullptr);
}

extern "C" int wt_tree_query_ex(wt_tree* t, int kind, const int64_t* ids, const int64_t* args,
                                void* out, uint64_t m, uint64_t chunk, int flags, void* stream,
                                int64_t* bad_index, float* ms_out, wt_query_stats* stats) {
  if (!t) return fail(WT_ERR_ARG, "NULL tree");
  if (kind < 0 || kind > 2) return fail(WT_ERR_ARG, "unknown query kind");
  if (ms_out) *ms_out = 0.f;
  if (stats) *stats = wt_query_stats{};
  if (bad_index) *bad_index = -1;
  if (m == 0) return WT_OK;
  if (!args || !out || (kind != WT_Q_ACCESS && !ids)) return fail(WT_ERR_ARG, "NULL buffer");
  CU(cudaSetDevice(t->device));
  const bool validate = (flags & WT_F_SYMBOLS) != 0;
  const int out_kind = kind != WT_Q_ACCESS ? 8
                       : (flags & WT_F_ACCESS_IDS) ? 8 : (int)t->dev.width;
  const size_t out_elem = (size_t)out_kind;
  std::lock_guard<std::mutex> lk(t->qmutex);
  if (flags & WT_F_DEVICE_PTRS) {
    cudaStream_t st = stream ? (cudaStream_t)stream : t->stream;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (validate) CU(cudaMemsetAsync(t->bad, 0xff, 8, st));
    if (ms_out) {
      CU(cudaEventCreate(&e0));
      CU(cudaEventCreate(&e1));
      CU(cudaEventRecord(e0, st));
    }
    if (flags & WT_F_SORT) {
      // sorted in slices of at most 2^31 queries (u32 slot indices);
      // WT_SORT_SLICE lowers the slice (tests exercise the multi-slice path)
      uint64_t slice_max = 1ull << 31;
      if (const char* e = getenv("WT_SORT_SLICE")) {
        const unsigned long long v = strtoull(e, nullptr, 10);
        if (v >= 1 && v < slice_max) slice_max = v;
      }
      const uint64_t slice = std::min<uint64_t>(m, slice_max);
      Scratch S{{}, st};
      QuerySortScratch Q{};
      Q.sel_kbits = select_kbits(t);
      TRY(S.get(&Q.hist, (1u << kQSortMaxBits) + 256));
      TRY(S.get(&Q.bucket_of, slice));
      TRY(S.get(&Q.sorted_args, slice));
      TRY(S.get(&Q.slot_of, slice));
      {
        u8* r;
        TRY(S.get(&r, slice * out_elem));
        Q.res = r;
      }
      // WT_F_PHASES: per-phase device times of a single-slice batch
      // (ms_out[1..3] = sort, walk, gather back to query order)
      const bool phases = (flags & WT_F_PHASES) && ms_out && slice == m;
      cudaEvent_t ph[3] = {nullptr, nullptr, nullptr};
      if (phases)
        for (auto& e : ph) CU(cudaEventCreate(&e));
      struct PhGuard { cudaEvent_t* p; ~PhGuard() { for (int i = 0; i < 3; ++i) if (p[i]) cudaEventDestroy(p[i]); } } pg{ph};
      for (uint64_t a = 0; a < m; a += slice) {
        const uint64_t cnt = std::min(slice, m - a);
        CU(launch_query_sorted(t->dev, kind, out_kind, validate,
                               ids ? (const i64*)ids + a : nullptr, (const i64*)args + a,
                               (u8*)out + a * out_elem, cnt, t->rate_log, a, t->bad, Q, st,
                               phases ? ph : nullptr));
      }
      if (phases) {
        CU(cudaEventRecord(e1, st));
        CU(cudaStreamSynchronize(st));
        CU(cudaEventElapsedTime(ms_out + 1, e0, ph[0]));
        CU(cudaEventElapsedTime(ms_out + 2, ph[0], ph[1]));
        CU(cudaEventElapsedTime(ms_out + 3, ph[1], ph[2]));
      }
    } else {
      CU(launch_query(t->dev, kind, out_kind, validate, (const i64*)ids, (const i64*)args, out, m,
                      t->rate_log, 0, t->bad, st));
    }
    if (ms_out) CU(cudaEventRecord(e1, st));
    if (validate && bad_index)
      CU(cudaMemcpyAsync(bad_index, t->bad, 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (ms_out) {
      CU(cudaEventElapsedTime(ms_out, e0, e1));
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      if (stats) stats->kernel_ms = stats->total_ms = *ms_out;
    }
    if (stats) {
      stats->chunks = 1;
      stats->chunk_records = m;
    }
    return WT_OK;
  }
  // host buffers: a 3-stage pipeline over two device chunk slots -- the
  // copy-in of chunk c+1, the kernel of chunk c and the copy-out of chunk c-1
  // run on three streams at once (batch.py:152-239 keeps at
  // most two chunks staged).  Copies are only asynchronous from pinned host
  // memory (the Python layer hands pinned result arrays for large batches).
  if (chunk == 0) chunk = 1ull << 22;
  if (chunk > m) chunk = m;
  const bool sorted = (flags & WT_F_SORT) != 0;
  // per slot: ids, args, out [+ sort scratch: buckets, slot_of, sorted args,
  // bucket_of, sorted-order results; each 16-byte aligned]
  const size_t sort_bytes =
      sorted ? ((1u << kQSortMaxBits) + 256) * 4 + chunk * (4 + 8 + 4 + out_elem) + 5 * 16 : 0;
  // narrow wire: texts below 2^32 (positions and ordinals fit u32); the
  // device slot grows by the chunk's u32 + u16 landing area
  // (rank / select only: an access query saves 4 B of PCIe, and packing it
  // costs more host memory bandwidth than that -- measured 5.9 -> 6.3 ms per
  // 3.3e7 access queries, against 11.7 -> 10.5 ms for rank)
  // Chunks below 2^20 queries stay wide: the wide pipeline enqueues every
  // chunk without a host wait, while a packed chunk holds the host loop for
  // its pack -- at 2^16-query chunks (the API default) that measured 1.5x
  // slower for rank, at 2^18 even, at 2^22 15 % faster.
  const bool wire = wire_enabled() && kind != WT_Q_ACCESS && t->meta.n <= 0xffffffffull &&
                    chunk >= wire_min_chunk();
  const size_t wire_bytes = wire ? chunk * 6 + 64 : 0;
  const size_t need = chunk * (16 + out_elem) + 64 + sort_bytes + wire_bytes;
  for (int i = 0; i < 3; ++i) {
    if (!t->qstream[i]) CU(cudaStreamCreateWithFlags(&t->qstream[i], cudaStreamNonBlocking));
    for (int j = 0; j < 2; ++j)
      if (!t->qev[i][j]) CU(cudaEventCreateWithFlags(&t->qev[i][j], cudaEventDisableTiming));
  }
  for (int i = 0; i < 2; ++i) {
    if (t->qbuf_bytes < need && t->qbuf[i]) {
      CU(cudaFree(t->qbuf[i]));
      t->qbuf[i] = nullptr;
    }
    if (!t->qbuf[i]) CU(cudaMalloc(&t->qbuf[i], need));
  }
  t->qbuf_bytes = std::max(t->qbuf_bytes, need);
  if (wire) {
    const size_t hb = chunk * 6 + 64;
    for (int i = 0; i < 2; ++i) {
      if (t->hst_bytes < hb && t->hst[i]) {
        // the slot's last copy-in must have drained before the buffer goes
        if (t->hev[i]) CU(cudaEventSynchronize(t->hev[i]));
        CU(cudaFreeHost(t->hst[i]));
        t->hst[i] = nullptr;
      }
      if (!t->hst[i]) CU(cudaHostAlloc(&t->hst[i], hb, cudaHostAllocPortable));
      if (!t->hev[i]) CU(cudaEventCreateWithFlags(&t->hev[i], cudaEventDisableTiming));
    }
    t->hst_bytes = std::max(t->hst_bytes, hb);
  }
  cudaStream_t sin = t->qstream[0], sk = t->qstream[1], sout = t->qstream[2];
  if (validate) {
    CU(cudaMemsetAsync(t->bad, 0xff, 8, sk));
  }
  const uint64_t nchunks = (m + chunk - 1) / chunk;
  // timing events (ms_out / stats), pooled in the tree: per chunk
  // [copy-in start, copy-in end, kernel end] + one after the last copy-out
  const bool timed = ms_out || stats;
  if (timed && t->tev.size() < 3 * nchunks + 1) {
    const size_t have = t->tev.size();
    t->tev.resize(3 * nchunks + 1, nullptr);
    for (size_t i = have; i < t->tev.size(); ++i) CU(cudaEventCreate(&t->tev[i]));
  }
  cudaEvent_t* ev = timed ? t->tev.data() : nullptr;
  int rc = WT_OK;
  uint64_t h2d_bytes = 0, narrow_chunks = 0;
  for (uint64_t c = 0; c < nchunks && rc == WT_OK; ++c) {
    const int s = (int)(c & 1);
    const uint64_t a = c * chunk, cnt = std::min(chunk, m - a);
    u8* base = (u8*)t->qbuf[s];
    i64* d_ids = (i64*)base;
    i64* d_args = (i64*)(base + chunk * 8);
    u8* d_out = base + chunk * 16;
    cudaError_t e = cudaSuccess;
    // narrow wire: pack chunk c into the slot's pinned staging once the
    // copy-in of chunk c-2 has read it (overlaps chunk c-1 on the wire)
    bool narrow = false;
    u32* d_w32 = nullptr;
    u16* d_w16 = nullptr;
    if (wire) {
      const uint64_t w16_off = (chunk * 4 + 15) & ~(uint64_t)15;
      u8* wp = (u8*)(((uintptr_t)(base + need - wire_bytes) + 15) & ~(uintptr_t)15);
      d_w32 = (u32*)wp;
      d_w16 = (u16*)(wp + w16_off);
      u32* h32 = (u32*)t->hst[s];
      u16* h16 = (u16*)((u8*)t->hst[s] + w16_off);
      if (c >= 2) e = cudaEventSynchronize(t->hev[s]);
      if (e == cudaSuccess)
        narrow = pack_wire(kind != WT_Q_ACCESS ? ids + a : nullptr, args + a, cnt, h16, h32);
      if (narrow) {
        if (c >= 2) e = cudaStreamWaitEvent(sin, t->qev[1][s], 0);
        if (e == cudaSuccess && ev) e = cudaEventRecord(ev[3 * c], sin);
        if (e == cudaSuccess && kind != WT_Q_ACCESS)
          e = cudaMemcpyAsync(d_w16, h16, cnt * 2, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_w32, h32, cnt * 4, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess) e = cudaEventRecord(t->hev[s], sin);
      }
    }
    // copy-in: slot s is free once the kernel of chunk c-2 has read it
    if (!narrow) {
      if (e == cudaSuccess && c >= 2) e = cudaStreamWaitEvent(sin, t->qev[1][s], 0);
      if (e == cudaSuccess && ev) e = cudaEventRecord(ev[3 * c], sin);
      if (e == cudaSuccess && kind != WT_Q_ACCESS)
        e = cudaMemcpyAsync(d_ids, ids + a, cnt * 8, cudaMemcpyHostToDevice, sin);
      if (e == cudaSuccess) e = cudaMemcpyAsync(d_args, args + a, cnt * 8, cudaMemcpyHostToDevice, sin);
    }
    const uint64_t in_elem = narrow ? (kind != WT_Q_ACCESS ? 6 : 4) : (kind != WT_Q_ACCESS ? 16 : 8);
    h2d_bytes += cnt * in_elem;
    narrow_chunks += narrow;
    if (e == cudaSuccess && ev) e = cudaEventRecord(ev[3 * c + 1], sin);
    if (e == cudaSuccess) e = cudaEventRecord(t->qev[0][s], sin);
    // kernel: inputs landed, and the copy-out of chunk c-2 has drained d_out
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sk, t->qev[0][s], 0);
    if (e == cudaSuccess && c >= 2) e = cudaStreamWaitEvent(sk, t->qev[2][s], 0);
    if (e == cudaSuccess && narrow)
      e = launch_widen(kind != WT_Q_ACCESS ? d_w16 : nullptr, d_w32, d_ids, d_args, cnt, sk);
    if (e == cudaSuccess && !sorted) {
      e = launch_query(t->dev, kind, out_kind, validate, d_ids, d_args, d_out, cnt, t->rate_log, a,
                       t->bad, sk);
    } else if (e == cudaSuccess) {
      u8* sp = (u8*)(((uintptr_t)(d_out + chunk * out_elem) + 15) & ~(uintptr_t)15);
      QuerySortScratch Q{};
      Q.sel_kbits = select_kbits(t);
      auto take = [&](size_t bytes) {
        u8* p = sp;
        sp = (u8*)(((uintptr_t)(sp + bytes) + 15) & ~(uintptr_t)15);
        return p;
      };
      Q.hist = (u32*)take(((1u << kQSortMaxBits) + 256) * 4);
      Q.slot_of = (u32*)take(chunk * 4);
      Q.sorted_args = (i64*)take(chunk * 8);
      Q.bucket_of = (u32*)take(chunk * 4);
      Q.res = take(chunk * out_elem);
      e = launch_query_sorted(t->dev, kind, out_kind, validate, d_ids, d_args, d_out, cnt,
                              t->rate_log, a, t->bad, Q, sk);
    }
    if (e == cudaSuccess && ev) e = cudaEventRecord(ev[3 * c + 2], sk);
    if (e == cudaSuccess) e = cudaEventRecord(t->qev[1][s], sk);
    // copy-out
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, t->qev[1][s], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync((u8*)out + a * out_elem, d_out, cnt * out_elem, cudaMemcpyDeviceToHost, sout);
    if (e == cudaSuccess) e = cudaEventRecord(t->qev[2][s], sout);
    if (e != cudaSuccess) rc = fail(WT_ERR_CUDA, std::string("query pipeline: ") + cudaGetErrorString(e));
  }
  if (rc == WT_OK && ev) {
    cudaError_t e = cudaEventRecord(ev[3 * nchunks], sout);
    if (e != cudaSuccess) rc = fail(WT_ERR_CUDA, cudaGetErrorString(e));
  }
  for (int i = 0; i < 3; ++i) {
    cudaError_t e = cudaStreamSynchronize(t->qstream[i]);
    if (e != cudaSuccess && rc == WT_OK) rc = fail(WT_ERR_CUDA, cudaGetErrorString(e));
  }
  if (timed && rc == WT_OK) {
    // device-time accounting of the pipeline, and the staging it actually
    // had: chunk c's queries occupy a device slot from the start of their
    // copy-in until the kernel has consumed them; the peak is the largest
    // record count staged at once (the reference's staging_peak_records,
    // batch.py:100-108).  Kernel time of chunk c = from the later of its
    // inputs landing and the previous kernel's end, to its end.
    float h2d = 0.f, kern = 0.f, prev_k = 0.f;
    std::vector<std::pair<float, int64_t>> edges;
    edges.reserve(2 * nchunks);
    for (uint64_t c = 0; c < nchunks; ++c) {
      float a = 0, b = 0, k1 = 0;
      cudaEventElapsedTime(&a, ev[0], ev[3 * c]);
      cudaEventElapsedTime(&b, ev[0], ev[3 * c + 1]);
      cudaEventElapsedTime(&k1, ev[0], ev[3 * c + 2]);
      h2d += b - a;
      kern += k1 - std::max(b, prev_k);
      prev_k = k1;
      const int64_t cnt = (int64_t)std::min(chunk, m - c * chunk);
      edges.push_back({a, cnt});
      edges.push_back({k1, -cnt});
    }
    float last_out = 0;
    cudaEventElapsedTime(&last_out, ev[0], ev[3 * nchunks]);
    // at equal times a release sorts before an acquire (slot handed over)
    std::sort(edges.begin(), edges.end());
    int64_t cur = 0, peak = 0;
    for (auto& e : edges) peak = std::max(peak, cur += e.second);
    if (ms_out) *ms_out = kern;
    if (stats) {
      stats->chunks = nchunks;
      stats->slots = nchunks > 1 ? 2 : 1;
      stats->chunk_records = chunk;
      stats->peak_records = (uint64_t)peak;
      stats->h2d_ms = h2d;
      stats->kernel_ms = kern;
      stats->d2h_ms = last_out - prev_k;  // the copy-out tail after the last kernel
      stats->total_ms = last_out;
      stats->h2d_bytes = h2d_bytes;
      stats->narrow_chunks = narrow_chunks;
    }
  }
  if (rc == WT_OK && validate && bad_index) {
    cudaError_t e = cudaMemcpy(bad_index, t->bad, 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = fail(WT_ERR_CUDA, cudaGetErrorString(e));
  }
  return rc;
}

// pinned host memory for result arrays (so the copy-out is asynchronous)
extern "C" int wt_host_alloc(uint64_t bytes, void** out) {
  if (!out) return fail(WT_ERR_ARG, "NULL out");
  *out = nullptr;
  if (!bytes) return WT_OK;
  if (cudaHostAlloc(out, bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    return fail(WT_ERR_OOM, "cudaHostAlloc failed");
  }
  return WT_OK;
}
extern "C" int wt_host_free(void* p) {
  if (p) cudaFreeHost(p);
  return WT_OK;
}
// page-lock an existing host range (a shared-memory result array the ranks
// of a node write disjoint slices of), so device->host copies into it are
// asynchronous DMA
extern "C" int wt_host_register(void* p, uint64_t bytes) {
  if (!p || !bytes) return WT_OK;
  CU(cudaHostRegister(p, bytes, cudaHostRegisterPortable));
  return WT_OK;
}
extern "C" int wt_host_unregister(void* p) {
  if (p) CU(cudaHostUnregister(p));
  return WT_OK;
}

// per-level bit-vector queries on a built tree (RankSelectIndex methods of
// tree.rs[l], rankselect.py:140-373); args / out are host int64 arrays
extern "C" int wt_tree_level_query(wt_tree* t, uint32_t level, int kind, const int64_t* args,
                                   int64_t* out, uint64_t m) {
  if (!t || level >= t->plan.L) return fail(WT_ERR_ARG, "bad level");
  if (kind < 0 || kind > 4) return fail(WT_ERR_ARG, "unknown bit query kind");
  if (m == 0) return WT_OK;
  CU(cudaSetDevice(t->device));
  cudaStream_t st = t->stream ? t->stream : 0;
  Scratch S{{}, st};
  i64 *da, *dout;
  TRY(S.get(&da, m));
  TRY(S.get(&dout, m));
  CU(cudaMemcpyAsync(da, args, m * 8, cudaMemcpyHostToDevice, st));
  CU(launch_bits_query(t->dev.lv[level], t->dev.l2_shift, t->dev.rate, t->rate_log, kind, da, dout,
                       m, st));
  CU(cudaMemcpyAsync(out, dout, m * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return WT_OK;
}

// ---------------------------------------------------------------------------
// NCCL replication (dlopen'ed so single-GPU use has no NCCL dependency)
// ---------------------------------------------------------------------------
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int (*nccl_get_uid_t)(ncclUniqueId*);
typedef int (*nccl_init_rank_t)(ncclComm_t*, int, ncclUniqueId, int);
typedef int (*nccl_bcast_t)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*nccl_destroy_t)(ncclComm_t);
typedef const char* (*nccl_errstr_t)(int);
typedef int (*nccl_group_t)(void);
typedef int (*nccl_allreduce_t)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);

struct NcclApi {
  bool ok = false;
  nccl_get_uid_t get_uid;
  nccl_init_rank_t init_rank;
  nccl_bcast_t bcast;
  nccl_destroy_t destroy;
  nccl_errstr_t errstr;
  nccl_group_t group_start, group_end;
  nccl_allreduce_t allreduce;
};
static NcclApi g_nccl;
static std::once_flag g_nccl_once;
static int nccl_load() {
  std::call_once(g_nccl_once, []() {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    g_nccl.get_uid = (nccl_get_uid_t)dlsym(h, "ncclGetUniqueId");
    g_nccl.init_rank = (nccl_init_rank_t)dlsym(h, "ncclCommInitRank");
    g_nccl.bcast = (nccl_bcast_t)dlsym(h, "ncclBroadcast");
    g_nccl.destroy = (nccl_destroy_t)dlsym(h, "ncclCommDestroy");
    g_nccl.errstr = (nccl_errstr_t)dlsym(h, "ncclGetErrorString");
    g_nccl.group_start = (nccl_group_t)dlsym(h, "ncclGroupStart");
    g_nccl.group_end = (nccl_group_t)dlsym(h, "ncclGroupEnd");
    g_nccl.allreduce = (nccl_allreduce_t)dlsym(h, "ncclAllReduce");
    g_nccl.ok = g_nccl.get_uid && g_nccl.init_rank && g_nccl.bcast && g_nccl.destroy &&
                g_nccl.group_start && g_nccl.group_end && g_nccl.allreduce;
  });
  if (!g_nccl.ok) return fail(WT_ERR_NCCL, "libnccl.so.2 not loadable");
  return WT_OK;
}
#define NC(call)                                                                        \
  do {                                                                                  \
    int r_ = (call);                                                                    \
    if (r_ != 0)                                                                        \
      return fail(WT_ERR_NCCL, std::string(#call) + ": " +                              \
                                   (g_nccl.errstr ? g_nccl.errstr(r_) : "nccl error")); \
  } while (0)

extern "C" int wt_nccl_unique_id(uint8_t id[128]) {
  TRY(nccl_load());
  ncclUniqueId u;
  NC(g_nccl.get_uid(&u));
  memcpy(id, u.internal, 128);
  return WT_OK;
}

// Root: its tree; others: NULL.  Small O(sigma) + metadata travel in one
// broadcast of a host-packed header; the words and directories are broadcast
// in place (ncclBroadcast over NVLink / NVSwitch), then every rank holds a
// complete device-resident replica.
extern "C" int wt_tree_replicate(wt_tree* root_tree, const uint8_t id[128], int rank, int world,
                                 int device, wt_tree** out, float* ms_out) {
  if (!out) return fail(WT_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (rank == 0 && !root_tree) return fail(WT_ERR_ARG, "root needs its tree");
  TRY(nccl_load());
  TRY(setup_device(device));
  cudaStream_t st;
  CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  ncclUniqueId u;
  memcpy(u.internal, id, 128);
  ncclComm_t comm;
  NC(g_nccl.init_rank(&comm, world, u, rank));
  struct CommGuard { ncclComm_t c; cudaStream_t s; ~CommGuard() { g_nccl.destroy(c); cudaStreamDestroy(s); } } cg{comm, st};
  // 1. header: meta + per-level meta + symbols + cum (device staging buffer)
  const size_t hdr_fixed = sizeof(wt_meta) + 16 * sizeof(wt_level_meta);
  std::vector<u8> hdr;
  uint64_t hdr_bytes = 0;
  if (rank == 0) {
    const wt_tree* t = root_tree;
    hdr.resize(hdr_fixed + t->plan.sigma * 2 + (t->plan.sigma + 1) * 8);
    memcpy(hdr.data(), &t->meta, sizeof(wt_meta));
    for (uint32_t l = 0; l < t->plan.L; ++l)
      memcpy(hdr.data() + sizeof(wt_meta) + l * sizeof(wt_level_meta), &t->lv[l].meta,
             sizeof(wt_level_meta));
    memcpy(hdr.data() + hdr_fixed, t->plan.symbols.data(), t->plan.sigma * 2);
    memcpy(hdr.data() + hdr_fixed + t->plan.sigma * 2, t->plan.cum.data(), (t->plan.sigma + 1) * 8);
    hdr_bytes = hdr.size();
  }
  u64* dsz;
  CU(cudaMalloc(&dsz, 8));
  CU(cudaMemcpy(dsz, &hdr_bytes, 8, cudaMemcpyHostToDevice));
  NC(g_nccl.bcast(dsz, dsz, 8, /*ncclUint8*/ 1, 0, comm, st));
  CU(cudaMemcpyAsync(&hdr_bytes, dsz, 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  cudaFree(dsz);
  hdr.resize(hdr_bytes);
  u8* dh;
  CU(cudaMalloc(&dh, hdr_bytes));
  if (rank == 0) CU(cudaMemcpy(dh, hdr.data(), hdr_bytes, cudaMemcpyHostToDevice));
  NC(g_nccl.bcast(dh, dh, hdr_bytes, 1, 0, comm, st));
  CU(cudaMemcpyAsync(hdr.data(), dh, hdr_bytes, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  cudaFree(dh);
  // 2. receivers allocate an identically shaped tree
  wt_tree* t = nullptr;
  int alloc_rc = WT_OK;
  if (rank == 0) {
    t = root_tree;
  } else if (!(t = new wt_tree()) ||
             cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete t;
    t = nullptr;
    alloc_rc = fail(WT_ERR_CUDA, "stream create failed");  // reported after the status reduce
  } else {
    t->device = device;
    memcpy(&t->meta, hdr.data(), sizeof(wt_meta));
    t->meta.device = (uint32_t)device;
    Plan& P = t->plan;
    P.sigma = t->meta.sigma;
    P.L = t->meta.levels;
    P.symbols.resize(P.sigma);
    memcpy(P.symbols.data(), hdr.data() + hdr_fixed, P.sigma * 2);
    std::vector<int64_t> cum(P.sigma + 1);
    memcpy(cum.data(), hdr.data() + hdr_fixed + P.sigma * 2, (P.sigma + 1) * 8);
    P.hist.resize(P.sigma);
    for (uint32_t i = 0; i < P.sigma; ++i) P.hist[i] = cum[i + 1] - cum[i];
    plan_codes(P);
    plan_shape(P, t->meta.l2_bits);
    alloc_rc = alloc_tree(t, st);
    if (alloc_rc == WT_OK)
      for (uint32_t l = 0; l < P.L; ++l)
        memcpy(&t->lv[l].meta, hdr.data() + sizeof(wt_meta) + l * sizeof(wt_level_meta),
               sizeof(wt_level_meta));
  }
  // every rank learns whether every receiver has its tree before any rank
  // enters the grouped broadcast (a rank that returned early would leave the
  // others blocked in the collective): max-reduce of the allocation status
  auto drop = [&]() {
    if (rank != 0 && t) {
      free_tree_arrays(t);
      delete t;
      t = nullptr;
    }
  };
  {
    int* dst_flag = nullptr;
    int any = alloc_rc != WT_OK ? 1 : 0;
    cudaError_t ce = cudaMalloc(&dst_flag, 4);
    if (ce == cudaSuccess) ce = cudaMemcpy(dst_flag, &any, 4, cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {  // still take part: the others are waiting on this rank
      any = 1;
      if (!dst_flag) cudaMalloc(&dst_flag, 4);
    }
    const int nr = dst_flag ? g_nccl.allreduce(dst_flag, dst_flag, 1, /*ncclInt32*/ 2, /*ncclMax*/ 2, comm, st) : 1;
    int all = 1;
    if (nr == 0 && cudaMemcpyAsync(&all, dst_flag, 4, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
        cudaStreamSynchronize(st) == cudaSuccess) {
      all = any ? 1 : all;
    } else {
      all = 1;
    }
    if (dst_flag) cudaFree(dst_flag);
    if (all) {
      drop();
      return alloc_rc != WT_OK ? alloc_rc : fail(WT_ERR_CUDA, "replicate: a receiver could not allocate its tree");
    }
  }
  // 3. bulk arrays, one grouped broadcast (a receiver's tree is freed on
  // any failure from here on)
  const int rc3 = [&]() -> int {
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    struct EvG { cudaEvent_t a, b; ~EvG() { cudaEventDestroy(a); cudaEventDestroy(b); } } eg{e0, e1};
    CU(cudaEventRecord(e0, st));
    NC(g_nccl.group_start());
    NC(g_nccl.bcast(t->words, t->words, t->plan.n_words * 8, 1, 0, comm, st));
    for (uint32_t l = 0; l < t->plan.L; ++l) {
      LevelHost& h = t->lv[l];
      if (h.meta.n_l1) NC(g_nccl.bcast(h.l1, h.l1, h.meta.n_l1 * 8, 1, 0, comm, st));
      if (h.meta.n_l2) NC(g_nccl.bcast(h.l2, h.l2, h.meta.n_l2 * 2, 1, 0, comm, st));
      if (h.meta.n_ones) NC(g_nccl.bcast(h.ones, h.ones, h.meta.n_ones * 8, 1, 0, comm, st));
      if (h.meta.n_zeros) NC(g_nccl.bcast(h.zeros, h.zeros, h.meta.n_zeros * 8, 1, 0, comm, st));
    }
    NC(g_nccl.group_end());
    CU(cudaEventRecord(e1, st));
    CU(cudaStreamSynchronize(st));
    if (ms_out) cudaEventElapsedTime(ms_out, e0, e1);
    if (rank != 0) {
      TRY(qlayouts_from_host_totals(t, st));
      fill_treedev(t);
    }
    return WT_OK;
  }();
  if (rc3 != WT_OK) {
    drop();
    return rc3;
  }
  *out = rank == 0 ? nullptr : t;
  return WT_OK;
}

// ---------------------------------------------------------------------------
// stand-alone bit vectors (rankselect.build_index over one region)
// ---------------------------------------------------------------------------
struct wt_bits {
  int device = 0;
  u64* words = nullptr;
  LevelHost h;
  uint32_t l2_bits = 512, l2_shift = 9;
  uint64_t rate = 1;
  int rate_log = 0;
  cudaStream_t stream = nullptr;
};

static LevelDev bits_dev(const wt_bits* b) {
  LevelDev d{};
  d.words = b->words;
  d.l1 = b->h.l1;
  d.l2 = b->h.l2;
  d.ones = b->h.ones;
  d.zeros = b->h.zeros;
  d.n_bits = b->h.meta.n_bits;
  d.total_ones = b->h.meta.total_ones;
  d.n_ones = b->h.meta.n_ones;
  d.n_zeros = b->h.meta.n_zeros;
  d.n_l1 = b->h.meta.n_l1;
  d.n_l2 = b->h.meta.n_l2;
  return d;
}

static void free_bits(wt_bits* b) {
  cudaSetDevice(b->device);
  for (void* p : {(void*)b->words, (void*)b->h.l1, (void*)b->h.l2, (void*)b->h.ones,
                  (void*)b->h.zeros})
    if (p) cudaFree(p);
  if (b->stream) cudaStreamDestroy(b->stream);
}

extern "C" int wt_bits_build(const uint64_t* words, uint64_t n_bits, int words_on_device,
                             uint32_t l2_bits, uint64_t sample_rate, int device, wt_bits** out) {
  if (!out) return fail(WT_ERR_ARG, "out is NULL");
  *out = nullptr;
  TRY(check_params(l2_bits, sample_rate));
  TRY(setup_device(device));
  wt_bits* b = new wt_bits();
  b->device = device;
  b->l2_bits = l2_bits;
  while ((1u << b->l2_shift) < l2_bits) ++b->l2_shift;
  while ((1u << b->l2_shift) > l2_bits) --b->l2_shift;
  b->rate = sample_rate;
  b->rate_log = rate_log_of(sample_rate);
  auto body = [&]() -> int {
    CU(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
    cudaStream_t st = b->stream;
    const uint64_t nw = (n_bits + 63) / 64;
    wt_level_meta& m = b->h.meta;
    m.n_bits = n_bits;
    m.n_l1 = (n_bits + kL1Bits - 1) / kL1Bits;
    m.n_l2 = (n_bits + l2_bits - 1) / l2_bits;
    TRY(dalloc(&b->words, nw + 1, st));
    if (nw) CU(cudaMemcpyAsync(b->words, words, nw * 8,
                               words_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    TRY(dalloc(&b->h.l1, m.n_l1, st));
    TRY(dalloc(&b->h.l2, m.n_l2, st));
    TRY(dalloc(&b->h.ones, n_bits / sample_rate, st));
    TRY(dalloc(&b->h.zeros, n_bits / sample_rate, st));
    Scratch S{{}, st};
    const uint32_t tiles = bits_tiles(n_bits);
    u64* status;
    u32* agg;
    u64* total;
    TRY(S.get(&status, tiles));
    TRY(S.get(&agg, 1));
    TRY(S.get(&total, 1));
    CU(cudaMemsetAsync(status, 0, std::max<uint32_t>(tiles, 1) * 8, st));
    CU(cudaMemsetAsync(agg, 0, 4, st));
    CU(cudaMemsetAsync(total, 0, 8, st));
    BitsParams p{};
    p.words = b->words;
    p.n_bits = n_bits;
    p.l1 = b->h.l1;
    p.l2 = b->h.l2;
    p.ones = b->h.ones;
    p.zeros = b->h.zeros;
    p.ones_cap = n_bits / sample_rate;
    p.zeros_cap = n_bits / sample_rate;
    p.status = status;
    p.agg = agg;
    p.counter = agg;
    p.total_out = total;
    p.l2_log = b->l2_shift;
    p.rate_log = b->rate_log;
    p.rate = sample_rate;
    CU(launch_bits_directory(p, st));
    uint64_t tot = 0;
    CU(cudaMemcpyAsync(&tot, total, 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    m.total_ones = tot;
    m.n_ones = tot / sample_rate;
    m.n_zeros = (n_bits - tot) / sample_rate;
    return WT_OK;
  };
  int rc = body();
  if (rc != WT_OK) {
    if (b->stream) cudaStreamSynchronize(b->stream);
    free_bits(b);
    delete b;
    return rc;
  }
  *out = b;
  return WT_OK;
}

// RankSelectIndex.read (rankselect.py:397-411): a directory deserialized (and
// validated) on the host is uploaded as is -- the queries then answer from
// the stored L1 / L2 / samples, as the reference's do.
extern "C" int wt_bits_from_arrays(const uint64_t* words, uint64_t n_bits, uint32_t l2_bits,
                                   uint64_t sample_rate, uint64_t total_ones, const int64_t* l1,
                                   uint64_t n_l1, const uint16_t* l2, uint64_t n_l2,
                                   const int64_t* ones, uint64_t n_ones, const int64_t* zeros,
                                   uint64_t n_zeros, int device, wt_bits** out) {
  if (!out) return fail(WT_ERR_ARG, "out is NULL");
  *out = nullptr;
  TRY(check_params(l2_bits, sample_rate));
  if (n_l1 != (n_bits + kL1Bits - 1) / kL1Bits || n_l2 != (n_bits + l2_bits - 1) / l2_bits)
    return fail(WT_ERR_ARG, "directory lengths do not match n_bits");
  if (total_ones > n_bits) return fail(WT_ERR_ARG, "total_ones > n_bits");
  TRY(setup_device(device));
  wt_bits* b = new wt_bits();
  b->device = device;
  b->l2_bits = l2_bits;
  while ((1u << b->l2_shift) < l2_bits) ++b->l2_shift;
  while ((1u << b->l2_shift) > l2_bits) --b->l2_shift;
  b->rate = sample_rate;
  b->rate_log = rate_log_of(sample_rate);
  auto body = [&]() -> int {
    CU(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
    cudaStream_t st = b->stream;
    const uint64_t nw = (n_bits + 63) / 64;
    wt_level_meta& m = b->h.meta;
    m.n_bits = n_bits;
    m.n_l1 = n_l1;
    m.n_l2 = n_l2;
    m.total_ones = total_ones;
    m.n_ones = n_ones;
    m.n_zeros = n_zeros;
    TRY(dalloc(&b->words, nw + 1, st));
    TRY(dalloc(&b->h.l1, n_l1, st));
    TRY(dalloc(&b->h.l2, n_l2, st));
    TRY(dalloc(&b->h.ones, n_ones, st));
    TRY(dalloc(&b->h.zeros, n_zeros, st));
    if (nw) CU(cudaMemcpyAsync(b->words, words, nw * 8, cudaMemcpyHostToDevice, st));
    if (n_l1) CU(cudaMemcpyAsync(b->h.l1, l1, n_l1 * 8, cudaMemcpyHostToDevice, st));
    if (n_l2) CU(cudaMemcpyAsync(b->h.l2, l2, n_l2 * 2, cudaMemcpyHostToDevice, st));
    if (n_ones) CU(cudaMemcpyAsync(b->h.ones, ones, n_ones * 8, cudaMemcpyHostToDevice, st));
    if (n_zeros) CU(cudaMemcpyAsync(b->h.zeros, zeros, n_zeros * 8, cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));
    return WT_OK;
  };
  int rc = body();
  if (rc != WT_OK) {
    if (b->stream) cudaStreamSynchronize(b->stream);
    free_bits(b);
    delete b;
    return rc;
  }
  *out = b;
  return WT_OK;
}

extern "C" int wt_bits_level_meta(const wt_bits* b, wt_level_meta* out) {
  if (!b || !out) return fail(WT_ERR_ARG, "NULL argument");
  *out = b->h.meta;
  return WT_OK;
}

extern "C" int wt_bits_get(const wt_bits* b, int what, void* dst, uint64_t cap) {
  if (!b) return fail(WT_ERR_ARG, "NULL bits");
  CU(cudaSetDevice(b->device));
  const wt_level_meta& m = b->h.meta;
  switch (what) {
    case WT_A_WORDS: return copy_out(dst, b->words, (m.n_bits + 63) / 64 * 8, cap, true);
    case WT_A_L1: return copy_out(dst, b->h.l1, m.n_l1 * 8, cap, true);
    case WT_A_L2: return copy_out(dst, b->h.l2, m.n_l2 * 2, cap, true);
    case WT_A_ONES: return copy_out(dst, b->h.ones, m.n_ones * 8, cap, true);
    case WT_A_ZEROS: return copy_out(dst, b->h.zeros, m.n_zeros * 8, cap, true);
    default: return fail(WT_ERR_ARG, "unknown array selector");
  }
}

extern "C" int wt_bits_query(wt_bits* b, int kind, const int64_t* args, int64_t* out, uint64_t m,
                             int flags) {
  if (!b) return fail(WT_ERR_ARG, "NULL bits");
  if (kind < 0 || kind > 4) return fail(WT_ERR_ARG, "unknown bit query kind");
  if (m == 0) return WT_OK;
  CU(cudaSetDevice(b->device));
  cudaStream_t st = b->stream;
  const LevelDev d = bits_dev(b);
  if (flags & WT_F_DEVICE_PTRS) {
    CU(launch_bits_query(d, b->l2_shift, b->rate, b->rate_log, kind, (const i64*)args, (i64*)out, m, st));
    CU(cudaStreamSynchronize(st));
    return WT_OK;
  }
  Scratch S{{}, st};
  i64 *da, *dout;
  TRY(S.get(&da, m));
  TRY(S.get(&dout, m));
  CU(cudaMemcpyAsync(da, args, m * 8, cudaMemcpyHostToDevice, st));
  CU(launch_bits_query(d, b->l2_shift, b->rate, b->rate_log, kind, da, dout, m, st));
  CU(cudaMemcpyAsync(out, dout, m * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return WT_OK;
}

extern "C" int wt_bits_destroy(wt_bits* b) {
  if (!b) return WT_OK;
  free_bits(b);
  delete b;
  return WT_OK;
}
