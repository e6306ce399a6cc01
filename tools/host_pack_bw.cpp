// host-side packing throughput probe (iteration tool): i64 ids/args -> u16/u32
// wire records with T threads, and u32 -> i64 widening; prints GB/s of host
// traffic and queries/s.   g++ -O3 -march=native -pthread tools/host_pack_bw.cpp
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
int main(int argc, char** argv) {
  const size_t m = argc > 1 ? strtoull(argv[1], 0, 10) : (1ull << 25);
  int64_t *ids = (int64_t*)aligned_alloc(64, m * 8), *args = (int64_t*)aligned_alloc(64, m * 8);
  int64_t* out = (int64_t*)aligned_alloc(64, m * 8);
  uint16_t* w16 = (uint16_t*)aligned_alloc(64, m * 2);
  uint32_t* w32 = (uint32_t*)aligned_alloc(64, m * 4);
  for (size_t i = 0; i < m; ++i) { ids[i] = i & 255; args[i] = (i * 2654435761ull) & 0x3fffffff; }
  memset(out, 0, m * 8); memset(w16, 0, m * 2); memset(w32, 0, m * 4);
  for (int T : {1, 2, 4, 8, 12, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          const size_t a = m * t / T, b = m * (t + 1) / T;
          uint64_t bad = 0;
          for (size_t i = a; i < b; ++i) {
            const uint64_t c = (uint64_t)ids[i], p = (uint64_t)args[i];
            bad |= (c >> 16) | (p >> 32);
            w16[i] = (uint16_t)c; w32[i] = (uint32_t)p;
          }
          if (bad) w16[a] ^= 1;
        });
      for (auto& x : th) x.join();
      auto t1 = std::chrono::steady_clock::now();
      th.clear();
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          const size_t a = m * t / T, b = m * (t + 1) / T;
          for (size_t i = a; i < b; ++i) out[i] = (int64_t)w32[i];
        });
      for (auto& x : th) x.join();
      auto t2 = std::chrono::steady_clock::now();
      const double p = std::chrono::duration<double>(t1 - t0).count(),
                   u = std::chrono::duration<double>(t2 - t1).count();
      printf("T=%2d pack %.2f ms (%.1f GB/s, %.0f Mq/s)  widen %.2f ms (%.1f GB/s)\n", T, p * 1e3,
             m * 22 / p / 1e9, m / p / 1e6, u * 1e3, m * 12 / u / 1e9);
    }
  }
  printf("check %d %u %lld\n", (int)w16[7], w32[9], (long long)out[11]);
}
