// gather_peak.cu -- measured ceiling for the query kernels' access pattern:
// every thread walks `steps` dependent random 64-byte lines of a table much
// larger than L2 (the rank-line layout: one line per rank step).  Reports
// line-bytes/s, i.e. the HBM throughput random 64 B lines can reach on this
// B200, next to a plain streaming copy measured the same way.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gather_peak.cu -o tools/gather_peak
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ ulonglong2 ld_line16(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L2::64B.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

__global__ void walk(const ulonglong2* __restrict__ lines, uint64_t n_lines, uint64_t m, int steps,
                     uint64_t* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  uint64_t x = i * 0x9E3779B97F4A7C15ull + 12345;
  uint64_t acc = 0;
  for (int s = 0; s < steps; ++s) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 29;
    const uint64_t li = (x + acc) & (n_lines - 1);  // dependent on the previous line
    const ulonglong2* L = lines + li * 4;
    const ulonglong2 a = ld_line16(L), b = ld_line16(L + 1), c = ld_line16(L + 2), d = ld_line16(L + 3);
    acc += (a.x ^ b.y ^ c.x ^ d.y) & 1;
  }
  out[i] = acc;
}

__global__ void copyk(const uint4* __restrict__ a, uint4* __restrict__ b, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main() {
  const uint64_t bytes = 2ull << 30;  // 2 GiB table (>> 126 MB L2), power of two lines
  const uint64_t n_lines = bytes / 64;
  ulonglong2* lines;
  uint64_t* out;
  const uint64_t m = 33333334;
  cudaMalloc(&lines, bytes);
  cudaMemset(lines, 0x5a, bytes);
  cudaMalloc(&out, m * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int steps : {1, 8}) {
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      walk<<<(unsigned)((m + 255) / 256), 256>>>(lines, n_lines, m, steps, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 3)
        printf("{\"probe\": \"random_64B_lines\", \"steps\": %d, \"lines_per_s\": %.4g, \"GB_per_s\": %.1f}\n",
               steps, m * steps / (ms / 1e3), m * steps * 64.0 / (ms / 1e3) / 1e9);
    }
  }
  const uint64_t half = bytes / 2 / 16;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    copyk<<<148 * 8, 512>>>((const uint4*)lines, (uint4*)lines + half, half);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep == 3)
      printf("{\"probe\": \"stream_copy\", \"GB_per_s\": %.1f}\n", 2.0 * half * 16 / (ms / 1e3) / 1e9);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
