// Streaming-bandwidth sweep on one B200 (tuning tool, not product code):
// what read/write mix, vector count per thread, CTA size and residency reach
// the highest HBM throughput?  Prints one line per configuration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

#include "../common.cuh"

using namespace mco;

template <int NR, int NW, int U, bool HINT>
__global__ void stream_kernel(float* const* bufs, uint64_t nvec) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = tid; base < nvec; base += stride * U) {
    float v[U][NR > 0 ? NR : 1][8] = {};
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = base + u * stride;
      if (vi < nvec) {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          if (HINT)
            ld_stream(bufs[r] + vi * 8, v[u][r]);
          else
            ld_stream(bufs[r] + vi * 8, v[u][r]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = base + u * stride;
      if (vi < nvec) {
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float s = 0.f;
#pragma unroll
          for (int r = 0; r < NR; ++r) s += v[u][r][j];
          o[j] = s;
        }
#pragma unroll
        for (int w = 0; w < NW; ++w) st_stream(bufs[w] + vi * 8, o);
        if (NW == 0 && o[0] == 12345.f) bufs[0][0] = o[1];
      }
    }
  }
}

template <int NR, int NW, int U>
void run(const char* name, float* const* dbufs, uint64_t n, int sms) {
  auto k = stream_kernel<NR, NW, U, true>;
  for (int threads : {256, 512}) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, 0);
    for (int bps : {1, 2, 4, 8}) {
      if (bps > per_sm) continue;
      const int grid = sms * bps;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      k<<<grid, threads>>>(dbufs, n / 8);
      cudaEventRecord(a);
      const int it = 5;
      for (int i = 0; i < it; ++i) k<<<grid, threads>>>(dbufs, n / 8);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)n * 4 * (NR + NW);
      printf("%-10s U=%d threads=%d ctas/sm=%d (max %d): %.1f GB/s\n", name, U, threads, bps,
             per_sm, bytes * it / (ms * 1e-3) / 1e9);
    }
  }
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t n = 1ull << 30;  // 4 GiB per buffer
  std::vector<float*> bufs(7);
  float** dbufs;
  cudaMalloc(&dbufs, sizeof(float*) * 7);
  if (argc > 1) {  // staggered sub-buffers of one allocation: stagger bytes = argv[1]
    const uint64_t stg = strtoull(argv[1], nullptr, 10);
    char* big;
    cudaMalloc(&big, 7 * (n * 4 + stg) + 4096);
    cudaMemset(big, 0, 7 * (n * 4 + stg));
    for (int i = 0; i < 7; ++i) bufs[i] = (float*)(big + i * (n * 4 + stg));
    cudaMemcpy(dbufs, bufs.data(), sizeof(float*) * 7, cudaMemcpyHostToDevice);
    printf("stagger %llu bytes\n", (unsigned long long)stg);
    run<6, 5, 1>("adan6r5w", dbufs, n, sms);
    run<4, 3, 1>("adamw4r3w", dbufs, n, sms);
    return 0;
  }
  for (auto& p : bufs) {
    cudaMalloc(&p, n * 4);
    cudaMemset(p, 0, n * 4);
  }
  cudaMemcpy(dbufs, bufs.data(), sizeof(float*) * 7, cudaMemcpyHostToDevice);
  run<6, 5, 1>("adan6r5w", dbufs, n, sms);
  run<1, 1, 1>("copy", dbufs, n, sms);
  run<1, 1, 2>("copy", dbufs, n, sms);
  run<1, 1, 4>("copy", dbufs, n, sms);
  run<1, 0, 4>("read", dbufs, n, sms);
  run<0, 1, 4>("write", dbufs, n, sms);
  run<4, 3, 1>("adamw4r3w", dbufs, n, sms);
  run<4, 3, 2>("adamw4r3w", dbufs, n, sms);
  run<6, 5, 1>("adan6r5w", dbufs, n, sms);
  run<2, 1, 2>("lomo2r1w", dbufs, n, sms);
  run<2, 1, 4>("lomo2r1w", dbufs, n, sms);
  printf("done\n");
  return 0;
}
