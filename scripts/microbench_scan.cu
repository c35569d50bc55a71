// Microbenchmark: latency of one warp streaming one 10 KB row (u8) with U
// 128-bit loads in flight per lane, rows cold (HBM) vs warm (L2).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench_scan.cu
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int U>
__global__ void scan_rows(const uint4* __restrict__ kT, int lda16, int nrows, const int* rows,
                          unsigned long long* out, unsigned* sink) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (w >= nrows) return;
  const uint4* r = kT + (size_t)rows[w] * lda16;
  unsigned acc = 0;
  __syncwarp();
  const unsigned long long t0 = gt();
  for (int v = 0; v < lda16; v += 32 * U) {
    uint4 x[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int vi = v + j * 32 + lane;
      x[j] = vi < lda16 ? __ldg(r + vi) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) acc += __vcmpeq4(x[j].x, 0x05050505u) | x[j].y ^ x[j].z ^ x[j].w;
    if (__ballot_sync(0xffffffffu, acc == 0x12345678u)) break;
  }
  const unsigned long long t1 = gt();
  if (lane == 0) out[w] = t1 - t0;
  if (acc == 0x9u) sink[0] = acc;
}

int main() {
  const int n = 10000, lda = 10240, lda16 = lda / 16;
  const size_t bytes = (size_t)n * lda;
  uint4* kT;
  cudaMalloc(&kT, bytes);
  cudaMemset(kT, 1, bytes);
  void* flush;
  cudaMalloc(&flush, 512u << 20);
  int* rows;
  cudaMalloc(&rows, 4096 * 4);
  std::vector<int> hr(4096);
  for (int i = 0; i < 4096; ++i) hr[i] = (int)((i * 2654435761u) % n);
  cudaMemcpy(rows, hr.data(), 4096 * 4, cudaMemcpyHostToDevice);
  unsigned long long* out;
  cudaMallocManaged(&out, 4096 * 8);
  unsigned* sink;
  cudaMalloc(&sink, 4);
  for (int nw : {148, 1184}) {
    for (int warm = 0; warm < 2; ++warm) {
      for (int u : {2, 4, 8, 16, 20}) {
        if (!warm) cudaMemset(flush, u, 512u << 20);
        else {  // warm: touch the rows first
          scan_rows<4><<<nw, 32>>>(kT, lda16, nw, rows, out, sink);
        }
        cudaDeviceSynchronize();
        switch (u) {
          case 2: scan_rows<2><<<nw, 32>>>(kT, lda16, nw, rows, out, sink); break;
          case 4: scan_rows<4><<<nw, 32>>>(kT, lda16, nw, rows, out, sink); break;
          case 8: scan_rows<8><<<nw, 32>>>(kT, lda16, nw, rows, out, sink); break;
          case 16: scan_rows<16><<<nw, 32>>>(kT, lda16, nw, rows, out, sink); break;
          case 20: scan_rows<20><<<nw, 32>>>(kT, lda16, nw, rows, out, sink); break;
        }
        cudaDeviceSynchronize();
        double mx = 0, avg = 0;
        for (int i = 0; i < nw; ++i) {
          mx = out[i] > mx ? out[i] : mx;
          avg += out[i];
        }
        printf("warps=%4d %s U=%2d  avg %.2f us  max %.2f us\n", nw, warm ? "L2  " : "HBM ", u,
               avg / nw / 1e3, mx / 1e3);
      }
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
