// Read-bandwidth calibration for the phase-1 propose scan: how fast can a
// B200 stream a 200 MB buffer (config 2, uint16 kT) with plain 128-bit loads
// vs 1-D TMA bulk copies?  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -o /tmp/bw_probe scripts/bw_probe.cu && /tmp/bw_probe [MB]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int U>
__global__ void ldg_min(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned m = 0xffffffffu;
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 x[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const size_t k = i + (size_t)j * blockDim.x;
      x[j] = k < n ? __ldg(p + k) : make_uint4(~0u, ~0u, ~0u, ~0u);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) m = __vminu2(m, __vminu2(__vminu2(x[j].x, x[j].y), __vminu2(x[j].z, x[j].w)));
  }
  if (m == 0x12345678u) out[0] = m;
}

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// one CTA per SM; W warps, each with a D-deep ring of C-byte chunks
template <int W, int D>
__global__ void tma_min(const char* __restrict__ p, size_t bytes, int C, unsigned* out) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) unsigned long long bar[W][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t nchunks = bytes / C;
  const size_t gw = (size_t)blockIdx.x * W + warp, nw = (size_t)gridDim.x * W;
  unsigned char* my = ring + (size_t)warp * D * C;
  if (lane == 0) {
    for (int s = 0; s < D; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const size_t items = gw < nchunks ? (nchunks - 1 - gw) / nw + 1 : 0;
  auto issue = [&](size_t it) {
    const int s = it % D;
    const char* src = p + (gw + it * nw) * C;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[warp][s])), "r"(C));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(my + (size_t)s * C)),
                 "l"(src), "r"(C), "r"(su32(&bar[warp][s])) : "memory");
  };
  if (lane == 0)
    for (size_t it = 0; it < items && it < D; ++it) issue(it);
  unsigned m = 0xffffffffu;
  for (size_t it = 0; it < items; ++it) {
    const int s = it % D;
    const unsigned par = (it / D) & 1;
    asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(
                     su32(&bar[warp][s])), "r"(par) : "memory");
    const uint4* v = reinterpret_cast<const uint4*>(my + (size_t)s * C);
    for (int i = lane; i < C / 16; i += 32) {
      const uint4 x = v[i];
      m = __vminu2(m, __vminu2(__vminu2(x.x, x.y), __vminu2(x.z, x.w)));
    }
    __syncwarp();
    if (lane == 0 && it + D < items) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(it + D);
    }
  }
  if (m == 0x12345678u) out[0] = m;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 12; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2 && ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? atoi(argv[1]) : 200;
  const size_t bytes = mb << 20;
  char* p;
  unsigned* out;
  cudaMalloc(&p, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(p, 1, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t n = bytes / 16;
  auto rep = [&](const char* name, float ms) {
    printf("%-34s %8.2f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  };
  for (int bpsm : {4, 8}) {
    char nm[64];
    snprintf(nm, 64, "ldg U=4 256thr x %d/SM", bpsm);
    rep(nm, timeit([&] { ldg_min<4><<<sms * bpsm, 256>>>((const uint4*)p, n, out); }));
    snprintf(nm, 64, "ldg U=8 256thr x %d/SM", bpsm);
    rep(nm, timeit([&] { ldg_min<8><<<sms * bpsm, 256>>>((const uint4*)p, n, out); }));
  }
  for (int C : {4096, 8192, 16384}) {
    char nm[64];
    {
      const size_t smem = 8 * 3 * (size_t)C;
      if (smem <= 220 * 1024) {
        cudaFuncSetAttribute(tma_min<8, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        snprintf(nm, 64, "tma W=8 D=3 C=%d", C);
        rep(nm, timeit([&] { tma_min<8, 3><<<sms, 256, smem>>>(p, bytes, C, out); }));
      }
    }
    {
      const size_t smem = 4 * 4 * (size_t)C;
      if (smem <= 220 * 1024) {
        cudaFuncSetAttribute(tma_min<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        snprintf(nm, 64, "tma W=4 D=4 C=%d", C);
        rep(nm, timeit([&] { tma_min<4, 4><<<sms, 128, smem>>>(p, bytes, C, out); }));
      }
    }
    {
      const size_t smem = 16 * 2 * (size_t)C;
      if (smem <= 220 * 1024) {
        cudaFuncSetAttribute(tma_min<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        snprintf(nm, 64, "tma W=16 D=2 C=%d", C);
        rep(nm, timeit([&] { tma_min<16, 2><<<sms, 512, smem>>>(p, bytes, C, out); }));
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
