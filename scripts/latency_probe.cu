// Dependent-latency probe for the phase loop's building blocks on B200
// (one warp, clock64 over a dependent chain of 2,000 operations):
// L2-hit load (ld.cg), 64-bit global atomicMin, fence.acq_rel.gpu (with and
// without an outstanding store), cluster barrier, DSMEM load / atomic.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/latency_probe scripts/latency_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int N = 2000;

__global__ void chain_kernel(unsigned* buf, unsigned long long* buf64, long long* out) {
  if (threadIdx.x != 0) return;
  // L2-hit pointer chase (buf[i] = next index, 1 MB ring -> L2 resident)
  unsigned j = 0;
  for (int i = 0; i < 200; ++i) j = __ldcg(buf + j);
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) j = __ldcg(buf + j);
  long long t1 = clock64();
  out[0] = (t1 - t0) / N;
  // dependent 64-bit atomicMin (address depends on the previous result)
  unsigned long long v = 0;
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = atomicMin(buf64 + ((v + i) & 1023) * 16, ~0ull - i);
  t1 = clock64();
  out[1] = (t1 - t0) / N + (v == 7 ? 1 : 0);
  // fence with nothing outstanding
  t0 = clock64();
  for (int i = 0; i < N; ++i) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  t1 = clock64();
  out[2] = (t1 - t0) / N;
  // store + fence
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    buf[(i * 977) & 262143] = i;
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  t1 = clock64();
  out[3] = (t1 - t0) / N;
  // red.release (fire and forget) + ld.acquire of the same word
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(buf + 300000) : "memory");
    unsigned x;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(buf + 300000) : "memory");
    j += x;
  }
  t1 = clock64();
  out[4] = (t1 - t0) / N + (j == 7 ? 1 : 0);
}

__global__ void cluster_kernel(long long* out) {
  __shared__ unsigned long long word[64];
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x < 64) word[threadIdx.x] = 0;
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) cl.sync();
  long long t1 = clock64();
  if (cl.block_rank() == 0 && threadIdx.x == 0) out[5] = (t1 - t0) / N;
  // DSMEM dependent load chain / atomics from CTA 0 to CTA 7
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    unsigned long long* remote = cl.map_shared_rank(word, (int)cl.num_blocks() - 1);
    unsigned long long v = 0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = remote[v & 31];
    t1 = clock64();
    out[6] = (t1 - t0) / N + (v == 77 ? 1 : 0);
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = atomicMin(remote + ((v + i) & 31), ~0ull - i);
    t1 = clock64();
    out[7] = (t1 - t0) / N + (v == 77 ? 1 : 0);
  }
  cl.sync();
}

int main() {
  unsigned* buf;
  unsigned long long* buf64;
  long long* out;
  cudaMalloc(&buf, 4 << 20);
  cudaMalloc(&buf64, 1 << 20);
  cudaMalloc(&out, 64);
  cudaMemset(buf64, 0xff, 1 << 20);
  unsigned* h = new unsigned[1 << 18];
  for (int i = 0; i < (1 << 18); ++i) h[i] = (unsigned)((i * 40503ull + 12345) % (1 << 18));
  cudaMemcpy(buf, h, 1 << 20, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    chain_kernel<<<1, 32>>>(buf, buf64, out);
    for (int cs : {8, 16}) {
      cudaFuncSetAttribute(cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, cluster_kernel, out);
      cudaDeviceSynchronize();
      long long o2[8];
      cudaMemcpy(o2, out, 64, cudaMemcpyDeviceToHost);
      printf("cluster %d: cluster.sync %lld | DSMEM load %lld | DSMEM atomicMin64 %lld (%s)\n", cs, o2[5], o2[6], o2[7],
             cudaGetErrorString(cudaGetLastError()));
    }
    cudaDeviceSynchronize();
    long long o[8];
    cudaMemcpy(o, out, 64, cudaMemcpyDeviceToHost);
    printf("cycles: L2-hit load %lld | atomicMin64 %lld | fence (idle) %lld | store+fence %lld | "
           "red.release+ld.acquire %lld | cluster.sync(16) %lld | DSMEM load %lld | DSMEM atomicMin64 %lld  (%s)\n",
           o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
