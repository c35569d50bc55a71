// Grid-barrier latency on B200: how long does one barrier of a persistent
// cooperative grid (148 blocks x 512 threads, one per SM) take, and what do
// the arrival form (one counter: red.release vs per-block flags: st.release)
// and the poll form (ld.acquire per iteration vs relaxed + one fence) cost?
// S > 0: each warp issues S scattered stores right before arriving (the
// chain outputs the phase loop writes just before its barrier).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/barrier_probe scripts/barrier_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int MODE, int P = 150>
__global__ void __launch_bounds__(512, 1) bar_kernel(unsigned* count, unsigned* flags, int iters,
                                                     int S, unsigned* junk, unsigned long long* out) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned target = 0;
  const unsigned long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    if (lane == 0)
      for (int s = 0; s < S; ++s)
        junk[((blockIdx.x * 16 + wib) * 977u + (unsigned)(it * 131 + s * 7919)) & ((1u << 22) - 1)] = it;
    __syncthreads();
    if constexpr (MODE == 0) {  // counter: red.release + ld.acquire polls (the phase loop's form)
      target += gridDim.x;
      if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        while ((int)(ld_acq(count) - target) < 0) {}
      }
    } else if constexpr (MODE == 1) {  // counter: red.release + relaxed polls + one fence
      target += gridDim.x;
      if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        while ((int)(ld_rlx(count) - target) < 0) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    } else if constexpr (MODE == 2) {  // per-block flags: st.release, warps poll 32 flags each
      if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"((unsigned)it) : "memory");
      if (wib * 32 < (int)gridDim.x) {
        const int f = wib * 32 + lane;
        while (true) {
          const unsigned v = f < (int)gridDim.x ? ld_rlx(flags + f) : (unsigned)it;
          if (__all_sync(0xffffffffu, (int)(v - (unsigned)it) >= 0)) break;
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    } else if constexpr (MODE == 3) {  // per-block flags, acquire polls
      if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"((unsigned)it) : "memory");
      if (wib * 32 < (int)gridDim.x) {
        const int f = wib * 32 + lane;
        while (true) {
          const unsigned v = f < (int)gridDim.x ? ld_acq(flags + f) : (unsigned)it;
          if (__all_sync(0xffffffffu, (int)(v - (unsigned)it) >= 0)) break;
        }
      }
    } else if constexpr (MODE == 4) {  // counter, atom (returns) + relaxed polls
      target += gridDim.x;
      if (threadIdx.x == 0) {
        unsigned old;
        asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(count) : "memory");
        if (old + 1 != target)
          while ((int)(ld_rlx(count) - target) < 0) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    if constexpr (MODE == 10 || MODE == 11 || MODE == 12) {  // two-level: groups of GS blocks
      constexpr int GS = MODE == 10 ? 8 : (MODE == 11 ? 16 : 12);
      const int ng = (gridDim.x + GS - 1) / GS;
      const int g = blockIdx.x / GS;
      const int gsize = min(GS, (int)gridDim.x - g * GS);
      if (threadIdx.x == 0) {
        unsigned* grp = flags + 32 * (g + 1);  // one 128-byte line per group
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(grp) : "memory");
        if (old + 1 == (unsigned)(it * gsize))  // last of its group
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        while ((int)(ld_acq(count) - (unsigned)(it * ng)) < 0) {}
      }
    }
    if constexpr (MODE == 5 || MODE == 6) {  // counter barrier, then every block reads all P slots
      target += gridDim.x;
      if (threadIdx.x < P) junk[(1u << 22) - 4096 + threadIdx.x * 2] = it;  // (slot stores, tags)
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        while ((int)(ld_acq(count) - target) < 0) {}
      }
      __syncthreads();
      unsigned v = threadIdx.x < P ? __ldcg(junk + (1u << 22) - 4096 + threadIdx.x * 2) : 0u;
      if (__syncthreads_or(v == 0xffffffffu)) out[1] = v;
    }
    if constexpr (MODE == 7 || MODE == 8) {  // dataflow: tagged 64-bit slots, every block polls all P
      unsigned long long* sl = reinterpret_cast<unsigned long long*>(junk + (1u << 22) - 8192);
      // slot s is written by block s % grid (one store each; its outputs)
      for (int s2 = blockIdx.x; s2 < P; s2 += gridDim.x)
        if (threadIdx.x == 0) {
          if constexpr (MODE == 7) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(sl + s2), "l"((unsigned long long)it << 32 | s2) : "memory");
          else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(sl + s2), "l"((unsigned long long)it << 32 | s2) : "memory");
        }
      bool ok = true;
      if ((int)threadIdx.x < P) {
        while (true) {
          unsigned long long v;
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(sl + threadIdx.x) : "memory");
          if ((int)((unsigned)(v >> 32) - (unsigned)it) >= 0) break;
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      __syncthreads_and(ok);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
}

template <int MODE>
float run(int grid, int iters, int S, unsigned* count, unsigned* flags, unsigned* junk,
          unsigned long long* out) {
  cudaMemset(count, 0, 4);
  cudaMemset(flags, 0, 65536);
  void* args[] = {&count, &flags, &iters, &S, &junk, &out};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchCooperativeKernel((void*)bar_kernel<MODE>, grid, 512, args, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  if (cudaGetLastError() != cudaSuccess) return -1;
  return ms * 1000.f / iters;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *count, *flags, *junk;
  unsigned long long* out;
  cudaMalloc(&count, 4);
  cudaMalloc(&flags, 65536);
  cudaMalloc(&junk, 4u << 22);
  cudaMalloc(&out, 16);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    printf("P=150 counter barrier + read of all slots after (current top): %.3f us\n", run<5>(sms, iters, 0, count, flags, junk, out));
    printf("P=150 dataflow: tagged slots st.release, every block polls all : %.3f us\n", run<7>(sms, iters, 0, count, flags, junk, out));
    printf("P=150 dataflow: tagged slots st.relaxed, every block polls all : %.3f us\n", run<8>(sms, iters, 0, count, flags, junk, out));
  }
  const char* names[] = {"counter red.release + ld.acquire polls", "counter red.release + relaxed polls + fence",
                         "per-block flags st.release + relaxed polls + fence", "per-block flags + acquire polls",
                         "counter atom.release (last skips poll) + relaxed polls"};
  for (int g : {148, 128, 96, 74, 48, 37, 16})
    printf("flat counter, grid %3d: %.3f us (S=4: %.3f us)\n", g, run<0>(g, iters, 0, count, flags, junk, out),
           run<0>(g, iters, 4, count, flags, junk, out));
  for (int rep = 0; rep < 2; ++rep) {
    printf("two-level, groups of 8 : %.3f us\n", run<10>(sms, iters, 0, count, flags, junk, out));
    printf("two-level, groups of 16: %.3f us\n", run<11>(sms, iters, 0, count, flags, junk, out));
    printf("two-level, groups of 12: %.3f us\n", run<12>(sms, iters, 0, count, flags, junk, out));
    printf("flat counter           : %.3f us\n", run<0>(sms, iters, 0, count, flags, junk, out));
    printf("two-level 8, S=4       : %.3f us\n", run<10>(sms, iters, 4, count, flags, junk, out));
    printf("flat counter, S=4      : %.3f us\n", run<0>(sms, iters, 4, count, flags, junk, out));
  }
  for (int S : {0, 4, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      float us[5] = {run<0>(sms, iters, S, count, flags, junk, out), run<1>(sms, iters, S, count, flags, junk, out),
                     run<2>(sms, iters, S, count, flags, junk, out), run<3>(sms, iters, S, count, flags, junk, out),
                     run<4>(sms, iters, S, count, flags, junk, out)};
      for (int m = 0; m < 5; ++m) printf("S=%2d grid=%d  %-55s %.3f us/barrier\n", S, sms, names[m], us[m]);
    }
  }
  return 0;
}
