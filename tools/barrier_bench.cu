// Grid-barrier microbenchmark (cooperative launch, one CTA per SM, 352
// threads): time per barrier for the monotonic-counter barrier used by the
// persistent apply and two alternatives, with and without global stores
// before each barrier (the release has to drain them).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/barrier_bench tools/barrier_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long atomAddRelease(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long ldAcquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void redRelease(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void stRelease(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// V0: current (atom.add.release returning, spin on the counter).
__device__ __forceinline__ void bar0(unsigned long long* c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long g = gridDim.x;
    const unsigned long long old = atomAddRelease(c, 1ULL);
    const unsigned long long target = (old / g + 1) * g;
    while (ldAcquire(c) < target) {
    }
  }
  __syncthreads();
}
// V1: red.release (no return), target from a per-CTA generation.
__device__ __forceinline__ void bar1(unsigned long long* c, unsigned long long& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    redRelease(c, 1ULL);
    while (ldAcquire(c) < target) {
    }
  }
  __syncthreads();
}
// V2: per-CTA arrival flags (128 B apart), CTA 0 warp 0 gathers, one
// release word everyone polls.
__device__ __forceinline__ void bar2(unsigned long long* flags, unsigned long long* rel, unsigned long long gen) {
  __syncthreads();
  if (blockIdx.x == 0) {
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) stRelease(flags + 0, gen);
      for (int k = threadIdx.x; k < gridDim.x; k += 32)
        while (ldAcquire(flags + 16 * k) < gen) {
        }
      __syncwarp();
      if (threadIdx.x == 0) stRelease(rel, gen);
    }
  } else if (threadIdx.x == 0) {
    stRelease(flags + 16 * blockIdx.x, gen);
    while (ldAcquire(rel) < gen) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long atomAddAcqRel(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
// V3: two-level counters. CTA b arrives on group counter b % G (own 128 B
// line); the group's last arriver bumps the top counter; all poll the top.
// All counters are monotonic from 0: generation q from the group counter.
__device__ __forceinline__ void bar3(unsigned long long* grp, unsigned long long* top, int G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int gi = blockIdx.x % G;
    const unsigned long long sz = gridDim.x / G + (gi < static_cast<int>(gridDim.x % G) ? 1 : 0);
    const unsigned long long old = atomAddRelease(grp + 16 * gi, 1ULL);
    const unsigned long long q = old / sz;
    if (old % sz == sz - 1) atomAddAcqRel(top, 1ULL);
    const unsigned long long target = (q + 1) * G;
    while (ldAcquire(top) < target) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long ldRelaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long atomAddRelaxed(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.relaxed.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
// V4: release arrival, relaxed polling, one acquire fence after.
__device__ __forceinline__ void bar4(unsigned long long* c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long g = gridDim.x;
    const unsigned long long old = atomAddRelease(c, 1ULL);
    const unsigned long long target = (old / g + 1) * g;
    while (ldRelaxed(c) < target) {
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
// V5: fence + relaxed atomic + relaxed polling + fence.
__device__ __forceinline__ void bar5(unsigned long long* c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long g = gridDim.x;
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const unsigned long long old = atomAddRelaxed(c, 1ULL);
    const unsigned long long target = (old / g + 1) * g;
    while (ldRelaxed(c) < target) {
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
// V6: as V4 without the trailing fence (timing only: not a correct barrier).
__device__ __forceinline__ void bar6(unsigned long long* c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long g = gridDim.x;
    const unsigned long long old = atomAddRelaxed(c, 1ULL);
    const unsigned long long target = (old / g + 1) * g;
    while (ldRelaxed(c) < target) {
    }
  }
  __syncthreads();
}

// V8: cluster-assisted. The cluster's CTAs meet at the hardware cluster
// barrier (release / acquire at cluster scope), its rank-0 CTA alone
// arrives on the global counter (grid / cluster-size arrivals instead of
// one per CTA) and polls, then the cluster meets again.
__device__ __forceinline__ void clusterSync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned clusterRank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned clusterSize() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void bar8(unsigned long long* c) {
  clusterSync();
  if (clusterRank() == 0 && threadIdx.x == 0) {
    const unsigned long long g = gridDim.x / clusterSize();
    const unsigned long long old = atomAddRelease(c, 1ULL);
    const unsigned long long target = (old / g + 1) * g;
    while (ldAcquire(c) < target) {
    }
  }
  clusterSync();
}

// V9: one arrival counter (acq_rel atomics, nobody polls it); the last
// arriver (thread 0) broadcasts the generation to per-CTA flag lines
// (128 B apart); every CTA polls only its own line.
// V10: as V9 with warp 0: lane 0 arrives, the last arriver's 32 lanes write
// the flags (grid/32 stores each).
// V11: V0 with a 32 ns back-off between polls.
__device__ __forceinline__ unsigned long long atomAddAcqRelU(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ void bar9(unsigned long long* c, unsigned long long* flags, unsigned long long gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long g = gridDim.x;
    const unsigned long long old = atomAddAcqRelU(c, 1ULL);
    if (old % g == g - 1)
      for (unsigned k = 0; k < gridDim.x; ++k) stRelease(flags + 16 * k, gen);
    while (ldAcquire(flags + 16 * blockIdx.x) < gen) {
    }
  }
  __syncthreads();
}
__device__ __forceinline__ void bar10(unsigned long long* c, unsigned long long* flags, unsigned long long gen) {
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned long long g = gridDim.x;
    unsigned long long old = 0;
    if (threadIdx.x == 0) old = atomAddAcqRelU(c, 1ULL);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old % g == g - 1) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      for (unsigned k = threadIdx.x; k < gridDim.x; k += 32)
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(flags + 16 * k), "l"(gen) : "memory");
    }
    if (threadIdx.x == 0)
      while (ldAcquire(flags + 16 * blockIdx.x) < gen) {
      }
    __syncwarp();
  }
  __syncthreads();
}
__device__ __forceinline__ void bar11(unsigned long long* c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long g = gridDim.x;
    const unsigned long long old = atomAddRelease(c, 1ULL);
    const unsigned long long target = (old / g + 1) * g;
    while (ldAcquire(c) < target) __nanosleep(32);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(352, 1) kern(int variant, int iters, int stores, unsigned long long* c,
                                               unsigned long long* flags, unsigned long long* rel, double* buf,
                                               long long* out) {
  unsigned long long target = ldAcquire(c);  // V1 base (a multiple of grid size)
  unsigned long long gen = ldAcquire(rel);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int s = 0; s < stores; ++s)
      buf[(static_cast<long long>(s) * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x] = it + s;
    if (variant == 0)
      bar0(c);
    else if (variant == 1)
      bar1(c, target);
    else if (variant == 2)
      bar2(flags, rel, ++gen);
    else if (variant == 4)
      bar4(c);
    else if (variant == 5)
      bar5(c);
    else if (variant == 7)
      bar6(c);
    else if (variant == 8)
      bar8(c);
    else if (variant == 9)
      bar9(c, flags, ++gen);
    else if (variant == 10)
      bar10(c, flags, ++gen);
    else if (variant == 11)
      bar11(c);
    else
      bar3(flags, rel + 16, variant - 2);
  }
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  unsigned long long *c, *flags, *rel;
  double* buf;
  long long* out;
  cudaMalloc(&c, 8);
  cudaMalloc(&flags, 8 * 16 * sms);
  cudaMalloc(&rel, 8 * 64);
  cudaMalloc(&buf, 8LL * 64 * sms * 352);
  cudaMalloc(&out, 8);
  cudaMemset(c, 0, 8);
  cudaMemset(flags, 0, 8 * 16 * sms);
  cudaMemset(rel, 0, 8 * 64);
  const int iters = 2000;
  for (int stores : {0, 8, 32}) {
    for (int v : {0, 1, 4, 5, 7, 9, 10, 11}) {
      cudaMemset(c, 0, 8);
      cudaMemset(flags, 0, 8 * 16 * sms);
      cudaMemset(rel, 0, 8 * 64);
      void* args[] = {&v, const_cast<int*>(&iters), &stores, &c, &flags, &rel, &buf, &out};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaLaunchCooperativeKernel((void*)kern, sms, 352, args, 0, 0);  // warm-up
      cudaMemset(c, 0, 8);
      cudaMemset(flags, 0, 8 * 16 * sms);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)kern, sms, 352, args, 0, 0);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("variant %2d stores/thread %2d: %.3f us per barrier (%s)\n", v, stores, 1e3 * ms / iters,
             cudaGetErrorString(err));
    }
  }
  for (int cs : {2, 4}) {
    for (int stores : {0, 8}) {
      int v = 8;
      cudaMemset(c, 0, 8);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(sms);
      cfg.blockDim = dim3(352);
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      at[1].id = cudaLaunchAttributeClusterDimension;
      at[1].val.clusterDim.x = cs;
      at[1].val.clusterDim.y = 1;
      at[1].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      int ncl = 0;
      cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &cfg);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaError_t el = cudaLaunchKernelEx(&cfg, kern, v, iters, stores, c, flags, rel, buf, out);
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, kern, v, iters, stores, c, flags, rel, buf, out);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("variant  8 cluster %d (max active clusters %d) stores/thread %2d: %.3f us per barrier (%s / %s)\n", cs,
             ncl, stores, 1e3 * ms / iters, cudaGetErrorString(el), cudaGetErrorString(err));
    }
  }
  return 0;
}
