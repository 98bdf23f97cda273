// Grid-wide barrier for cooperative (co-resident) launches.
#pragma once

#include <cstdint>

namespace tbt {

// One monotonic 64-bit arrival counter: each CTA adds 1 with release
// semantics and spins (acquire loads, no sleep) until the counter reaches the
// next multiple of the grid size. Nothing is reset, so consecutive barriers
// and launches need no generation word; the counter must start at a multiple
// of gridDim.x (0) for the first launch that uses it.
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

// Thread 0's arrival/wait part; callers wrap it in __syncthreads().
__device__ __forceinline__ void gridArriveWait(unsigned long long* counter) {
  const unsigned long long g = gridDim.x;
  const unsigned long long old = atomAddRelease(counter, 1ULL);
  const unsigned long long target = (old / g + 1) * g;
  uint32_t spin = 0;
  while (ldAcquire(counter) < target)
    if (++spin > (1u << 30)) __trap();
}

__device__ __forceinline__ void gridBarrierMono(unsigned long long* counter) {
  __syncthreads();
  if (threadIdx.x == 0) gridArriveWait(counter);
  __syncthreads();
}

}  // namespace tbt
