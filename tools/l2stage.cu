// Does staging part of a >L2 stream in L2 ahead of time shorten the stream?
// (not part of the product). A 134 MB buffer (the C2 half spectrum) is read
// through the apply's cp.async.bulk ring (4 stages x 32 KB per SM, chunks
// strided over the grid). Before each timed ring pass, a prefetch kernel
// issues cp.async.bulk.prefetch.L2 for the first X MB in ring order (each
// CTA its own first chunks) and a spin kernel waits ~12 us (the apply's
// transform phases); the ring pass is timed alone with events.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2506_04710_b200/csrc l2stage.cu -o l2stage
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace tbt;

constexpr int STAGES = 4;
constexpr uint32_t CHUNK = 32768;

__global__ void __launch_bounds__(288, 1) ringRead(const char* __restrict__ src, long long nchunks, int evictFirst,
                                                   double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CHUNK);
  uint64_t* empty = full + STAGES;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbarInit(full + s, 1); mbarInit(empty + s, 8); }
    fenceBarrierInit();
  }
  __syncthreads();
  long long mine = (nchunks - 1 - blockIdx.x) / gridDim.x + 1;
  if (warp == 8) {
    if (lane == 0) {
      uint64_t pol = evictFirst ? policyEvictFirst() : policyEvictLast();
      for (long long it = 0; it < mine; ++it) {
        int s = it % STAGES; uint32_t ph = (it / STAGES) & 1;
        mbarWait(empty + s, ph ^ 1u);
        mbarArriveExpectTx(full + s, CHUNK);
        bulkG2S(smem + s * CHUNK, src + (blockIdx.x + it * gridDim.x) * (long long)CHUNK, CHUNK, full + s, pol);
      }
    }
    return;
  }
  double acc = 0;
  for (long long it = 0; it < mine; ++it) {
    int s = it % STAGES; uint32_t ph = (it / STAGES) & 1;
    mbarWait(full + s, ph);
    // touch the stage like a consumer (8 warps x 32 lanes x 16 doubles)
    const double* d = reinterpret_cast<const double*>(smem + s * CHUNK);
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += d[threadIdx.x + 256 * u];
    __syncwarp();
    if (lane == 0) mbarArrive(empty + s);
  }
  if (acc == 1234.5) out[0] = acc;
}

// Each CTA prefetches its first `per` chunks (ring order) into L2.
__global__ void prefetchKernel(const char* __restrict__ src, long long nchunks, long long per) {
  if (threadIdx.x != 0) return;
  for (long long it = 0; it < per; ++it) {
    const long long c = blockIdx.x + it * gridDim.x;
    if (c < nchunks) bulkPrefetchL2(src + c * (long long)CHUNK, CHUNK);
  }
}

// Each CTA warms its first `per` chunks into L2 with real loads (ld.global, evict-last).
__global__ void warmKernel(const char* __restrict__ src, long long nchunks, long long per, double* out) {
  double acc = 0;
  for (long long it = 0; it < per; ++it) {
    const long long c = blockIdx.x + it * gridDim.x;
    if (c >= nchunks) break;
    const double* d = reinterpret_cast<const double*>(src + c * (long long)CHUNK);
    for (int k = threadIdx.x; k < (int)(CHUNK / 8); k += blockDim.x * 4) acc += __ldcg(d + k);  // one load per 32 B sector
  }
  if (acc == 1234.5) out[0] = acc;
}

__global__ void spin(long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < (unsigned long long)ns);
}

// Read-only L2 flush (no dirty lines left behind to write back).
__global__ void flushKernel(const double* p, long long n, double* out) {
  double acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) acc += p[i];
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  const long long bytes = 134LL << 20;
  const long long nch = bytes / CHUNK;
  char* buf; double* out; double* fl;
  const long long flN = (256LL << 20) / 8;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 8); cudaMalloc(&fl, flN * 8);
  cudaMemset(buf, 0, bytes); cudaMemset(fl, 0, flN * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t sm = STAGES * (size_t)CHUNK + 2 * STAGES * 8;
  cudaFuncSetAttribute(ringRead, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int ef : {1, 2}) {
   for (long long spinNs : {12000LL}) {
    for (long long mb : {0LL, 20LL, 40LL, 60LL, 80LL, 100LL}) {
      const long long per = (mb << 20) / CHUNK / sms;
      float best = 1e9, tot = 0;
      const int R = 20;
      for (int r = 0; r < R + 2; ++r) {
        flushKernel<<<sms * 4, 256>>>(fl, flN, out);
        spin<<<1, 32>>>(5000);
        if (per > 0 && ef == 1) prefetchKernel<<<sms, 32>>>(buf, nch, per);
        if (per > 0 && ef == 2) warmKernel<<<sms, 256>>>(buf, nch, per, out);
        spin<<<1, 32>>>(spinNs);
        cudaEventRecord(a);
        ringRead<<<sms, 288, sm>>>(buf, nch, 1, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (r >= 2) { best = ms < best ? ms : best; tot += ms; }
      }
      printf("%s spin %5lld ns prefetched %3lld MB: ring pass best %.2f us, mean %.2f us (%.0f GB/s on 134 MB)\n",
             ef == 1 ? "bulk-prefetch" : "warm-loads", spinNs, mb, best * 1e3, tot / R * 1e3, bytes / (best * 1e-3) / 1e9);
    }
   }
  }
  // L2-resident stream: a 48 MB buffer read back to back (fits in L2)
  {
    const long long nch48 = (48LL << 20) / CHUNK;
    float ms; const int R = 50;
    for (int r = 0; r < 3; ++r) ringRead<<<sms, 288, sm>>>(buf, nch48, 0, out);
    cudaEventRecord(a);
    for (int r = 0; r < R; ++r) ringRead<<<sms, 288, sm>>>(buf, nch48, 0, out);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("L2-resident 48 MB ring passes: %.2f us each (%.0f GB/s)\n", ms / R * 1e3, (48LL << 20) / (ms / R * 1e-3) / 1e9);
    const long long nch8 = (8LL << 20) / CHUNK;
    cudaEventRecord(a);
    for (int r = 0; r < R; ++r) ringRead<<<sms, 288, sm>>>(buf, nch8, 0, out);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("8 MB ring passes (launch + ramp floor): %.2f us each\n", ms / R * 1e3);
  }
  // back to back ring passes, no flush, no prefetch
  {
    float ms; const int R = 50;
    for (int r = 0; r < 3; ++r) ringRead<<<sms, 288, sm>>>(buf, nch, 1, out);
    cudaEventRecord(a);
    for (int r = 0; r < R; ++r) ringRead<<<sms, 288, sm>>>(buf, nch, 1, out);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("back-to-back ring passes: %.2f us each\n", ms / R * 1e3);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
