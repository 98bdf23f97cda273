// Read-bandwidth microbenchmarks on the B200 (not part of the product):
//  ldg   : LDG.128 streaming loads, UNROLL loads in flight per thread
//  ring  : warp-specialised cp.async.bulk ring, consumers only release slots
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2506_04710_b200/csrc bwtest.cu -o bwtest
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace tbt;

template <int UNROLL>
__global__ void ldgRead(const double2* __restrict__ p, long long n, double* out) {
  double acc = 0;
  long long stride = (long long)gridDim.x * blockDim.x * UNROLL;
  for (long long i = (long long)blockIdx.x * blockDim.x * UNROLL + threadIdx.x; i < n; i += stride) {
    double2 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      long long k = i + (long long)u * blockDim.x;
      v[u] = k < n ? __ldcs(p + k) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += v[u].x + v[u].y;
  }
  if (acc == 1234.5) out[0] = acc;
}

template <int STAGES>
__global__ void __launch_bounds__(288, 1) ringRead(const char* __restrict__ src, long long nchunks, uint32_t chunk,
                                                   double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * chunk);
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
      uint64_t pol = policyEvictFirst();
      for (long long it = 0; it < mine; ++it) {
        int s = it % STAGES; uint32_t ph = (it / STAGES) & 1;
        mbarWait(empty + s, ph ^ 1u);
        mbarArriveExpectTx(full + s, chunk);
        bulkG2S(smem + s * chunk, src + (blockIdx.x + it * gridDim.x) * (long long)chunk, chunk, full + s, pol);
      }
    }
    return;
  }
  double acc = 0;
  for (long long it = 0; it < mine; ++it) {
    int s = it % STAGES; uint32_t ph = (it / STAGES) & 1;
    mbarWait(full + s, ph);
    acc += reinterpret_cast<const double*>(smem + s * chunk)[threadIdx.x];
    __syncwarp();
    if (lane == 0) mbarArrive(empty + s);
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  const long long bytes = 1LL << 30;
  char* buf; double* out;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 8);
  cudaMemset(buf, 0, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](auto launch, const char* name, long long nbytes) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(a);
    const int R = 10;
    for (int r = 0; r < R; ++r) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %8.1f GB/s  (%.2f us per pass)\n", name, nbytes / (ms / R * 1e-3) / 1e9, ms / R * 1e3);
  };
  for (long long nb : {134LL << 20, 1LL << 30}) {
    printf("--- %lld MiB read\n", nb >> 20);
    long long n4 = nb / 16;
    for (int bpsm : {2, 4, 8}) {
      char nm[64]; snprintf(nm, 64, "ldg u4 256t x %d/SM", bpsm);
      timeit([&] { ldgRead<4><<<sms * bpsm, 256>>>((const double2*)buf, n4, out); }, nm, nb);
      snprintf(nm, 64, "ldg u8 256t x %d/SM", bpsm);
      timeit([&] { ldgRead<8><<<sms * bpsm, 256>>>((const double2*)buf, n4, out); }, nm, nb);
    }
    for (uint32_t chunk : {16384u, 32768u, 65536u}) {
      for (int st : {2, 3, 4, 6}) {
        size_t sm = st * (size_t)chunk + 2 * st * 8;
        if (sm > 227 * 1024) continue;
        long long nch = nb / chunk;
        char nm[64]; snprintf(nm, 64, "ring chunk %uK x %d stages", chunk >> 10, st);
        if (st == 2) { cudaFuncSetAttribute(ringRead<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
          timeit([&] { ringRead<2><<<sms, 288, sm>>>(buf, nch, chunk, out); }, nm, nb); }
        if (st == 3) { cudaFuncSetAttribute(ringRead<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
          timeit([&] { ringRead<3><<<sms, 288, sm>>>(buf, nch, chunk, out); }, nm, nb); }
        if (st == 4) { cudaFuncSetAttribute(ringRead<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
          timeit([&] { ringRead<4><<<sms, 288, sm>>>(buf, nch, chunk, out); }, nm, nb); }
        if (st == 6) { cudaFuncSetAttribute(ringRead<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
          timeit([&] { ringRead<6><<<sms, 288, sm>>>(buf, nch, chunk, out); }, nm, nb); }
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
