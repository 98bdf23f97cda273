// FP64 throughput on the B200: DFMA (vector) vs mma.sync.m8n8k4.f64 (DMMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64test.cu -o fp64test
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma(double* out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma(double* out, int iters) {
  double acc[4][2];
  double af = 1.0 + threadIdx.x * 1e-6, bf = 0.5;
#pragma unroll
  for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[k][0]), "+d"(acc[k][1])
                   : "d"(af), "d"(bf));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1];
  if (s == 12345.678) out[0] = s;
}

// Larger FP64 MMA shapes (sm_90+): m16n8k4 / m16n8k8 / m16n8k16.
template <int K>
__global__ void dmma16(double* out, int iters) {
  double acc[4][4];
  double af[K / 2], bf[K / 4];
#pragma unroll
  for (int k = 0; k < K / 2; ++k) af[k] = 1.0 + threadIdx.x * 1e-6 + k;
#pragma unroll
  for (int k = 0; k < K / 4; ++k) bf[k] = 0.5 + k;
#pragma unroll
  for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if constexpr (K == 4)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(acc[k][0]), "+d"(acc[k][1]), "+d"(acc[k][2]), "+d"(acc[k][3])
                     : "d"(af[0]), "d"(af[1]), "d"(bf[0]));
      else if constexpr (K == 8)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(acc[k][0]), "+d"(acc[k][1]), "+d"(acc[k][2]), "+d"(acc[k][3])
                     : "d"(af[0]), "d"(af[1]), "d"(af[2]), "d"(af[3]), "d"(bf[0]), "d"(bf[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                     "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(acc[k][0]), "+d"(acc[k][1]), "+d"(acc[k][2]), "+d"(acc[k][3])
                     : "d"(af[0]), "d"(af[1]), "d"(af[2]), "d"(af[3]), "d"(af[4]), "d"(af[5]), "d"(af[6]),
                       "d"(af[7]), "d"(bf[0]), "d"(bf[1]), "d"(bf[2]), "d"(bf[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1] + acc[k][2] + acc[k][3];
  if (s == 12345.678) out[0] = s;
}


// DMMA stream with NADD DADDs per 42 DMMAs feeding its B operands (the 3M
// complex product forms Ar+Ai / Br+Bi sums on the same FP64 pipe): what an
// interleaved DADD costs in DMMA slots. TF/s counts the DMMAs only.
template <int NADD>
__global__ void __launch_bounds__(256, 1) dmmaMix(double* out, int iters) {
  double acc[42][2];
  double af = 1.0 + threadIdx.x * 1e-6, bf[7], c = 1e-9 * threadIdx.x;
#pragma unroll
  for (int k = 0; k < 7; ++k) bf[k] = 0.5 + k;
#pragma unroll
  for (int k = 0; k < 42; ++k) acc[k][0] = acc[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 42; ++k) {
      if (NADD > 0 && k % 6 == 0 && k / 6 < NADD)
        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(bf[k / 6]) : "d"(c));
      if (NADD > 7 && k % 6 == 3 && k / 6 < NADD - 7)
        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(af) : "d"(c));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[k][0]), "+d"(acc[k][1])
                   : "d"(af), "d"(bf[k / 6]));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 42; ++k) s += acc[k][0] + acc[k][1];
  if (s == 12345.678) out[0] = s;
}

template <int NADD>
void runMix(double* out, int sms, int iters, cudaEvent_t a, cudaEvent_t b) {
  dim3 g(sms), t(256);
  dmmaMix<NADD><<<g, t>>>(out, 100);
  cudaEventRecord(a);
  dmmaMix<NADD><<<g, t>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * 256 * 42 * iters * (double)g.x * (t.x / 32);
  printf("DMMA x42 + %2d DADD per iteration, 8 warps/SM: %.1f TFLOP/s (DMMA only)\n", NADD, flops / (ms * 1e-3) / 1e12);
}


// DMMA issue rate against warps per SM sub-partition: NACC independent
// accumulators per warp, CTAs of `threads` threads, one CTA per SM.
template <int NACC>
__global__ void dmmaWarps(double* out, int iters) {
  double acc[NACC][2];
  double af = 1.0 + threadIdx.x * 1e-6, bf = 0.5;
#pragma unroll
  for (int k = 0; k < NACC; ++k) acc[k][0] = acc[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NACC; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[k][0]), "+d"(acc[k][1])
                   : "d"(af), "d"(bf));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < NACC; ++k) s += acc[k][0] + acc[k][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
void runWarps(double* out, int sms, int threads, int iters, cudaEvent_t a, cudaEvent_t b) {
  dim3 g(sms), t(threads);
  dmmaWarps<NACC><<<g, t>>>(out, 100);
  cudaEventRecord(a);
  dmmaWarps<NACC><<<g, t>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * 256 * NACC * iters * (double)g.x * (t.x / 32);
  printf("DMMA %2d independent accumulators, %2d warps/SM: %.1f TFLOP/s\n", NACC, threads / 32, flops / (ms * 1e-3) / 1e12);
}

template <int K>
void runDmma16(double* out, int sms, int bpsm, int iters, cudaEvent_t a, cudaEvent_t b) {
  dim3 g(sms * bpsm), t(256);
  dmma16<K><<<g, t>>>(out, 100);
  cudaEventRecord(a);
  dmma16<K><<<g, t>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * 16 * 8 * K * 4 * iters * (double)g.x * (t.x / 32);
  printf("DMMA m16n8k%-2d %d CTA/SM: %.1f TFLOP/s\n", K, bpsm, flops / (ms * 1e-3) / 1e12);
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int bpsm : {1, 2, 4, 8}) {
    dim3 g(sms * bpsm), t(256);
    dfma<<<g, t>>>(out, 100);
    cudaEventRecord(a);
    dfma<<<g, t>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * iters * (double)g.x * t.x;
    printf("DFMA  %d CTA/SM: %.1f TFLOP/s\n", bpsm, flops / (ms * 1e-3) / 1e12);
    dmma<<<g, t>>>(out, 100);
    cudaEventRecord(a);
    dmma<<<g, t>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    flops = 2.0 * 256 * 4 * iters * (double)g.x * (t.x / 32);
    printf("DMMA  %d CTA/SM: %.1f TFLOP/s\n", bpsm, flops / (ms * 1e-3) / 1e12);
    runDmma16<4>(out, sms, bpsm, iters / 2, a, b);
    runDmma16<8>(out, sms, bpsm, iters / 4, a, b);
    runDmma16<16>(out, sms, bpsm, iters / 8, a, b);
  }
  for (int th : {128, 256, 384, 512, 1024}) runWarps<1>(out, sms, th, 40000, a, b);
  for (int th : {128, 256, 384, 512, 1024}) runWarps<2>(out, sms, th, 20000, a, b);
  for (int th : {128, 256, 384, 512, 1024}) runWarps<8>(out, sms, th, 10000, a, b);
  runMix<0>(out, sms, 4000, a, b);
  runMix<3>(out, sms, 4000, a, b);
  runMix<7>(out, sms, 4000, a, b);
  runMix<9>(out, sms, 4000, a, b);
  runMix<14>(out, sms, 4000, a, b);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
