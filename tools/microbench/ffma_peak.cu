// FP32 FMA issue-rate microbenchmark for sm_100a (B200).
// Measures the FMA/clk/SM that register-only FFMA / FFMA2 (fma.rn.f32x2) loops reach,
// in the outer-product operand pattern the aggregation kernel uses
// (acc[p][d] += w[p] * c[d]). The result is the "alu" roofline denominator in DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>

#define NP 8
#define ND 4

__device__ __forceinline__ void ffma2(float2& acc, float2 a, float2 b) {
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long B = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long C = *reinterpret_cast<unsigned long long*>(&acc);
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
  acc = *reinterpret_cast<float2*>(&C);
}

// variant 0: scalar FFMA outer product NP x ND (32 accumulators)
__global__ void k_ffma(float* out, int iters, float seed) {
  float w[NP], c[ND], acc[NP][ND];
  for (int i = 0; i < NP; ++i) w[i] = seed * (threadIdx.x + i);
  for (int j = 0; j < ND; ++j) c[j] = seed * (threadIdx.x - j);
  for (int i = 0; i < NP; ++i) for (int j = 0; j < ND; ++j) acc[i][j] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
      for (int j = 0; j < ND; ++j) acc[i][j] = fmaf(w[i], c[j], acc[i][j]);
#pragma unroll
    for (int i = 0; i < NP; ++i) w[i] = __int_as_float(__float_as_int(w[i]) ^ 1);
  }
  float s = 0.f;
  for (int i = 0; i < NP; ++i) for (int j = 0; j < ND; ++j) s += acc[i][j];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

// variant 1: FFMA2, acc pairs over d: (p,d),(p,d+1) += (w,w)*(c_d,c_d+1)
__global__ void k_ffma2_dup(float* out, int iters, float seed) {
  float2 w[NP], c[ND / 2], acc[NP][ND / 2];
  for (int i = 0; i < NP; ++i) { float t = seed * (threadIdx.x + i); w[i] = make_float2(t, t); }
  for (int j = 0; j < ND / 2; ++j) c[j] = make_float2(seed * threadIdx.x, seed * j);
  for (int i = 0; i < NP; ++i) for (int j = 0; j < ND / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
      for (int j = 0; j < ND / 2; ++j) ffma2(acc[i][j], w[i], c[j]);
#pragma unroll
    for (int i = 0; i < NP; ++i) { w[i].x = __int_as_float(__float_as_int(w[i].x) ^ 1); w[i].y = w[i].x; }
  }
  float s = 0.f;
  for (int i = 0; i < NP; ++i) for (int j = 0; j < ND / 2; ++j) s += acc[i][j].x + acc[i][j].y;
  if (s == 1.2345f) out[threadIdx.x] = s;
}

// variant 2: FFMA2 without the per-iteration weight rewrite (pure issue ceiling)
__global__ void k_ffma2_pure(float* out, int iters, float seed) {
  float2 w[NP], c[ND / 2], acc[NP][ND / 2];
  for (int i = 0; i < NP; ++i) { float t = seed * (threadIdx.x + i); w[i] = make_float2(t, t + 1.f); }
  for (int j = 0; j < ND / 2; ++j) c[j] = make_float2(seed * threadIdx.x, seed * j);
  for (int i = 0; i < NP; ++i) for (int j = 0; j < ND / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
      for (int j = 0; j < ND / 2; ++j) ffma2(acc[i][j], w[i], c[j]);
  }
  float s = 0.f;
  for (int i = 0; i < NP; ++i) for (int j = 0; j < ND / 2; ++j) s += acc[i][j].x + acc[i][j].y;
  if (s == 1.2345f) out[threadIdx.x] = s;
}

// variant 3: scalar FFMA without weight rewrite
__global__ void k_ffma_pure(float* out, int iters, float seed) {
  float w[NP], c[ND], acc[NP][ND];
  for (int i = 0; i < NP; ++i) w[i] = seed * (threadIdx.x + i);
  for (int j = 0; j < ND; ++j) c[j] = seed * (threadIdx.x - j);
  for (int i = 0; i < NP; ++i) for (int j = 0; j < ND; ++j) acc[i][j] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
      for (int j = 0; j < ND; ++j) acc[i][j] = fmaf(w[i], c[j], acc[i][j]);
  }
  float s = 0.f;
  for (int i = 0; i < NP; ++i) for (int j = 0; j < ND; ++j) s += acc[i][j];
  if (s == 1.2345f) out[threadIdx.x] = s;
}


__device__ __forceinline__ void ffma2s(float2& acc, float a, float2 b) {
  unsigned long long A, B = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long C = *reinterpret_cast<unsigned long long*>(&acc);
  asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
  acc = *reinterpret_cast<float2*>(&C);
}

// variant 4: FFMA2 with a scalar (broadcast) weight operand: (p,d),(p,d+1) += w_p * (c_d, c_d+1)
__global__ void k_ffma2_bcast(float* out, int iters, float seed) {
  float w[NP]; float2 c[ND / 2], acc[NP][ND / 2];
  for (int i = 0; i < NP; ++i) w[i] = seed * (threadIdx.x + i);
  for (int j = 0; j < ND / 2; ++j) c[j] = make_float2(seed * threadIdx.x, seed * j);
  for (int i = 0; i < NP; ++i) for (int j = 0; j < ND / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
      for (int j = 0; j < ND / 2; ++j) ffma2s(acc[i][j], w[i], c[j]);
  }
  float s = 0.f;
  for (int i = 0; i < NP; ++i) for (int j = 0; j < ND / 2; ++j) s += acc[i][j].x + acc[i][j].y;
  if (s == 1.2345f) out[threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K kern, int blocks, int threads, int iters, double fma_per_thread_iter) {
  float* out; cudaMalloc(&out, 4096);
  kern<<<blocks, threads>>>(out, 10, 1e-7f);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(out, iters, 1e-7f);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  double fmas = (double)blocks * threads * iters * fma_per_thread_iter;
  int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double tflops = 2 * fmas / (best * 1e-3) / 1e12;
  double per_clk_sm = fmas / (best * 1e-3) / (clk * 1e3) / sms;
  printf("%-14s blocks=%d thr=%d  %.3f ms  %.2f TFLOP/s  %.1f FMA/clk/SM (at attr clock %d MHz, %d SMs)\n",
         name, blocks, threads, best, tflops, per_clk_sm, clk / 1000, sms);
  cudaFree(out);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 20000;
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (1024 / tpb);
    run("ffma", k_ffma, blocks, tpb, iters, NP * ND);
    run("ffma_pure", k_ffma_pure, blocks, tpb, iters, NP * ND);
    run("ffma2_dup", k_ffma2_dup, blocks, tpb, iters, NP * ND);
    run("ffma2_pure", k_ffma2_pure, blocks, tpb, iters, NP * ND);
    run("ffma2_bcast", k_ffma2_bcast, blocks, tpb, iters, NP * ND);
  }
  return 0;
}
