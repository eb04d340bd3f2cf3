// Ceiling of the walker's FMA stream (fbs::RingRows<4>) from the shared-memory
// cost ring, as a function of the number of stream warps per SM (one CTA per SM,
// NWARP warps, all streaming; no cost phase, no prologue, no WTA).  Tells whether
// one stream warp per scheduler can keep the FFMA2 pipe busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ring_stream ring_stream.cu -lcuda
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_1807_02044_b200/csrc/fbs_fused.cuh"
using namespace fbs;

template <int R, int NWARP, int HPY>
__global__ void __launch_bounds__(NWARP * 32, 1) k_ring(int reps, float* out) {
  using G = WGeo<R>;
  constexpr int K1 = 2 * R + 1;
  constexpr int RS = K1 * K1 * kPX;
  extern __shared__ __align__(128) float sm[];
  float* ring = sm;                                 // [SR][SC][64]
  float* w = sm + G::SR * G::SC * kDB;              // [NWARP][PY][K1][K1][4]
  const int nring = G::SR * G::SC * kDB, nw = (NWARP < 8 ? NWARP : 8) * G::WPW + 4;
  for (int i = threadIdx.x; i < nring + nw; i += blockDim.x) sm[i] = 1e-3f * (i % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane >> 4, dq = lane & 15;
  const int wx = (warp % 4) * kPX, wy = ((warp / 4) % 2) * G::PY;
  const float* col = ring + wx * kDB + 4 * dq;
  const float* wsm0 = w + (warp % 8) * G::WPW + half * HPY * RS;
  float acc = 0.f;
  for (int it = 0; it < reps; ++it) {
    float2 num[HPY][kPX][2];
#pragma unroll
    for (int py = 0; py < HPY; ++py)
#pragma unroll
      for (int px = 0; px < kPX; ++px) num[py][px][0] = num[py][px][1] = make_float2(0.f, 0.f);
    const int base = (wy + half * HPY + it) % G::SR;
    const float* wsm = wsm0 + (it & 1) * 4;  // not loop-invariant (no hoisting)
    float4 head[kPX];
#pragma unroll
    for (int j = 0; j < kPX; ++j) head[j] = *reinterpret_cast<const float4*>(col + base * G::SC * kDB + j * kDB);
    RingRows<G, 0, HPY + 2 * R, HPY>::run(col, base, wsm, head, num);
#pragma unroll
    for (int py = 0; py < HPY; ++py)
#pragma unroll
      for (int px = 0; px < kPX; ++px) acc += num[py][px][0].x + num[py][px][1].y;
  }
  if (acc == 1.2345f) out[threadIdx.x] = acc;
}

template <int NWARP, int HPY = 3>
static void run() {
  constexpr int R = 4;
  using G = WGeo<R>;
  const size_t smem = (size_t)(G::SR * G::SC * kDB + (NWARP < 8 ? NWARP : 8) * G::WPW + 4) * 4;
  float* out;
  cudaMalloc(&out, 4096);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_ring<R, NWARP, HPY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int reps = 400;
  k_ring<R, NWARP, HPY><<<sms, NWARP * 32, smem>>>(4, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int t = 0; t < 5; ++t) {
    cudaEventRecord(a);
    k_ring<R, NWARP, HPY><<<sms, NWARP * 32, smem>>>(reps, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double ffma2 = (double)sms * NWARP * reps * HPY * kPX * 2 * 81;  // per warp: 2 halves share the count
  const double flops = ffma2 * 32 * 2 * 2;
  printf("R=4 HPY=%d warps/SM=%2d smem=%zu B: %.3f ms, %.1f TFLOP/s, %.2f FFMA2/clk/SM (at 1.965 GHz) err=%s\n", HPY, NWARP,
         smem, best, flops / best / 1e9, ffma2 / sms / (best * 1e-3 * 1.965e9),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<4>();
  run<8>();
  run<12>();
  run<16>();
  run<8, 2>();
  run<12, 2>();
  run<16, 2>();
  run<8, 1>();
  run<16, 1>();
  return 0;
}
