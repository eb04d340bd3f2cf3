// Shared-memory wavefronts per warp-wide load for the address patterns the
// aggregation stream uses (read with ncu l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld):
//   mode 0: LDS.128, one address for the whole warp
//   mode 1: LDS.128, one address per half-warp (two distinct)
//   mode 2: LDS.64,  one address for the whole warp
//   mode 3: LDS.64,  one address per half-warp
//   mode 4: LDS.32,  one address per half-warp
//   mode 5: LDS.128, one address per quarter-warp (four distinct, disjoint banks)
//   mode 6: LDS.128, one address per quarter-warp (four distinct, same banks)
//   mode 7: LDS.128, one address per eighth-warp (eight distinct, disjoint banks)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_wavefronts lds_wavefronts.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_lds(float* out, int iters) {
  __shared__ __align__(16) float s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = (float)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const int base = (it * 8) & 2047;
    if (MODE == 0) { float4 v = *reinterpret_cast<float4*>(&s[base]); acc += v.x + v.y + v.z + v.w; }
    if (MODE == 1) { float4 v = *reinterpret_cast<float4*>(&s[base + 4 * half + 32 * half]); acc += v.x + v.y + v.z + v.w; }
    if (MODE == 2) { float2 v = *reinterpret_cast<float2*>(&s[base]); acc += v.x + v.y; }
    if (MODE == 3) { float2 v = *reinterpret_cast<float2*>(&s[base + 2 * half + 32 * half]); acc += v.x + v.y; }
    if (MODE == 4) { acc += s[base + half * 33]; }
    if (MODE == 5) { float4 v = *reinterpret_cast<float4*>(&s[base + 4 * (lane >> 3)]); acc += v.x + v.y + v.z + v.w; }
    if (MODE == 6) { float4 v = *reinterpret_cast<float4*>(&s[base + 32 * (lane >> 3)]); acc += v.x + v.y + v.z + v.w; }
    if (MODE == 7) { float4 v = *reinterpret_cast<float4*>(&s[base + 4 * (lane >> 2)]); acc += v.x + v.y + v.z + v.w; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 256 * sizeof(float));
  k_lds<0><<<148, 256>>>(out, 1024);
  k_lds<1><<<148, 256>>>(out, 1024);
  k_lds<2><<<148, 256>>>(out, 1024);
  k_lds<3><<<148, 256>>>(out, 1024);
  k_lds<4><<<148, 256>>>(out, 1024);
  k_lds<5><<<148, 256>>>(out, 1024);
  k_lds<6><<<148, 256>>>(out, 1024);
  k_lds<7><<<148, 256>>>(out, 1024);
  printf("done %d\n", (int)cudaDeviceSynchronize());
  return 0;
}
