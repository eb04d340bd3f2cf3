// fbs_kernels.cuh — shared device pieces of the sm_100a fast bilateral stereo
// (FBS) hot path (PAPER.md, arXiv 1807.02044; "P:Lnn" = PAPER.md line).  The
// kernels of the production path are in fbs_fused.cuh:
//   k_prep    block statistics (Eq.(2)(3), "pre-calculated" P:L84)
//   k_fbs     twin NCC costs (Eq.(1)) computed into shared memory and
//             bilateral aggregation (Eq.(6)-(8)) + WTA
//   k_final   LRC (Eq.(9), left reference P:L203) + parabola
//             subpixel (Eq.(10))
// This file: constants, the FFMA2 row kernel of the aggregation stream, the WTA
// butterfly, the LRC/subpixel rule and the debug select path.
//
// Design notes (DESIGN.md §6 has the rationale and the rooflines):
//  * NCC in exact integer arithmetic: N = 9·Σ i_l i_r − S_l S_r and V = 9·Σ i² − S²
//    are integers < 2^24; c = N · (V_l^{-1/2} · V_r^{-1/2}) in fp32 (algebraically
//    identical to Eq.(1)-(3); R#5).  The 3x3 dot product is three DP4A on
//    packed 3-pixel columns.
//  * Aggregation: each lane holds 4 disparities (2 FFMA2 pairs) of a 64-disparity
//    block; the two half-warps take the upper and lower halves of the warp's
//    pixel sub-tile.  One FFMA2 per (output pixel, tap, disparity pair) with the
//    warp-uniform weight w(p,q) = ω_d ω_r as a broadcast scalar operand (SASS:
//    FFMA2 R, Rw.F32, Rc.F32x2).
//  * Undefined costs are stored as -0.0 and drop out of the numerator; the
//    d-independent validity (border / textureless block of the guide's own image)
//    is folded into the weights, and per (warp sub-tile, d-block) the denominator
//    takes one exact form (FAST / EDGE / GENERAL / EMPTY, see k_fbs).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fbs {

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in
// the stream finishes; pdl_wait() blocks until that predecessor has completed
// and its memory is visible, pdl_trigger() lets the successor launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

constexpr float kSent = -2.0f;   // undefined aggregated cost / exported cost (R#7)
constexpr float kUndef = -0.0f;  // undefined cost in the cost ring (never a defined NCC value)
constexpr int kMaxRadius = 10;   // FBS_MAX_RADIUS (volume path)
constexpr int kFusedMaxRadius = 6;  // the fused path's largest radius
constexpr int kWsMaxRadius = 4;  // radii run by the warp-specialised walker (fbs_ws.cuh)
// Smallest tap weight the handle accepts, as -log2 (FBS_MAX_WEIGHT_EXP2, R#13):
// 2^-124 stays a normal fp32 after ex2.approx.ftz and any rounding of the exponent.
constexpr double kMaxWeightExp2 = 124.0;
constexpr int kDB = 64;          // disparities per block (16 lanes x 4)
constexpr int kPX = 4;           // warp sub-tile width  (pixels)
constexpr int kTYMax = 12;       // tallest walker step of any radius

// Padded guide images (written by k_prep): i(q) as a float, with an R-pixel
// margin of kGuideUndef outside the frame.  A pixel whose own block is
// undefined stores i + kGuideFlag: as a tap q it is >= 2^23 - 255 away from any
// intensity, so its weight 2^(nkr Δ² + cd) flushes to exactly +0 (nkr <= -2e-12,
// see fbs_create), and as a centre p its intensity is recovered exactly (i + 2^23
// is exact in fp32).
constexpr float kGuideUndef = 1e30f;
constexpr float kGuideFlag = 8388608.0f;
__host__ __device__ constexpr int guide_pitch(int W, int R) { return ((W + 15) / 16 * 16 + 2 * R + 4 + 3) / 4 * 4; }
__host__ __device__ constexpr int guide_rows(int H, int R) { return (H + kTYMax - 1) / kTYMax * kTYMax + kTYMax + 2 * R; }

// fill a buffer with a float value (guide margins = kGuideUndef)
__global__ void k_fill(float* p, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// Band scatter (fbs_compute_rows_scatter): the final map of the band's rows is
// stored into every buffer of the set — full [H][W] frames, e.g. the peers'
// symmetric-memory buffers mapped into this GPU (NVLink P2P stores) — instead
// of the band-relative output; n = 0: the usual output.
constexpr int kMaxScatter = 8;
struct OutSet {
  float* p[kMaxScatter];
  int n;
};

// ---------------------------------------------------------------------------
// Stage 4: Eq.(9) LRC (tolerance 1, R#17) then Eq.(10) subpixel on aggregated
// costs (R#19, R#21).  d_int: left WTA disparity or -1; e: d_R(u - d_int, v) or -1.
__device__ __forceinline__ float finalize_pixel(int d_int, int e, float c0, float cm, float cp,
                                                int d_min, int d_max) {
  if (d_int < 0 || e < 0) return -1.0f;
  if (abs(d_int - e) > 1) return -1.0f;
  float ds = (float)d_int;
  if (d_int > d_min && d_int < d_max && cm != kSent && cp != kSent) {
    const float den = __fsub_rn(__fadd_rn(2.0f * cm, 2.0f * cp), 4.0f * c0);
    if (fabsf(den) >= 1e-9f) {
      float delta = __fdiv_rn(__fsub_rn(cm, cp), den);
      delta = fminf(0.5f, fmaxf(-0.5f, delta));
      ds = __fadd_rn(ds, delta);
    }
  }
  return ds;
}

// ---------------------------------------------------------------------------
// Bilateral aggregation building blocks.
//
// Undefined costs are stored as -0.0f (a defined NCC is never -0.0: N = 0 gives
// +0.0), so they add nothing to the numerator Σ w c whatever their weight; the
// denominator Σ w over the defined taps is the only place validity enters.
// Per (warp sub-tile, d-block) the denominator takes one of four exact forms:
//   FAST     every tap defined but for the guide's own blocks (folded into w'):
//            den = Σ_q w'(p,q), d-independent
//   EDGE     additionally only the frame edge cuts taps off (x - d < 1 on the
//            left pass, x + d > W-2 on the right): den = a per-pixel suffix /
//            prefix sum of the window's column sums, indexed by d
//   GENERAL  the other image has textureless blocks in range: explicit den by
//            FFMA2 over the validity of every tap
//   EMPTY    (special case of GENERAL) no block of the other image in range is
//            defined: every aggregated cost is SENT, no arithmetic
// Sub-tiles are anchored at multiples of their size in frame coordinates, so
// the form a pixel gets never depends on the row band being computed.
enum { kFast = 0, kEdge = 1, kGeneral = 2, kEmpty = 3 };


__device__ __forceinline__ void ffma2(float2& acc, float w, float2 c) {
  unsigned long long A, B = *reinterpret_cast<unsigned long long*>(&c);
  unsigned long long C = *reinterpret_cast<unsigned long long*>(&acc);
  asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(w));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
  acc = *reinterpret_cast<float2*>(&C);
}

__device__ __forceinline__ bool is_undef(float c) { return __float_as_uint(c) == 0x80000000u; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// 1/x for x > 0: MUFU reciprocal + one Newton step (<= 1 ulp; no slow path)
__device__ __forceinline__ float rcp_nr(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return __fmul_rn(r, __fmaf_rn(-x, r, 2.0f));
}

// Order-preserving map float -> u32 (larger float <=> larger key).
__device__ __forceinline__ unsigned fkey(float v) {
  const unsigned b = __float_as_uint(v);
  return b ^ ((unsigned)((int)b >> 31) | 0x80000000u);
}
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}
__device__ __forceinline__ unsigned long long shfl_xor64(unsigned long long v, int m) {
  const unsigned lo = __shfl_xor_sync(0xffffffffu, (unsigned)v, m);
  const unsigned hi = __shfl_xor_sync(0xffffffffu, (unsigned)(v >> 32), m);
  return ((unsigned long long)hi << 32) | lo;
}

// ---- 4 disparities per lane: lanes 0-15 and 16-31 (half-warps) take the
// upper and lower 4 x HPY halves of the warp's sub-tile; every broadcast
// weight load then feeds 2 FFMA2 per pixel (halving the L1 wavefronts per FMA).

// num[pyl][px][pair] += Σ_dx w(pyl, r - pyl, dx, px) · c[px + dx]  for cost row r
template <int R, int NPY, int r>
__device__ __forceinline__ void row_fma4(const float4* c, const float* __restrict__ wsm,
                                         float2 (&num)[NPY][kPX][2]) {
  constexpr int K1 = 2 * R + 1;
#pragma unroll
  for (int dx = 0; dx < K1; ++dx) {
#pragma unroll
    for (int pyl = 0; pyl < NPY; ++pyl) {
      const int dy = r - pyl;
      if (dy >= 0 && dy <= 2 * R) {
        const float4 w = reinterpret_cast<const float4*>(wsm + (pyl * K1 + dy) * K1 * kPX)[dx];
        const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int px = 0; px < kPX; ++px) {
          const float4 cc = c[dx + px];
          ffma2(num[pyl][px][0], wv[px], make_float2(cc.x, cc.y));
          ffma2(num[pyl][px][1], wv[px], make_float2(cc.z, cc.w));
        }
      }
    }
  }
}

// Argmax of each half-warp's 16 pixel slots (k[s] = this lane's best key of slot
// s): a transposing butterfly within the half-warp, 8+4+2+1 = 15 u64 shuffles;
// afterwards lane l holds slot l & 15 of its half.
__device__ __forceinline__ unsigned long long wta_butterfly16(unsigned long long (&k)[16], int lane) {
#pragma unroll
  for (int lvl = 0; lvl < 4; ++lvl) {
    const int n = 8 >> lvl;
    const bool up = lane & n;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const unsigned long long keep = up ? k[n + i] : k[i];
      const unsigned long long send = up ? k[i] : k[n + i];
      k[i] = umax64(keep, shfl_xor64(send, n));
    }
  }
  return k[0];
}

// The same for 8 slots (2 x 4 pixels per half-warp): the transposing butterfly
// within each group of 8 lanes, then the two groups of a half combined
// (4+2+1+1 = 8 u64 shuffles); afterwards lanes l and l ^ 8 hold slot l & 7.
__device__ __forceinline__ unsigned long long wta_butterfly8(unsigned long long (&k)[8], int lane) {
#pragma unroll
  for (int lvl = 0; lvl < 3; ++lvl) {
    const int n = 4 >> lvl;
    const bool up = lane & n;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const unsigned long long keep = up ? k[n + i] : k[i];
      const unsigned long long send = up ? k[i] : k[n + i];
      k[i] = umax64(keep, shfl_xor64(send, n));
    }
  }
  return umax64(k[0], shfl_xor64(k[0], 8));
}

// ---------------------------------------------------------------------------
// Debug select path: WTA over a given [H][W][D] volume (same rules as k_fbs:
// highest value, smallest d on ties, all-SENT -> -1); for the left volume also
// the record (c(d*-1), c(d*), c(d*+1)) k_final reads.
__global__ void k_select_wta(const float* __restrict__ agg, int W, int H, int D, int d_min,
                             int32_t* __restrict__ disp, float4* __restrict__ agg3) {
  const size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (p >= (size_t)W * H) return;
  const float* col = agg + p * D;
  float best = -INFINITY;
  int bi = 0;
  for (int k = 0; k < D; ++k) {
    const float v = col[k];
    if (v > best) { best = v; bi = k; }
  }
  disp[p] = best > kSent ? d_min + bi : -1;
  if (agg3) agg3[p] = make_float4(bi > 0 ? col[bi - 1] : kSent, col[bi], bi + 1 < D ? col[bi + 1] : kSent, 0.f);
}

}  // namespace fbs
