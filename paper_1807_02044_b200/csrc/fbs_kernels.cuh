// fbs_kernels.cuh — sm_100a kernels of the fast bilateral stereo (FBS) hot path.
//
// Stages (PAPER.md, arXiv 1807.02044; "P:Lnn" = PAPER.md line):
//   k_stats      block statistics once per image          Eq.(2)(3)
//   k_cost       twin NCC cost volumes                     Eq.(1)
//   k_agg        bilateral aggregation + WTA (+ LRC +      Eq.(6)-(8) P:L118-132, P:L199,
//                subpixel epilogue on the left pass)       P:L201, Eq.(9)(10)
//   k_select_*   WTA/LRC/subpixel from given volumes (debug / parity only)
//
// Design notes (DESIGN.md §6 has the full rationale and rooflines):
//  * NCC is evaluated in exact integer arithmetic: N = 9·Σ i_l i_r − S_l S_r and
//    V = 9·Σ i² − S² are integers < 2^24, c = N · V_l^{-1/2} · V_r^{-1/2} in fp32
//    (algebraically identical to Eq.(1)-(3); R#5).  The 3x3 dot product
//    is three DP4A on packed rows.
//  * Aggregation: lanes <-> disparity pairs (32 lanes x 2 d = 64 d per warp), one
//    FFMA2 per (output pixel, tap) with the warp-uniform bilateral weight
//    w(p,q) = ω_d ω_r as a broadcast scalar operand (SASS: FFMA2 R, Rw.F32, Rc.F32x2).
//    Weights are d-independent: computed once per pixel window into shared memory
//    and reused across every disparity block ("pre-calculated").
//  * d-independent validity (border / textureless block of the guide's own image)
//    is folded into the weights; the d-dependent part (the other image's block at
//    x∓d) only matters near the left/right frame edge and textureless regions,
//    detected per (CTA tile, d-block) and handled by an exact slow path with an
//    explicit denominator.  Both paths produce bit-identical results.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fbs {

constexpr float kSent = -2.0f;   // undefined cost / aggregated cost (R#7)
constexpr int kMaxRadius = 6;    // FBS_MAX_RADIUS
constexpr int kDB = 64;          // disparities per warp block (32 lanes x 2)
constexpr int kPX = 4;           // warp sub-tile width  (pixels)
constexpr int kPY = 8;           // warp sub-tile height (pixels)
constexpr int kNWX = 4;          // warps across a CTA tile
constexpr int kNWY = 2;          // warps down a CTA tile
constexpr int kTX = kPX * kNWX;  // CTA tile 16 x 16
constexpr int kTY = kPY * kNWY;
constexpr int kThreads = 32 * kNWX * kNWY;
constexpr int kTStride = 68;     // WTA transpose row stride (floats): 16B aligned, conflict-free

// ---------------------------------------------------------------------------
// Stage 1: block statistics.  For each pixel of rows [r0, r1):
//   P  = i(x-1) | i(x)<<8 | i(x+1)<<16   (packed row, DP4A operand)
//   S  = Σ i over the 3x3 block, V = 9 Σ i² − S²   (Eq.(2)(3) x 81, exact integers)
//   def = interior && V > 0   (σ >= σ_floor; textureless => NCC undefined, R#7)
//   rs = V^{-1/2} (IEEE sqrt, IEEE division), 0 when !def
__global__ void k_stats(const uint8_t* __restrict__ img, int W, int H, int r0, int r1,
                        uint32_t* __restrict__ P, int32_t* __restrict__ S,
                        float* __restrict__ rs, uint8_t* __restrict__ def) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = r0 + blockIdx.y;
  if (x >= W || y >= r1) return;
  const size_t i = (size_t)y * W + x;
  uint32_t pk = 0;
  if (x >= 1 && x <= W - 2)
    pk = (uint32_t)img[i - 1] | ((uint32_t)img[i] << 8) | ((uint32_t)img[i + 1] << 16);
  P[i] = pk;
  int s = 0, q = 0, ok = 0;
  if (x >= 1 && x <= W - 2 && y >= 1 && y <= H - 2) {
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int v = img[(size_t)(y + dy) * W + (x + dx)];
        s += v;
        q += v * v;
      }
    ok = (9 * q - s * s) > 0;
  }
  S[i] = s;
  const int V = 9 * q - s * s;
  rs[i] = ok ? __fdiv_rn(1.0f, __fsqrt_rn((float)V)) : 0.0f;
  def[i] = (uint8_t)ok;
}

// ---------------------------------------------------------------------------
// Stage 2: NCC cost.  ncc(xl, xr, y): left block centred (xl,y), right (xr,y).
// The left volume evaluates (x, x-d), the right volume (x'+d, x'): the same
// function of the same operands, so right(u-d,v,d) == left(u,v,d) bit-exactly
// (P:L86 twin volumes).
struct CostArgs {
  int W, H, D, d_min, Dp, Wv, R, r0, r1;
  const uint32_t *PL, *PR;
  const int32_t *SL, *SR;
  const float *rL, *rR;
  const uint8_t *defL, *defR;
  float* vol;
};

__device__ __forceinline__ float ncc_cost(const CostArgs& a, int xl, int xr, int y) {
  if (xr < 0 || xl > a.W - 1) return kSent;
  const size_t il = (size_t)y * a.W + xl, ir = (size_t)y * a.W + xr;
  if (!a.defL[il] || !a.defR[ir]) return kSent;
  unsigned dot = __dp4a(__ldg(a.PL + il - a.W), __ldg(a.PR + ir - a.W), 0u);
  dot = __dp4a(__ldg(a.PL + il), __ldg(a.PR + ir), dot);
  dot = __dp4a(__ldg(a.PL + il + a.W), __ldg(a.PR + ir + a.W), dot);
  const int N = 9 * (int)dot - __ldg(a.SL + il) * __ldg(a.SR + ir);
  float c = __fmul_rn(__fmul_rn((float)N, __ldg(a.rL + il)), __ldg(a.rR + ir));
  return fminf(1.0f, fmaxf(-1.0f, c));  // clamp to [-1,1] (R#8)
}

// grid: (ceil(W/8), r1-r0, Dp/64); block 256 = 8 warps, warp <-> pixel x, lane <-> d pair
template <int SIDE>
__global__ void __launch_bounds__(256) k_cost(CostArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x = blockIdx.x * 8 + warp;
  const int y = a.r0 + blockIdx.y;
  if (x >= a.W || y >= a.r1) return;
  const int di0 = blockIdx.z * kDB + 2 * lane;
  float2 out;
  float* o = &out.x;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int di = di0 + k;
    const int d = a.d_min + di;
    float c = kSent;
    if (di < a.D) c = SIDE == 0 ? ncc_cost(a, x, x - d, y) : ncc_cost(a, x + d, x, y);
    o[k] = c;
  }
  float* dst = a.vol + ((size_t)(y + a.R) * a.Wv + (x + a.R)) * a.Dp + di0;
  *reinterpret_cast<float2*>(dst) = out;
}

// fill a buffer with a float value (volume margins = SENT)
__global__ void k_fill(float* p, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// padded volume -> [H][W][D] export (debug)
__global__ void k_export_vol(const float* __restrict__ vol, int W, int H, int D, int Dp, int Wv, int R,
                             float* __restrict__ out) {
  const size_t n = (size_t)W * H * D;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int di = (int)(i % D);
    const size_t p = i / D;
    const int x = (int)(p % W), y = (int)(p / W);
    out[i] = vol[((size_t)(y + R) * Wv + (x + R)) * Dp + di];
  }
}

// ---------------------------------------------------------------------------
// Stage 4 helpers shared by the fused epilogue and the debug select path.
//
// Eq.(9) LRC (tolerance 1, R#17) then Eq.(10) subpixel on aggregated costs
// (R#19, R#21).  d_int: left WTA disparity or -1; e: d_R(u - d_int, v) or -1.
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
// Stage 3: fused bilateral aggregation + WTA (+ LRC + subpixel when SIDE == 0).
struct AggArgs {
  int W, H, D, d_min, d_max, Dp, Wv, r0, r1;
  const float* vol;        // this side's cost volume, padded layout
  const uint8_t* guide;    // this side's image (Eq.(8) guide, R#11)
  const uint8_t* def_self; // block-defined mask of the guide image (folded into w)
  const uint8_t* def_other;// block-defined mask of the other image (x -+ d validity)
  int32_t* disp_int;       // SIDE 1: d_R map [H][W] (required); SIDE 0: optional d_L
  const int32_t* disp_r;   // SIDE 0: d_R map for the LRC
  float* disp_out;         // SIDE 0: final map rows [r0, r1) at (y - r0) * W + x
  float* agg_export;       // optional [H][W][D] export of the aggregated volume
  float wd[(2 * kMaxRadius + 1) * (2 * kMaxRadius + 1)];  // ω_d, Eq.(7)
  float wr[256];                                          // ω_r, Eq.(8)
};

__device__ __forceinline__ void ffma2(float2& acc, float w, float2 c) {
  unsigned long long A, B = *reinterpret_cast<unsigned long long*>(&c);
  unsigned long long C = *reinterpret_cast<unsigned long long*>(&acc);
  asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(w));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
  acc = *reinterpret_cast<float2*>(&C);
}

template <int R>
struct AggSmem {
  static constexpr int K1 = 2 * R + 1;
  static constexpr int WPW = kPY * K1 * K1 * kPX;   // weights per warp
  float w[kNWX * kNWY][WPW];                        // [warp][py][dy][dx][px]
  float rinv[kNWX * kNWY][32];                      // 1 / Σ_q w'(p,q), 0 if none
  float wr[256];
  float tb[kNWX * kNWY][8 * kTStride];              // WTA transpose, 8 pixels per round
  float bv[kNWX * kNWY][32], bcm[kNWX * kNWY][32], bcp[kNWX * kNWY][32], lastv[kNWX * kNWY][32];
  int bd[kNWX * kNWY][32], pend[kNWX * kNWY][32];
};

// Does any tap of this CTA tile need the explicit denominator for d-block b?
// (the other image's block at x -+ d undefined somewhere in range; conservative)
template <int SIDE, int R>
__device__ __forceinline__ bool need_slow(const AggArgs& a, int x0, int y0, int b) {
  const int qy0 = max(y0 - R, 1), qy1 = min(y0 + kTY - 1 + R, a.H - 2);
  const int qx0 = max(x0 - R, 1), qx1 = min(x0 + kTX - 1 + R, a.W - 2);
  const int d_lo = a.d_min + b * kDB, d_hi = min(d_lo + kDB - 1, a.d_max);
  int flag = 0;
  if (qy0 <= qy1 && qx0 <= qx1) {
    int lo, hi;
    if (SIDE == 0) { lo = qx0 - d_hi; hi = qx1 - d_lo; flag = lo < 1; }
    else { lo = qx0 + d_lo; hi = qx1 + d_hi; flag = hi > a.W - 2; }
    lo = max(lo, 0); hi = min(hi, a.W - 1);
    const int span = hi - lo + 1, rows = qy1 - qy0 + 1;
    for (int i = threadIdx.x; !flag && i < span * rows; i += kThreads) {
      const int yy = qy0 + i / span, xx = lo + i % span;
      flag = !a.def_other[(size_t)yy * a.W + xx];
    }
  }
  return __syncthreads_or(flag) != 0;
}

// FMA over the window rows for output rows [PY0, PY0+NPY) of the warp sub-tile.
// SLOW: explicit denominator (c undefined -> 0 in num, 0 in den).
template <int R, int PY0, int NPY, bool SLOW>
__device__ __forceinline__ void agg_rows(const float* __restrict__ vbase, size_t rowstride, int Dp,
                                         const float* __restrict__ wsm, float2 (&num)[NPY][kPX],
                                         float2 (&den)[NPY][kPX]) {
  constexpr int K1 = 2 * R + 1;
  constexpr int NC = kPX + 2 * R;
#pragma unroll
  for (int py = 0; py < NPY; ++py)
#pragma unroll
    for (int px = 0; px < kPX; ++px) {
      num[py][px] = make_float2(0.f, 0.f);
      if (SLOW) den[py][px] = make_float2(0.f, 0.f);
    }
#pragma unroll 1
  for (int r = PY0; r < PY0 + NPY + 2 * R; ++r) {
    float2 c[NC], v[NC];
    const float* rowp = vbase + (size_t)r * rowstride;
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      c[j] = __ldg(reinterpret_cast<const float2*>(rowp + (size_t)j * Dp));
      if (SLOW) {
        v[j].x = c[j].x == kSent ? 0.f : 1.f;
        v[j].y = c[j].y == kSent ? 0.f : 1.f;
        c[j].x = c[j].x == kSent ? 0.f : c[j].x;
        c[j].y = c[j].y == kSent ? 0.f : c[j].y;
      }
    }
#pragma unroll
    for (int pyl = 0; pyl < NPY; ++pyl) {
      const int dy = r - (PY0 + pyl);
      if (dy >= 0 && dy <= 2 * R) {
        const float4* wp = reinterpret_cast<const float4*>(wsm + ((PY0 + pyl) * K1 + dy) * K1 * kPX);
#pragma unroll
        for (int dx = 0; dx < K1; ++dx) {
          const float4 w = wp[dx];
          ffma2(num[pyl][0], w.x, c[dx + 0]);
          ffma2(num[pyl][1], w.y, c[dx + 1]);
          ffma2(num[pyl][2], w.z, c[dx + 2]);
          ffma2(num[pyl][3], w.w, c[dx + 3]);
          if (SLOW) {
            ffma2(den[pyl][0], w.x, v[dx + 0]);
            ffma2(den[pyl][1], w.y, v[dx + 1]);
            ffma2(den[pyl][2], w.z, v[dx + 2]);
            ffma2(den[pyl][3], w.w, v[dx + 3]);
          }
        }
      }
    }
  }
}

// WTA over one 8-pixel round (2 sub-tile rows): transpose through shared memory,
// each pixel scanned by 4 lanes x 16 d, combined with xor shuffles.
// Strictly-greater updates in ascending d => ties go to the smallest d (R#15).
template <int R>
__device__ __forceinline__ void wta_round(const AggArgs& a, AggSmem<R>& sm, int warp, int lane,
                                          int b, int nblk, int pyrow0, const float2 (&agg)[2][kPX],
                                          int sx, int sy) {
  float* tb = sm.tb[warp];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int px = 0; px < kPX; ++px)
      *reinterpret_cast<float2*>(tb + (i * kPX + px) * kTStride + 2 * lane) = agg[i][px];
  __syncwarp();
  const int j = lane >> 2, qq = lane & 3;
  const float* row = tb + j * kTStride;
  float vals[16];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 t = *reinterpret_cast<const float4*>(row + 16 * qq + 4 * k);
    vals[4 * k + 0] = t.x; vals[4 * k + 1] = t.y; vals[4 * k + 2] = t.z; vals[4 * k + 3] = t.w;
  }
  const int dbase = b * kDB + 16 * qq;  // disparity index (d - d_min) of vals[0]
  float best = -INFINITY;
  int bi = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const float v = (dbase + k < a.D) ? vals[k] : kSent;
    vals[k] = v;
    if (v > best) { best = v; bi = dbase + k; }
  }
#pragma unroll
  for (int m = 1; m <= 2; m <<= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, m);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  const int pyl = j >> 2, px = j & 3;
  const int pix = (pyrow0 + pyl) * kPX + px;  // pixel index within the warp sub-tile
  const int x = sx + px, y = sy + pyrow0 + pyl;
  if (a.agg_export && x < a.W && y < a.r1 && y >= a.r0) {
    float* dst = a.agg_export + ((size_t)y * a.W + x) * a.D;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (dbase + k < a.D) dst[dbase + k] = vals[k];
  }
  if (qq == 0) {
    const int loc = bi - b * kDB;
    float v_b = best;
    float cm_b = loc > 0 ? row[loc - 1] : sm.lastv[warp][pix];
    float cp_b = loc < kDB - 1 ? row[loc + 1] : kSent;
    if (b == 0) {
      sm.bv[warp][pix] = v_b; sm.bd[warp][pix] = bi; sm.bcm[warp][pix] = loc > 0 ? cm_b : kSent;
      sm.bcp[warp][pix] = cp_b; sm.pend[warp][pix] = (loc == kDB - 1);
    } else {
      if (sm.pend[warp][pix]) { sm.bcp[warp][pix] = row[0]; sm.pend[warp][pix] = 0; }
      if (v_b > sm.bv[warp][pix]) {
        sm.bv[warp][pix] = v_b; sm.bd[warp][pix] = bi; sm.bcm[warp][pix] = cm_b;
        sm.bcp[warp][pix] = cp_b; sm.pend[warp][pix] = (loc == kDB - 1);
      }
    }
    sm.lastv[warp][pix] = row[kDB - 1];
  }
  (void)nblk;
  __syncwarp();
}

template <int R>
__device__ __forceinline__ void to_agg(const float2& num, const float2& den, float2& out) {
  out.x = den.x > 0.f ? __fmul_rn(num.x, __fdiv_rn(1.0f, den.x)) : kSent;
  out.y = den.y > 0.f ? __fmul_rn(num.y, __fdiv_rn(1.0f, den.y)) : kSent;
}

// grid: (ceil(W/16), ceil((r1-r0)/16)); block 256 (8 warps, each a 4x8 sub-tile)
template <int SIDE, int R>
__global__ void __launch_bounds__(kThreads, (R <= 4) ? 2 : 1) k_agg(const AggArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  AggSmem<R>& sm = *reinterpret_cast<AggSmem<R>*>(smraw);
  constexpr int K1 = 2 * R + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = blockIdx.x * kTX, y0 = a.r0 + blockIdx.y * kTY;
  const int sx = x0 + (warp % kNWX) * kPX, sy = y0 + (warp / kNWX) * kPY;

  for (int i = threadIdx.x; i < 256; i += kThreads) sm.wr[i] = a.wr[i];
  __syncthreads();

  // ---- weights w'(p,q) = def_self(q) · ω_d(q-p) · ω_r(|i(q) - i(p)|), Eq.(6)-(8) ----
  {
    const int py = lane / kPX, px = lane % kPX;
    const int x = sx + px, y = sy + py;
    float* wsm = sm.w[warp];
    float wsum = 0.f;
    const bool inimg = x < a.W && y < a.H;
    const int gp = inimg ? a.guide[(size_t)y * a.W + x] : 0;
#pragma unroll 1
    for (int dy = 0; dy < K1; ++dy) {
      const int qy = y + dy - R;
#pragma unroll
      for (int dx = 0; dx < K1; ++dx) {
        const int qx = x + dx - R;
        float w = 0.f;
        if (inimg && qx >= 0 && qx < a.W && qy >= 0 && qy < a.H) {
          const size_t qi = (size_t)qy * a.W + qx;
          if (a.def_self[qi]) w = __fmul_rn(a.wd[dy * K1 + dx], sm.wr[abs((int)a.guide[qi] - gp)]);
        }
        wsum = __fadd_rn(wsum, w);  // dy-major, dx-minor: the FMA loop's order
        wsm[((py * K1 + dy) * K1 + dx) * kPX + px] = w;
      }
    }
    sm.rinv[warp][lane] = wsum > 0.f ? __fdiv_rn(1.0f, wsum) : 0.f;
  }
  __syncwarp();

  const int nblk = (a.D + kDB - 1) / kDB;
  const size_t rowstride = (size_t)a.Wv * a.Dp;
  for (int b = 0; b < nblk; ++b) {
    // volume row (sy - R + r) + R = sy + r; column (sx - R + j) + R = sx + j
    const float* vbase = a.vol + ((size_t)sy * a.Wv + sx) * a.Dp + b * kDB + 2 * lane;
    const bool slow = need_slow<SIDE, R>(a, x0, y0, b);
    if (!slow) {
      float2 num[kPY][kPX], den_unused[kPY][kPX];
      agg_rows<R, 0, kPY, false>(vbase, rowstride, a.Dp, sm.w[warp], num, den_unused);
#pragma unroll
      for (int rr = 0; rr < kPY / 2; ++rr) {
        float2 agg[2][kPX];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int px = 0; px < kPX; ++px) {
            const float ri = sm.rinv[warp][(2 * rr + i) * kPX + px];
            const float2 n = num[2 * rr + i][px];
            agg[i][px].x = ri > 0.f ? __fmul_rn(n.x, ri) : kSent;
            agg[i][px].y = ri > 0.f ? __fmul_rn(n.y, ri) : kSent;
          }
        wta_round<R>(a, sm, warp, lane, b, nblk, 2 * rr, agg, sx, sy);
      }
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float2 num[kPY / 2][kPX], den[kPY / 2][kPX];
        if (h == 0) agg_rows<R, 0, kPY / 2, true>(vbase, rowstride, a.Dp, sm.w[warp], num, den);
        else agg_rows<R, kPY / 2, kPY / 2, true>(vbase, rowstride, a.Dp, sm.w[warp], num, den);
#pragma unroll
        for (int rr = 0; rr < kPY / 4; ++rr) {
          float2 agg[2][kPX];
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int px = 0; px < kPX; ++px) to_agg<R>(num[2 * rr + i][px], den[2 * rr + i][px], agg[i][px]);
          wta_round<R>(a, sm, warp, lane, b, nblk, h * (kPY / 2) + 2 * rr, agg, sx, sy);
        }
      }
    }
  }

  // ---- epilogue: one lane per sub-tile pixel ----
  {
    const int py = lane / kPX, px = lane % kPX;
    const int x = sx + px, y = sy + py;
    if (x < a.W && y < a.r1) {
      const float bv = sm.bv[warp][lane];
      const int d_int = bv > kSent ? a.d_min + sm.bd[warp][lane] : -1;
      const size_t pi = (size_t)y * a.W + x;
      if (SIDE == 1) {
        a.disp_int[pi] = d_int;
      } else {
        if (a.disp_int) a.disp_int[pi] = d_int;
        int e = -1;
        if (d_int >= 0 && x - d_int >= 0) e = a.disp_r[pi - d_int];
        a.disp_out[(size_t)(y - a.r0) * a.W + x] =
            finalize_pixel(d_int, e, bv, sm.bcm[warp][lane], sm.bcp[warp][lane], a.d_min, a.d_max);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Debug select path: WTA over given [H][W][D] volumes, then LRC + subpixel.
__global__ void k_select_wta(const float* __restrict__ agg, int W, int H, int D, int d_min,
                             int32_t* __restrict__ disp, float* __restrict__ c3) {
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
  if (c3) {
    c3[3 * p + 0] = best;
    c3[3 * p + 1] = bi > 0 ? col[bi - 1] : kSent;
    c3[3 * p + 2] = bi < D - 1 ? col[bi + 1] : kSent;
  }
}

__global__ void k_select_final(const int32_t* __restrict__ dl, const int32_t* __restrict__ dr,
                               const float* __restrict__ c3, int W, int H, int d_min, int d_max,
                               float* __restrict__ out) {
  const size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (p >= (size_t)W * H) return;
  const int x = (int)(p % W);
  const int d = dl[p];
  int e = -1;
  if (d >= 0 && x - d >= 0) e = dr[p - d];
  out[p] = finalize_pixel(d, e, c3[3 * p], c3[3 * p + 1], c3[3 * p + 2], d_min, d_max);
}

}  // namespace fbs
