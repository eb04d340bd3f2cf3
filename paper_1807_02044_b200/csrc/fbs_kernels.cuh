// fbs_kernels.cuh — sm_100a kernels of the fast bilateral stereo (FBS) hot path.
//
// Stages (PAPER.md, arXiv 1807.02044; "P:Lnn" = PAPER.md line):
//   k_cost       block statistics (Eq.(2)(3), "pre-calculated" P:L84) fused
//                with the twin NCC cost volumes (Eq.(1)), both sides
//   k_agg        bilateral aggregation (Eq.(6)-(8), tables) + WTA
//                (P:L140), both sides in one grid
//   k_finalize   LRC (Eq.(9), left reference P:L203) + parabola
//                subpixel (Eq.(10))
//   k_select_*   WTA from given volumes (debug / parity only)
//
// Design notes (DESIGN.md §6 has the rationale and the rooflines):
//  * NCC in exact integer arithmetic: N = 9·Σ i_l i_r − S_l S_r and V = 9·Σ i² − S²
//    are integers < 2^24; c = (N · V_l^{-1/2}) · V_r^{-1/2} in fp32 (algebraically
//    identical to Eq.(1)-(3); R#5).  The 3x3 dot product is three DP4A on
//    packed 3-pixel rows.
//  * Aggregation: lanes <-> disparity pairs (32 lanes x 2 d = 64 d per block), one
//    FFMA2 per (output pixel, tap) with the warp-uniform weight w(p,q) = ω_d ω_r as a
//    broadcast scalar operand (SASS: FFMA2 R, Rw.F32, Rc.F32x2).  Weights are
//    d-independent: computed once per pixel window into shared memory and reused
//    across every disparity block ("pre-calculated").
//  * The d-independent validity (border / textureless block of the guide's own image)
//    is folded into the weights; the d-dependent part (the other image's block at
//    x -+ d) only matters near the frame edges and textureless regions, detected per
//    (CTA tile, d-block) and handled by an exact slow path with an explicit
//    denominator.  Both paths give bit-identical results.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fbs {

constexpr float kSent = -2.0f;   // undefined cost / aggregated cost (R#7)
constexpr int kMaxRadius = 6;    // FBS_MAX_RADIUS
constexpr int kDB = 64;          // disparities per block (32 lanes x 2)
constexpr int kPX = 4;           // warp sub-tile width  (pixels)
#ifndef FBS_PY
#define FBS_PY 6
#endif
constexpr int kPY = FBS_PY;      // warp sub-tile height (pixels)
constexpr int kNWX = 4;          // warps across a CTA tile
constexpr int kNWY = 2;          // warps down a CTA tile
constexpr int kTX = kPX * kNWX;  // CTA tile 16 x 12
constexpr int kTY = kPY * kNWY;
constexpr int kPYS = kPY % 4 == 0 ? 4 : 2;  // slow-path rows per pass
constexpr int kThreads = 32 * kNWX * kNWY;
constexpr int kTStride = 68;     // WTA transpose row stride (floats): 16B aligned, conflict-free
constexpr int kCX = 64;          // cost kernel: pixels per CTA (multiple of 32)
// Range-weight LUT indexed by Δ + 255 for Δ = i(q) - i(p) in [-255, 255]; an
// undefined tap q stores kGuideSent instead of i(q) + 255, landing in the zero tail.
constexpr int kGuideSent = 1021;
constexpr int kLut = 1024;

// Cost volume layout: [Hv][nblk][Wv][64] floats; pixel (x, y), disparity index
// di = b*64 + dl lives at ((vy*nblk + b)*Wv + vx)*64 + dl with vy = y + R,
// vx = x + R.  A pixel column step is a constant 256 B (immediate load offsets).
__host__ __device__ __forceinline__ size_t vol_at(int vy, int b, int vx, int nblk, int Wv) {
  return (((size_t)vy * nblk + b) * Wv + vx) * kDB;
}

// ---------------------------------------------------------------------------
// Stage 1+2: block statistics fused with the twin NCC cost volumes.
struct CostArgs {
  int W, H, D, d_min, nblk, Wv, R, r0, r1, Wb;  // [r0, r1): cost rows; Wb = words per mask row
  const uint8_t *L, *Rimg;
  float *volL, *volR;
  uint8_t *defL, *defR;                         // block-defined masks (bytes), rows [r0, r1)
  uint32_t *bitsL, *bitsR;                      // the same masks bit-packed [H][Wb]
};

// Eq.(2)(3) x 81 in integers: packed rows P (i(x-1) | i(x)<<8 | i(x+1)<<16 of rows
// y-1, y, y+1), S = Σ i, and V^{-1/2} (0 when the block is a border or
// textureless block, or x is outside the image: σ < σ_floor <=> V = 0, R#7).
__device__ __forceinline__ void block_pack(const uint8_t* __restrict__ img, int W, int H, int x, int y,
                                           uint4& P, float& rs) {
  P = make_uint4(0u, 0u, 0u, 0u);
  rs = 0.f;
  if (x < 1 || x > W - 2 || y < 1 || y > H - 2) return;
  int s = 0, q = 0;
  uint32_t pk[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const uint8_t* row = img + (size_t)(y - 1 + k) * W + x - 1;
    const uint32_t a = row[0], b = row[1], c = row[2];
    pk[k] = a | (b << 8) | (c << 16);
    s += (int)(a + b + c);
    q += (int)(a * a + b * b + c * c);
  }
  const int V = 9 * q - s * s;
  P = make_uint4(pk[0], pk[1], pk[2], (uint32_t)s);
  if (V > 0) rs = __fdiv_rn(1.0f, __fsqrt_rn((float)V));
}

// side 0: left volume c(x, x-d); side 1: right volume c(x'+d, x').  The same
// function of the same operands ((N · r_left) · r_right), so
// right(u-d,v,d) == left(u,v,d) bit-exactly.
template <int SIDE>
__device__ __forceinline__ void cost_side(const CostArgs& a, uint4* csm) {
  const int y = a.r0 + blockIdx.y;
  const int x0 = blockIdx.x * kCX;
  const int dspan = a.nblk * kDB;
  const uint8_t* self_img = SIDE == 0 ? a.L : a.Rimg;
  const uint8_t* oth_img = SIDE == 0 ? a.Rimg : a.L;
  const int olo = SIDE == 0 ? x0 - a.d_min - dspan + 1 : x0 + a.d_min;
  const int ocount = kCX + dspan - 1;
  uint4* sP = csm;
  uint4* oP = csm + kCX;
  float* sR = reinterpret_cast<float*>(csm + kCX + ocount);
  float* oR = sR + kCX;
  for (int i = threadIdx.x; i < kCX + ocount; i += blockDim.x) {
    uint4 P;
    float rs;
    if (i < kCX) {
      block_pack(self_img, a.W, a.H, x0 + i, y, P, rs);
      sP[i] = P; sR[i] = rs;
      const bool ok = rs != 0.f;
      const unsigned bits = __ballot_sync(0xffffffffu, ok);  // kCX is a multiple of 32
      if (x0 + i < a.W) (SIDE == 0 ? a.defL : a.defR)[(size_t)y * a.W + x0 + i] = ok;
      if ((i & 31) == 0 && x0 + i < a.W) (SIDE == 0 ? a.bitsL : a.bitsR)[(size_t)y * a.Wb + (x0 + i) / 32] = bits;
    } else {
      const int j = i - kCX;
      block_pack(oth_img, a.W, a.H, olo + j, y, P, rs);
      oP[j] = P; oR[j] = rs;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* vol = SIDE == 0 ? a.volL : a.volR;
  for (int xi = warp; xi < kCX; xi += 8) {
    const int x = x0 + xi;
    if (x >= a.W) break;
    const uint4 ps = sP[xi];
    const float rsf = sR[xi];
    float* vp = vol + vol_at(y + a.R, 0, x + a.R, a.nblk, a.Wv) + 2 * lane;
    for (int b = 0; b < a.nblk; ++b) {
      const int di0 = b * kDB + 2 * lane;
      // other-image staging index of disparity index di: x -+ (d_min + di) - olo
      const int j0 = SIDE == 0 ? xi + dspan - 1 - di0 : xi + di0;
      float o[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int j = SIDE == 0 ? j0 - k : j0 + k;
        const float rof = oR[j];
        const uint4 po = oP[j];
        unsigned dot = __dp4a(ps.x, po.x, 0u);
        dot = __dp4a(ps.y, po.y, dot);
        dot = __dp4a(ps.z, po.z, dot);
        const int N = 9 * (int)dot - (int)ps.w * (int)po.w;
        const float rl = SIDE == 0 ? rsf : rof, rr = SIDE == 0 ? rof : rsf;
        float c = __fmul_rn(__fmul_rn((float)N, rl), rr);
        c = fminf(1.0f, fmaxf(-1.0f, c));  // clamp (R#8)
        o[k] = (rsf != 0.f && rof != 0.f && di0 + k < a.D) ? c : kSent;
      }
      *reinterpret_cast<float2*>(vp + (size_t)b * a.Wv * kDB) = make_float2(o[0], o[1]);
    }
  }
}

// grid: (ceil(W/kCX), r1-r0, 2 sides); block 256 = 8 warps; warp <-> pixel, lane <-> d pair.
__global__ void __launch_bounds__(256) k_cost(CostArgs a) {
  extern __shared__ uint4 csm[];
  if (blockIdx.z == 0) cost_side<0>(a, csm);
  else cost_side<1>(a, csm);
}

// fill a buffer with a float value (volume margins = SENT)
__global__ void k_fill(float* p, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// padded volume -> [H][W][D] export (debug)
__global__ void k_export_vol(const float* __restrict__ vol, int W, int H, int D, int nblk, int Wv, int R,
                             float* __restrict__ out) {
  const size_t n = (size_t)W * H * D;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int di = (int)(i % D);
    const size_t p = i / D;
    const int x = (int)(p % W), y = (int)(p / W);
    out[i] = vol[vol_at(y + R, di / kDB, x + R, nblk, Wv) + di % kDB];
  }
}

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

// rows [r0, r1): out[(y - r0)*W + x]
__global__ void k_finalize(const int32_t* __restrict__ dl, const int32_t* __restrict__ dr,
                           const float4* __restrict__ c3, int W, int r0, int r1, int d_min, int d_max,
                           float* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = r0 + blockIdx.y;
  if (x >= W || y >= r1) return;
  const size_t p = (size_t)y * W + x;
  const int d = dl[p];
  int e = -1;
  if (d >= 0 && x - d >= 0) e = dr[p - d];
  const float4 c = c3[p];
  out[(size_t)(y - r0) * W + x] = finalize_pixel(d, e, c.x, c.y, c.z, d_min, d_max);
}

// ---------------------------------------------------------------------------
// Stage 3: fused bilateral aggregation + WTA, both sides in one grid.
struct AggArgs {
  int W, H, D, d_min, d_max, nblk, Wv, r0, r1;
  const float *volL, *volR;      // cost volumes (padded layout)
  const uint8_t *L, *Rimg;       // guides (Eq.(8); right image guides the right volume, R#11)
  const uint8_t *defL, *defR;    // block-defined masks
  const uint32_t *bitsL, *bitsR; // the same masks bit-packed [H][Wb]
  int Wb;
  int32_t *dL, *dR;              // WTA maps [H][W]
  float4* c3;                    // left: (c(d*), c(d*-1), c(d*+1), -) [H][W]
  float *exportL, *exportR;      // optional [H][W][D] aggregated volumes
  unsigned long long* tile_stats;  // optional [2]: (fast, slow) (CTA tile, d-block) decisions
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
  static constexpr int GW = kTX + 2 * R, GH = kTY + 2 * R;
  float w[kNWX * kNWY][WPW];                        // [warp][py][dy][dx][px]
  float rinv[kNWX * kNWY][32];                      // 1 / Σ_q w'(p,q), 0 if none
  float lut[kLut];                                  // ω_r(|Δ|) at Δ + 255, zero tail
  float tb[kNWX * kNWY][8 * kTStride];              // WTA transpose, 8 pixels per round
  float bv[kNWX * kNWY][32], bcm[kNWX * kNWY][32], bcp[kNWX * kNWY][32], lastv[kNWX * kNWY][32];
  int bd[kNWX * kNWY][32], pend[kNWX * kNWY][32];
  int g[GH * GW];                                   // 4*(i(q)+255), or 4*kGuideSent if undefined
};

// Does any tap of this CTA tile need the explicit denominator for d-block b?
// (the other image's block at x -+ d undefined somewhere in range; conservative)
// One 32-bit word of the bit-packed mask per thread.
template <int R>
__device__ __forceinline__ bool need_slow(const AggArgs& a, int side, int x0, int y0, int b) {
  const int qy0 = max(y0 - R, 1), qy1 = min(y0 + kTY - 1 + R, a.H - 2);
  const int qx0 = max(x0 - R, 1), qx1 = min(x0 + kTX - 1 + R, a.W - 2);
  const int d_lo = a.d_min + b * kDB, d_hi = min(d_lo + kDB - 1, a.d_max);
  const uint32_t* bits = side == 0 ? a.bitsR : a.bitsL;
  int flag = 0;
  if (qy0 <= qy1 && qx0 <= qx1) {
    int lo, hi;
    if (side == 0) { lo = qx0 - d_hi; hi = qx1 - d_lo; flag = lo < 1; }
    else { lo = qx0 + d_lo; hi = qx1 + d_hi; flag = hi > a.W - 2; }
    if (!flag) {
      const int w0 = lo >> 5, nw = (hi >> 5) - w0 + 1, rows = qy1 - qy0 + 1;
      for (int i = threadIdx.x; i < nw * rows; i += kThreads) {
        const int yy = qy0 + i / nw, wi = w0 + i % nw;
        uint32_t m = 0xffffffffu;
        if (wi == w0) m &= 0xffffffffu << (lo & 31);
        if (wi == (hi >> 5)) m &= 0xffffffffu >> (31 - (hi & 31));
        flag |= (~__ldg(bits + (size_t)yy * a.Wb + wi) & m) != 0u;
      }
    }
  }
  return __syncthreads_or(flag) != 0;
}

// One cost row r of the fast path: all tap tests are template constants, so the
// FFMA2 stream is branch- and predicate-free (template recursion guarantees the
// unroll; a #pragma unroll over 14 rows was re-rolled by the compiler into a
// predicated loop).
template <int R, int NPY, int PY0, int r>
__device__ __forceinline__ void row_fma(const float2* c, const float* __restrict__ wsm,
                                        float2 (&num)[NPY][kPX]) {
  constexpr int K1 = 2 * R + 1;
#pragma unroll
  for (int dx = 0; dx < K1; ++dx) {
#pragma unroll
    for (int pyl = 0; pyl < NPY; ++pyl) {
      const int dy = r - pyl;
      if (dy >= 0 && dy <= 2 * R) {
        const float4 w = reinterpret_cast<const float4*>(wsm + ((PY0 + pyl) * K1 + dy) * K1 * kPX)[dx];
        ffma2(num[pyl][0], w.x, c[dx + 0]);
        ffma2(num[pyl][1], w.y, c[dx + 1]);
        ffma2(num[pyl][2], w.z, c[dx + 2]);
        ffma2(num[pyl][3], w.w, c[dx + 3]);
      }
    }
  }
}

template <int R, int r, int NR>
struct FastRows {
  static __device__ __forceinline__ void run(const float* __restrict__ vb, size_t rowstride,
                                             const float* __restrict__ wsm, float2 (&cn)[kPX + 2 * R],
                                             float2 (&num)[kPY][kPX]) {
    constexpr int NC = kPX + 2 * R;
    float2 c[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) c[j] = cn[j];
    if constexpr (r + 1 < NR) {
      const float* rp = vb + (size_t)(r + 1) * rowstride;
#pragma unroll
      for (int j = 0; j < NC; ++j) cn[j] = __ldg(reinterpret_cast<const float2*>(rp + j * kDB));
    }
    row_fma<R, kPY, 0, r>(c, wsm, num);
    FastRows<R, r + 1, NR>::run(vb, rowstride, wsm, cn, num);
  }
};
template <int R, int NR>
struct FastRows<R, NR, NR> {
  static __device__ __forceinline__ void run(const float*, size_t, const float*, float2 (&)[kPX + 2 * R],
                                             float2 (&)[kPY][kPX]) {}
};

// Fast path: every tap's other-image block is defined in this d-block, so the
// denominator is the d-independent Σ w'.  Software-pipelined: row r+1's cost
// pairs are in flight while row r is consumed.
template <int R>
__device__ __forceinline__ void agg_fast(const float* __restrict__ vb, size_t rowstride,
                                         const float* __restrict__ wsm, float2 (&num)[kPY][kPX]) {
  constexpr int NC = kPX + 2 * R;
#pragma unroll
  for (int py = 0; py < kPY; ++py)
#pragma unroll
    for (int px = 0; px < kPX; ++px) num[py][px] = make_float2(0.f, 0.f);
  float2 cn[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) cn[j] = __ldg(reinterpret_cast<const float2*>(vb + j * kDB));
  FastRows<R, 0, kPY + 2 * R>::run(vb, rowstride, wsm, cn, num);
}

// Slow path for output rows [PY0, PY0+NPY): explicit num and den (undefined
// costs contribute 0 to both), same tap order as the fast path, so every
// pixel gets bit-identical results on either path.
template <int R, int PY0, int NPY>
__device__ __forceinline__ void agg_slow(const float* __restrict__ vb, size_t rowstride,
                                         const float* __restrict__ wsm, float2 (&num)[NPY][kPX],
                                         float2 (&den)[NPY][kPX]) {
  constexpr int K1 = 2 * R + 1;
  constexpr int NC = kPX + 2 * R;
  constexpr int NR = NPY + 2 * R;
#pragma unroll
  for (int py = 0; py < NPY; ++py)
#pragma unroll
    for (int px = 0; px < kPX; ++px) {
      num[py][px] = make_float2(0.f, 0.f);
      den[py][px] = make_float2(0.f, 0.f);
    }
  const float* vb0 = vb + (size_t)PY0 * rowstride;
  float2 c[NC], cn[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) cn[j] = __ldg(reinterpret_cast<const float2*>(vb0 + j * kDB));
#pragma unroll
  for (int r = 0; r < NR; ++r) {
#pragma unroll
    for (int j = 0; j < NC; ++j) c[j] = cn[j];
    if (r + 1 < NR) {
      const float* rp = vb0 + (size_t)(r + 1) * rowstride;
#pragma unroll
      for (int j = 0; j < NC; ++j) cn[j] = __ldg(reinterpret_cast<const float2*>(rp + j * kDB));
    }
    float2 v[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      v[j].x = c[j].x == kSent ? 0.f : 1.f;
      v[j].y = c[j].y == kSent ? 0.f : 1.f;
      c[j].x = c[j].x == kSent ? 0.f : c[j].x;
      c[j].y = c[j].y == kSent ? 0.f : c[j].y;
    }
#pragma unroll
    for (int dx = 0; dx < K1; ++dx) {
#pragma unroll
      for (int pyl = 0; pyl < NPY; ++pyl) {
        const int dy = r - pyl;
        if (dy < 0 || dy > 2 * R) continue;
        const float4 w = reinterpret_cast<const float4*>(wsm + ((PY0 + pyl) * K1 + dy) * K1 * kPX)[dx];
        ffma2(num[pyl][0], w.x, c[dx + 0]);
        ffma2(num[pyl][1], w.y, c[dx + 1]);
        ffma2(num[pyl][2], w.z, c[dx + 2]);
        ffma2(num[pyl][3], w.w, c[dx + 3]);
        ffma2(den[pyl][0], w.x, v[dx + 0]);
        ffma2(den[pyl][1], w.y, v[dx + 1]);
        ffma2(den[pyl][2], w.z, v[dx + 2]);
        ffma2(den[pyl][3], w.w, v[dx + 3]);
      }
    }
  }
}

// slow path over the whole sub-tile in passes of kPYS rows (register budget)
template <int R, int P>
__device__ __forceinline__ void slow_pass(const AggArgs& a, AggSmem<R>& sm, float* exp_out, const float* vb,
                                          size_t rowstride, int warp, int lane, int b, int sx, int sy);

// WTA over one 8-pixel round (2 sub-tile rows): transpose through shared memory,
// each pixel scanned by 4 lanes x 16 d, combined with xor shuffles.
// Strictly-greater updates in ascending d => ties go to the smallest d (R#15).
template <int R>
__device__ __forceinline__ void wta_round(const AggArgs& a, AggSmem<R>& sm, float* exp_out, int warp,
                                          int lane, int b, int pyrow0, const float2 (&agg)[2][kPX],
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
  if (exp_out && x < a.W && y < a.r1 && y >= a.r0) {
    float* dst = exp_out + ((size_t)y * a.W + x) * a.D;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (dbase + k < a.D) dst[dbase + k] = vals[k];
  }
  if (qq == 0) {
    const int loc = bi - b * kDB;
    const float v_b = best;
    const float cm_b = loc > 0 ? row[loc - 1] : sm.lastv[warp][pix];
    const float cp_b = loc < kDB - 1 ? row[loc + 1] : kSent;
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
  __syncwarp();
}

__device__ __forceinline__ void to_agg(const float2& num, const float2& den, float2& out) {
  out.x = den.x > 0.f ? __fmul_rn(num.x, __fdiv_rn(1.0f, den.x)) : kSent;
  out.y = den.y > 0.f ? __fmul_rn(num.y, __fdiv_rn(1.0f, den.y)) : kSent;
}

template <int R, int P>
__device__ __forceinline__ void slow_pass(const AggArgs& a, AggSmem<R>& sm, float* exp_out, const float* vb,
                                          size_t rowstride, int warp, int lane, int b, int sx, int sy) {
  if constexpr (P * kPYS < kPY) {
    float2 num[kPYS][kPX], den[kPYS][kPX];
    agg_slow<R, P * kPYS, kPYS>(vb, rowstride, sm.w[warp], num, den);
#pragma unroll
    for (int rr = 0; rr < kPYS / 2; ++rr) {
      float2 agg[2][kPX];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int px = 0; px < kPX; ++px) to_agg(num[2 * rr + i][px], den[2 * rr + i][px], agg[i][px]);
      wta_round<R>(a, sm, exp_out, warp, lane, b, P * kPYS + 2 * rr, agg, sx, sy);
    }
    slow_pass<R, P + 1>(a, sm, exp_out, vb, rowstride, warp, lane, b, sx, sy);
  }
}

// grid: (ceil(W/kTX), ceil((r1-r0)/kTY), 2 sides); block 256 (8 warps, each a kPX x kPY sub-tile)
template <int R>
__global__ void __launch_bounds__(kThreads, (R <= 4) ? 2 : 1) k_agg(const AggArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  AggSmem<R>& sm = *reinterpret_cast<AggSmem<R>*>(smraw);
  constexpr int K1 = 2 * R + 1;
  constexpr int GW = AggSmem<R>::GW, GH = AggSmem<R>::GH;
  const int side = blockIdx.z;  // 0: left volume / left guide, 1: right
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = blockIdx.x * kTX, y0 = a.r0 + blockIdx.y * kTY;
  const int wx = (warp % kNWX) * kPX, wy = (warp / kNWX) * kPY;
  const int sx = x0 + wx, sy = y0 + wy;
  const uint8_t* guide = side == 0 ? a.L : a.Rimg;
  const uint8_t* def_self = side == 0 ? a.defL : a.defR;

  for (int i = threadIdx.x; i < kLut; i += kThreads) {
    const int dlt = i - 255;
    sm.lut[i] = (dlt >= -255 && dlt <= 255) ? a.wr[abs(dlt)] : 0.f;
  }
  for (int i = threadIdx.x; i < GH * GW; i += kThreads) {
    const int qx = x0 - R + i % GW, qy = y0 - R + i / GW;
    int g = kGuideSent;
    if (qx >= 0 && qx < a.W && qy >= 0 && qy < a.H) {
      const size_t qi = (size_t)qy * a.W + qx;
      if (def_self[qi]) g = guide[qi] + 255;
    }
    sm.g[i] = 4 * g;  // byte offset into sm.lut before subtracting 4*i(p)
  }
  __syncthreads();

  // ---- weights w'(p,q) = def_self(q) · ω_d(q-p) · ω_r(|i(q) - i(p)|), Eq.(6)-(8) ----
  if (lane < kPX * kPY) {
    const int py = lane / kPX, px = lane % kPX;
    // pixels outside the frame get some in-frame guide value: their outputs are discarded
    const int x = min(sx + px, a.W - 1), y = min(sy + py, a.H - 1);
    float* wsm = sm.w[warp];
    const char* lutp = reinterpret_cast<const char*>(sm.lut) - 4 * (int)guide[(size_t)y * a.W + x];
    const int* gq = sm.g + (wy + py) * GW + (wx + px);
    float wsum = 0.f;
#pragma unroll
    for (int dy = 0; dy < K1; ++dy)
#pragma unroll
      for (int dx = 0; dx < K1; ++dx) {
        const float wr = *reinterpret_cast<const float*>(lutp + gq[dy * GW + dx]);
        const float w = __fmul_rn(a.wd[dy * K1 + dx], wr);
        wsum = __fadd_rn(wsum, w);  // dy-major, dx-minor: the FMA loops' order
        wsm[((py * K1 + dy) * K1 + dx) * kPX + px] = w;
      }
    sm.rinv[warp][lane] = wsum > 0.f ? __fdiv_rn(1.0f, wsum) : 0.f;
  }
  __syncwarp();

  const float* vol = side == 0 ? a.volL : a.volR;
  float* exp_out = side == 0 ? a.exportL : a.exportR;
  const size_t rowstride = (size_t)a.nblk * a.Wv * kDB;
  for (int b = 0; b < a.nblk; ++b) {
    // volume row (sy - R + r) + R = sy + r; column (sx - R + j) + R = sx + j
    const float* vb = vol + vol_at(sy, b, sx, a.nblk, a.Wv) + 2 * lane;
    const bool slow = need_slow<R>(a, side, x0, y0, b);
    if (a.tile_stats && threadIdx.x == 0) atomicAdd(a.tile_stats + (slow ? 1 : 0), 1ull);
    if (!slow) {
      float2 num[kPY][kPX];
      agg_fast<R>(vb, rowstride, sm.w[warp], num);
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
        wta_round<R>(a, sm, exp_out, warp, lane, b, 2 * rr, agg, sx, sy);
      }
    } else {
      slow_pass<R, 0>(a, sm, exp_out, vb, rowstride, warp, lane, b, sx, sy);
    }
  }

  // ---- epilogue: one lane per sub-tile pixel ----
  if (lane < kPX * kPY) {
    const int py = lane / kPX, px = lane % kPX;
    const int x = sx + px, y = sy + py;
    if (x < a.W && y < a.r1) {
      const float bv = sm.bv[warp][lane];
      const int d_int = bv > kSent ? a.d_min + sm.bd[warp][lane] : -1;
      const size_t pi = (size_t)y * a.W + x;
      if (side == 1) {
        a.dR[pi] = d_int;
      } else {
        a.dL[pi] = d_int;
        a.c3[pi] = make_float4(bv, sm.bcm[warp][lane], sm.bcp[warp][lane], 0.f);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Debug select path: WTA over a given [H][W][D] volume (same rules as k_agg).
__global__ void k_select_wta(const float* __restrict__ agg, int W, int H, int D, int d_min,
                             int32_t* __restrict__ disp, float4* __restrict__ c3) {
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
  if (c3) c3[p] = make_float4(best, bi > 0 ? col[bi - 1] : kSent, bi < D - 1 ? col[bi + 1] : kSent, 0.f);
}

}  // namespace fbs
