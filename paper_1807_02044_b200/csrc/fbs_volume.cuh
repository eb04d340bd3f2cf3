// fbs_volume.cuh — the volume path of the sm_100a FBS hot path (round-1 design,
// kept as the default: measured faster than the fused walker on every
// configuration).  Three launches per frame:
//   k_cost      block statistics (Eq.(2)(3), "pre-calculated" P:L84) and
//               the twin NCC cost volumes (Eq.(1)) of both sides, written to
//               a padded [Hv][nblk][Wv][64] f32 volume per side (L2-resident at
//               Teddy: 2 x 45 MB of the 126 MB L2)
//   k_agg       bilateral aggregation (Eq.(6)-(8)) + WTA (P:L140,
//               P:L201), both sides per launch, costs read by LDG
//   k_finalize  LRC (Eq.(9)) + parabola subpixel (Eq.(10))
// Everything lives in namespace fbs::vol; fbs_fused.cuh / fbs_ws.cuh hold the
// fused path (costs computed into shared memory, never written to HBM).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fbs_kernels.cuh"  // fbs::OutSet (band scatter)

namespace fbs {
namespace vol {


// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in
// the stream finishes; pdl_wait() blocks until that predecessor has completed
// and its memory is visible, pdl_trigger() lets the successor launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

constexpr float kSent = -2.0f;   // undefined aggregated cost / exported cost (R#7)
constexpr float kUndef = -0.0f;  // undefined cost inside the volumes (never a defined NCC value)
constexpr int kMaxRadius = 10;   // FBS_MAX_RADIUS (volume path; the fused path stops at 6)
constexpr int kDB = 64;          // disparities per block (32 lanes x 2)
constexpr int kPX = 4;           // warp sub-tile width  (pixels)
constexpr int kPYMax = 6;        // warp sub-tile height (pixels) for radius <= 5
constexpr int kNWX = 4;          // warps across a CTA tile
constexpr int kTX = kPX * kNWX;  // CTA tile width (16)

// Per-radius CTA geometry of k_agg: the weight buffers grow as (2ρ+1)², so the
// largest radius uses one warp row (4 warps, 16x6 tiles) to keep several CTAs
// resident per SM.
// ρ >= 7 (NEXT-1, the paper's Fig. 7 range): one output row per half-warp, the
// stream as a cost-row loop (the unrolled form would not fit the instruction
// cache), two CTAs per SM up to ρ = 8 and one beyond (weights: 2 K1² x 4 px per warp).
template <int R>
struct AggGeom {
  static constexpr int HPY = R >= 7 ? 1 : (R >= 6 ? 2 : 3);  // output rows per half-warp
  static constexpr int PY = 2 * HPY;              // warp sub-tile height (4 x PY pixels)
  static constexpr int NWY = 2;                   // warps down a CTA tile
  static constexpr int NW = kNWX * NWY;
  static constexpr int TY = PY * NWY;             // CTA tile height
  static constexpr int THREADS = 32 * NW;
  static constexpr int MINB = R >= 9 ? 1 : 2;     // CTAs per SM the registers are budgeted for
  static constexpr bool kRolled = R >= 7;         // cost-row loop instead of the unrolled stream
  static constexpr int CWS = R >= 7 ? 96 : 64;    // classification words per warp (PY + 2R <= 24 rows x 4)
};
constexpr int kTYMax = kPYMax * 2;                // tallest CTA tile of any radius
__host__ __device__ constexpr int agg_tile_h(int R) { return R >= 7 ? 4 : (R >= 6 ? 4 : kPYMax) * 2; }

#ifndef FBS_KCX
#define FBS_KCX 64
#endif
constexpr int kCX = FBS_KCX;     // cost kernel: pixels per CTA (multiple of 32)
// Padded guide images for k_agg (written by k_cost): i(q) as a float, with an
// R-pixel margin of kGuideUndef outside the frame.  A pixel whose own block is
// undefined stores i + kGuideFlag: as a tap q it is >= 2^23 - 255 away from any
// intensity, so its weight flushes to exactly +0 (nkr <= -2e-12, fbs_create), and as a
// centre p its intensity is recovered exactly (i + 2^23 is exact in fp32).
constexpr float kGuideUndef = 1e30f;
constexpr float kGuideFlag = 8388608.0f;
__host__ __device__ constexpr int guide_pitch(int W, int R) { return ((W + 15) / 16 * 16 + 2 * R + 4 + 3) / 4 * 4; }
__host__ __device__ constexpr int guide_rows(int H, int R) { return (H + kTYMax - 1) / kTYMax * kTYMax + kTYMax + 2 * R; }

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
  int vbase;                                     // frame row of volume row R (0; band handles: first cost row)
  const uint8_t *L, *Rimg;
  float *volL, *volR;
  uint32_t *bitsL, *bitsR;                      // block-defined masks, bit-packed [H][Wb]
  float *gpadL, *gpadR;                         // padded guide images [guide_rows][Wg] (k_agg)
  int Wg;
};

// Cost kernel shared memory for a staging of ncol image columns and nblkpos
// block positions (self + other image).
//   column c of row y:  packed column P = i(x,y-1) | i(x,y) << 8 | i(x,y+1) << 16,
//                        column sum and sum of squares (Eq.(2)(3) split by columns)
//   block at x:          S = Σ_3x3 i, r = V^{-1/2} with V = 9 Σ i² - S² (exact
//                        integers < 2^24), r = 0 for a border or textureless block
//                        (σ < σ_floor <=> V = 0, R#7)
struct CostStage {
  uint32_t* cP;
  int* cS;
  int* cQ;
  int2* bSR;  // (S, r bits)
};

// side 0: left volume c(x, x-d); side 1: right volume c(x'+d, x').  The same
// function of the same operands (N · (r_self · r_other), a commutative product),
// so right(u-d,v,d) == left(u,v,d) bit-exactly.
// NRUN: runs of 8 pixels per warp.  NRUN = 1: a lane per disparity pair of a 64-slot
// block (32 pairs); NRUN = 4 (D <= 16): 8 lanes per run (8 pairs = 16 disparities), four
// runs per warp and a 4x wider CTA, so no lane computes padding slots (they keep the
// undefined value the volumes were filled with at create).
template <int SIDE, int NRUN>
__device__ __forceinline__ void cost_side(const CostArgs& a, unsigned char* smraw) {
  constexpr int kCX = vol::kCX * NRUN;  // pixels per CTA
  const int y = a.r0 + blockIdx.y;
  const int x0 = blockIdx.x * kCX;
  const int dspan = a.nblk * kDB;
  const uint8_t* self_img = SIDE == 0 ? a.L : a.Rimg;
  const uint8_t* oth_img = SIDE == 0 ? a.Rimg : a.L;
  // other-image block positions olo .. olo + ocount - 1 (x -+ d over the block range)
  const int olo = SIDE == 0 ? x0 - a.d_min - dspan + 1 : x0 + a.d_min;
  const int ocount = kCX + dspan - 1;
  const int ncs = kCX + 2, nco = ocount + 2;  // columns: self x0-1 .., other olo-1 ..
  uint32_t* cP = reinterpret_cast<uint32_t*>(smraw);
  int* cS = reinterpret_cast<int*>(cP + ncs + nco);
  int* cQ = cS + ncs + nco;
  int2* bSR = reinterpret_cast<int2*>(cQ + ncs + nco + ((ncs + nco) & 1));  // self kCX, then other ocount
  const bool row_ok = y >= 1 && y <= a.H - 2;
  // 1. columns (coalesced byte loads of the three rows)
  for (int i = threadIdx.x; i < ncs + nco; i += blockDim.x) {
    const bool self = i < ncs;
    const int x = self ? x0 - 1 + i : olo - 1 + (i - ncs);
    const uint8_t* img = self ? self_img : oth_img;
    uint32_t P = 0u;
    int cs = 0, cq = 0;
    if (row_ok && x >= 0 && x < a.W) {
      const uint32_t u0 = img[(size_t)(y - 1) * a.W + x], u1 = img[(size_t)y * a.W + x],
                     u2 = img[(size_t)(y + 1) * a.W + x];
      P = u0 | (u1 << 8) | (u2 << 16);
      cs = (int)(u0 + u1 + u2);
      cq = (int)(u0 * u0 + u1 * u1 + u2 * u2);
    }
    cP[i] = P; cS[i] = cs; cQ[i] = cq;
  }
  __syncthreads();
  // 2. block statistics; the self blocks also write the guide image and the masks
  for (int j = threadIdx.x; j < kCX + ocount; j += blockDim.x) {
    const bool self = j < kCX;
    const int c = self ? j : ncs + (j - kCX);  // first of the block's three columns
    const int x = self ? x0 + j : olo + (j - kCX);
    const int S = cS[c] + cS[c + 1] + cS[c + 2];
    const int V = 9 * (cQ[c] + cQ[c + 1] + cQ[c + 2]) - S * S;
    float rs = 0.f;
    if (row_ok && x >= 1 && x <= a.W - 2 && V > 0) {  // MUFU rsqrt + one Newton step (~1 ulp)
      const float v = (float)V;                        // exact: V < 2^24
      float r;
      asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
      rs = __fmul_rn(r, __fmaf_rn(__fmul_rn(-0.5f * v, r), r, 1.5f));
    }
    bSR[j] = make_int2(S, __float_as_int(rs));
    if (self) {
      const bool ok = rs != 0.f;
      const unsigned bits = __ballot_sync(0xffffffffu, ok);  // kCX is a multiple of 32
      if (x < a.W) {
        const float gi = (float)self_img[(size_t)y * a.W + x] + (ok ? 0.f : kGuideFlag);
        (SIDE == 0 ? a.gpadL : a.gpadR)[(size_t)(y + a.R) * a.Wg + x + a.R] = gi;
      }
      if ((j & 31) == 0 && x < a.W) (SIDE == 0 ? a.bitsL : a.bitsR)[(size_t)y * a.Wb + x / 32] = bits;
    }
  }
  __syncthreads();
  // 3. values: warp <-> 8 consecutive pixels, lane <-> disparity pair.  The 3x3 dot
  // product is the sum of three column dots (one DP4A each); along the 8 pixels a
  // column dot is shared by three blocks, so 10 DP4A give 8 dot products.
  const int lane32 = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int LPR = 32 / NRUN;         // lanes per run
  const int lane = lane32 % LPR;         // disparity pair within the run
  float* vol = SIDE == 0 ? a.volL : a.volR;
  constexpr int PPW = vol::kCX / 8;      // pixels per run
  const int xw = (warp * NRUN + lane32 / LPR) * PPW;
  const int npx = min(PPW, a.W - (x0 + xw));
  if (npx <= 0) return;
  float* vp = vol + vol_at(y + a.R - a.vbase, 0, x0 + xw + a.R, a.nblk, a.Wv) + 2 * lane;
  const size_t bstride = (size_t)a.Wv * kDB;  // next d-block of the same pixel
  const uint32_t* cPs = cP + xw;               // self column of block xw + m: cPs[m .. m+2]
  const int2* sSR = bSR + xw;
  const int2* oSR = bSR + kCX;
  for (int b = 0; b < a.nblk; ++b) {
    const int di0 = b * kDB + 2 * lane;
    const bool pad0 = di0 >= a.D, pad1 = di0 + 1 >= a.D;
    // other-image block index of (pixel xw + m, disparity index di0 + k): jo + m -+ k
    const int jo = SIDE == 0 ? xw + dspan - 1 - di0 : xw + di0;
    const uint32_t* cPo = cP + ncs + jo;  // other column of (m, k=0): cPo[m], k=1: cPo[m -+ 1]
    uint32_t po[PPW + 3];                 // other columns jo + m - 1 (SIDE 0) / jo + m (SIDE 1)
#pragma unroll
    for (int m = 0; m < PPW + 3; ++m) po[m] = cPo[SIDE == 0 ? m - 1 : m];
    int cd0[PPW + 2], cd1[PPW + 2];       // column dots for k = 0, 1
#pragma unroll
    for (int m = 0; m < PPW + 2; ++m) {
      const uint32_t ps = cPs[m];
      cd0[m] = (int)__dp4a(ps, SIDE == 0 ? po[m + 1] : po[m], 0u);
      cd1[m] = (int)__dp4a(ps, SIDE == 0 ? po[m] : po[m + 1], 0u);
    }
    float* vb = vp + (size_t)b * bstride;
    // one pixel's two values (u = pixel within the warp's run)
    auto value2 = [&](int u) {
      const int2 ss = sSR[u];
      const float rsf = __int_as_float(ss.y);
      float o[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int2 so = oSR[SIDE == 0 ? jo + u - k : jo + u + k];
        const float rof = __int_as_float(so.y);
        const int dot = k == 0 ? cd0[u] + cd0[u + 1] + cd0[u + 2] : cd1[u] + cd1[u + 1] + cd1[u + 2];
        const int N = 9 * dot - ss.x * so.x;
        // (V_l V_r)^{-1/2} as one product (commutative, so both sides get the same
        // bits); zero iff either block is undefined (each factor >= 8.8e-4)
        const float P = __fmul_rn(rsf, rof);
        const float c = fminf(1.0f, fmaxf(-1.0f, __fmul_rn((float)N, P)));  // clamp (R#8)
        o[k] = P != 0.f ? c : kUndef;
      }
      if (pad0) o[0] = kUndef;  // padded disparity slots of the last block
      if (pad1) o[1] = kUndef;
      *reinterpret_cast<float2*>(vb + u * kDB) = make_float2(o[0], o[1]);
    };
    if (npx == PPW) {  // every CTA column but the frame's last: no per-pixel guard
#pragma unroll
      for (int u = 0; u < PPW; ++u) value2(u);
    } else {
#pragma unroll
      for (int u = 0; u < PPW; ++u) {
        if (u >= npx) break;
        value2(u);
      }
    }
  }
}

__host__ __device__ constexpr size_t cost_smem_bytes(int nblk, int nrun = 1) {
  return (size_t)(kCX * nrun + 2 + kCX * nrun + nblk * kDB + 1) * 12 + 8 +
         (size_t)(kCX * nrun + kCX * nrun + nblk * kDB - 1) * 8;
}
constexpr bool cost_runs4(int D) { return D <= 16; }  // k_cost<4>: 8 lanes x 2 disparities per run

// grid: (ceil(W/kCX), r1-r0, 2 sides); block 256 = 8 warps; warp <-> pixel, lane <-> d pair.
// k_cost is issue-bound (~75 % issue active, the rest barrier / load stalls): a
// 48-register cap puts 5 CTAs (40 warps) on an SM instead of 4 at 59 registers
// (A/B: k_cost 30.4 -> 28.6 us at Teddy; 6 CTAs at 40 registers: 28.7 us, spills)
#ifndef FBS_KCOST_MINB
#define FBS_KCOST_MINB 5
#endif
template <int NRUN>
__global__ void __launch_bounds__(256, FBS_KCOST_MINB) k_cost(CostArgs a) {
  extern __shared__ __align__(16) unsigned char csm[];
  pdl_trigger();  // k_agg may be scheduled now; it waits for our results in pdl_wait()
  if (blockIdx.z == 0) cost_side<0, NRUN>(a, csm);
  else cost_side<1, NRUN>(a, csm);
}

// fill a buffer with a float value (volume margins = kUndef)
__global__ void k_fill(float* p, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// padded volume -> [H][W][D] export (debug), undefined -> kSent
__global__ void k_export_vol(const float* __restrict__ vol, int W, int H, int D, int nblk, int Wv, int R,
                             float* __restrict__ out) {
  const size_t n = (size_t)W * H * D;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int di = (int)(i % D);
    const size_t p = i / D;
    const int x = (int)(p % W), y = (int)(p / W);
    const float c = vol[vol_at(y + R, di / kDB, x + R, nblk, Wv) + di % kDB];
    out[i] = __float_as_uint(c) == 0x80000000u ? kSent : c;
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

// rows [r0, r1): out[(y - r0)*W + x]; aggregated costs from the left pass's
// [H][nblk][W][64] store
template <bool SCATTER>
__global__ void k_finalize(const int32_t* __restrict__ dl, const int32_t* __restrict__ dr,
                           const float* __restrict__ aggL, const float4* __restrict__ agg3, int nblk, int W,
                           int r0, int r1, int d_min, int d_max, int abase, float* __restrict__ out,
                           const short2* __restrict__ rng, const OutSet os) {
  pdl_wait();  // k_agg's maps
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = r0 + blockIdx.y;
  if (x >= W || y >= r1) return;
  const size_t p = (size_t)y * W + x;
  const int d = dl[p];
  int e = -1;
  if (d >= 0 && x - d >= 0) e = dr[p - d];
  float c0 = kSent, cm = kSent, cp = kSent;
  if (d >= 0 && agg3) {  // compact record written by k_agg
    const float4 v = agg3[p];
    cm = v.x; c0 = v.y; cp = v.z;
  } else if (d >= 0) {
    auto at = [&](int di) { return aggL[(((size_t)(y - abase) * nblk + di / kDB) * W + x) * kDB + di % kDB]; };
    const int di = d - d_min;
    const short2 r = rng ? rng[p] : make_short2(-32768, 32767);  // RANGED: R#33
    c0 = at(di);
    if (d > d_min && d - 1 >= r.x) cm = at(di - 1);
    if (d < d_max && d + 1 <= r.y) cp = at(di + 1);
  }
  const float v = finalize_pixel(d, e, c0, cm, cp, d_min, d_max);
  if constexpr (!SCATTER) {
    out[(size_t)(y - r0) * W + x] = v;
  } else {
    for (int k = 0; k < os.n; ++k) os.p[k][p] = v;  // band scatter: frame coordinates
  }
}

// Sparse search range (NEXT-4, R#31): feature points = valid seeds (>= 0) of a seed
// disparity map; per frame-anchored T x T tile the range [floor(min) - m, ceil(max) + m]
// of its seeds (left image) and of the forward-warped seeds (right image,
// x_r = x - round(s)), clipped to [d_min, d_max]; tiles without seeds: full range.
constexpr int kRangeTile = 16;
__global__ void k_range_init(int* tiles, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) tiles[i] = (i & 1) ? -0x7fffffff : 0x7fffffff;  // (min, max) pairs
}
__global__ void k_range_seeds(const float* __restrict__ seed, int W, int H, int tx, int* tl, int* tr) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= W) return;
  const float s = seed[(size_t)y * W + x];
  if (!(s >= 0.f)) return;
  const int lo = (int)floorf(s), hi = (int)ceilf(s);
  int* t = tl + 2 * ((y / kRangeTile) * tx + x / kRangeTile);
  atomicMin(t, lo);
  atomicMax(t + 1, hi);
  const int xr = x - (int)floorf(s + 0.5f);
  if (xr >= 0 && xr < W) {
    int* u = tr + 2 * ((y / kRangeTile) * tx + xr / kRangeTile);
    atomicMin(u, lo);
    atomicMax(u + 1, hi);
  }
}
__global__ void k_range_expand(const int* __restrict__ tl, const int* __restrict__ tr, int W, int H, int tx,
                               int d_min, int d_max, int margin, short2* __restrict__ rl, short2* __restrict__ rr) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= W) return;
  const int t = 2 * ((y / kRangeTile) * tx + x / kRangeTile);
  const int* src[2] = {tl + t, tr + t};
  short2* dst[2] = {rl, rr};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int a = src[k][0], b = src[k][1];
    dst[k][(size_t)y * W + x] = a > b ? make_short2((short)d_min, (short)d_max)
                                      : make_short2((short)max(d_min, a - margin), (short)min(d_max, b + margin));
  }
}

// KEYS: the left record (c(d*-1), c(d*), c(d*+1)) of every pixel of rows [r0, r1)
// for the disparity-range split (same sources and rules as k_finalize; the
// neighbours come from the handle's whole range, which includes one disparity
// beyond each end of the competing range).
__global__ void k_records(const int32_t* __restrict__ dl, const float* __restrict__ aggL,
                          const float4* __restrict__ agg3, int nblk, int W, int r0, int r1, int d_min, int d_max,
                          int abase, float4* __restrict__ rec) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = r0 + blockIdx.y;
  if (x >= W || y >= r1) return;
  const size_t p = (size_t)y * W + x;
  const int d = dl[p];
  float c0 = kSent, cm = kSent, cp = kSent;
  if (d >= 0 && agg3) {
    const float4 v = agg3[p];
    cm = v.x; c0 = v.y; cp = v.z;
  } else if (d >= 0) {
    auto at = [&](int di) { return aggL[(((size_t)(y - abase) * nblk + di / kDB) * W + x) * kDB + di % kDB]; };
    const int di = d - d_min;
    c0 = at(di);
    if (d > d_min) cm = at(di - 1);
    if (d < d_max) cp = at(di + 1);
  }
  rec[p] = make_float4(cm, c0, cp, 0.f);
}

// LRC + subpixel from (reduced) keys and records: the disparity-range split's last
// step; identical rules to k_finalize on the global range [d_min, d_max].
__global__ void k_finalize_keys(const unsigned long long* __restrict__ kl, const unsigned long long* __restrict__ kr,
                                const float4* __restrict__ rec, int W, int H, int d_min, int d_max,
                                float* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= W || y >= H) return;
  const size_t p = (size_t)y * W + x;
  const unsigned long long k = kl[p];
  const int d = k ? (int)(0xffffffffu - (unsigned)(k & 0xffffffffu)) : -1;
  int e = -1;
  if (d >= 0 && x - d >= 0) {
    const unsigned long long ke = kr[p - d];
    e = ke ? (int)(0xffffffffu - (unsigned)(ke & 0xffffffffu)) : -1;
  }
  float c0 = kSent, cm = kSent, cp = kSent;
  if (d >= 0) {
    const float4 v = rec[p];
    cm = v.x; c0 = v.y; cp = v.z;
  }
  out[p] = finalize_pixel(d, e, c0, cm, cp, d_min, d_max);
}

// left aggregated store -> [H][W][D] export (debug)
__global__ void k_export_agg(const float* __restrict__ aggL, int W, int H, int D, int nblk,
                             float* __restrict__ out) {
  const size_t n = (size_t)W * H * D;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int di = (int)(i % D);
    const size_t p = i / D;
    const int x = (int)(p % W), y = (int)(p / W);
    out[i] = aggL[(((size_t)y * nblk + di / kDB) * W + x) * kDB + di % kDB];
  }
}

// ---------------------------------------------------------------------------
// Stage 3: fused bilateral aggregation + WTA, both sides in one grid.
//
// Undefined costs are stored as -0.0f (a defined NCC is never -0.0: N = 0 gives
// +0.0), so they add nothing to the numerator Σ w c whatever their weight; the
// denominator Σ w over the defined taps is the only place validity enters.
// Per (CTA tile, d-block) the denominator takes one of three exact forms:
//   FAST     every tap defined but for the guide's own blocks (folded into w'):
//            den = Σ_q w'(p,q), d-independent
//   EDGE     additionally only the frame edge cuts taps off (x - d < 1 on the
//            left pass, x + d > W-2 on the right): den = a per-pixel suffix /
//            prefix sum of the window's column sums, indexed by d
//   GENERAL  the other image has textureless blocks in range: explicit den by
//            FFMA2 over the validity of every tap
// Tiles are anchored at multiples of the tile size in frame coordinates, so the
// form a pixel gets never depends on the row band being computed.
struct AggArgs {
  int W, H, D, d_min, d_max, nblk, Wv, r0, r1;  // output rows [r0, r1)
  int vbase, abase;               // frame rows of volume row R and of aggL row 0 (0 for full-frame handles)
  int ty0;                       // first tile row (tiles anchored at multiples of the tile height)
  const float *volL, *volR;      // cost volumes (padded layout)
  const float *gpadL, *gpadR;    // padded guide images (Eq.(8); the right image guides the right volume, R#11)
  int Wg;
  const uint32_t *bitsL, *bitsR; // block-defined masks, bit-packed [H][Wb]
  int Wb;
  int32_t *dL, *dR;              // WTA maps [H][W]
  float* aggL;                   // left aggregated costs, [H][nblk][W][64] (read by k_finalize)
  float4* agg3;                  // if set (one d-block, no export): only (c(d*-1), c(d*), c(d*+1)) per
                                 // left pixel, [H][W] float4, instead of aggL
  float* exportR;                // optional [H][W][D] right aggregated volume (debug)
  // KEYS instantiation (disparity-range split, NEXT-3): only local disparity indices
  // [c_lo, c_hi] compete in the WTA; the per-pixel keys (global d) are written out
  int c_lo, c_hi;
  unsigned long long* keys_out[2];
  // RANGED instantiation (sparse search range, NEXT-4): per-pixel suggested range
  // (lo, hi) of the left / right image, short2 [H][W]; only those d compete
  const short2* ranges[2];
  unsigned long long* tile_stats;  // optional [4]: FAST / EDGE / GENERAL / EMPTY (sub-tile, d-block) counts
  float cd[(2 * kMaxRadius + 1) * (2 * kMaxRadius + 1)];  // log2 ω_d = -log2(e)(dx²+dy²)/γ_d², Eq.(7)
  float nkr;                                               // -log2(e)/γ_r²: log2 ω_r = nkr Δ², Eq.(8)
};

enum { kFast = 0, kEdge = 1, kGeneral = 2, kEmpty = 3 };


__device__ __forceinline__ void ffma2(float2& acc, float w, float2 c) {
  unsigned long long A, B = *reinterpret_cast<unsigned long long*>(&c);
  unsigned long long C = *reinterpret_cast<unsigned long long*>(&acc);
  asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(w));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
  acc = *reinterpret_cast<float2*>(&C);
}

__device__ __forceinline__ bool is_undef(float c) { return __float_as_uint(c) == 0x80000000u; }

template <int R>
struct AggSmem {
  static constexpr int K1 = 2 * R + 1;
  static constexpr int WPW = AggGeom<R>::PY * K1 * K1 * kPX;  // weights per warp
  static constexpr int NW = AggGeom<R>::NW;
  static constexpr int GW = (kTX + 2 * R + 3) / 4 * 4, GH = AggGeom<R>::TY + 2 * R;
  // shared-memory row stride of the guide tile: the prologue's 24 lanes read
  // rows py (stride GWS) x columns px; a stride = 24 (mod 32) would put rows
  // py and py + 4 in the same banks
  static constexpr int GWS = GW % 32 == 24 ? GW + 4 : GW;
  // single-d-block frames keep the left pass's aggregated costs on chip: row py of
  // the sub-tile ([px][64]) goes into its own weight row once that row is dead
  // (room when K1² >= 64), else into a separate buffer
  static constexpr bool kAlias = K1 * K1 >= kDB;
  float w[NW][WPW];                                 // [warp][py][dy][dx][px]
  float val[NW][kAlias ? 4 : AggGeom<R>::PY * kPX * kDB];
  float rinv[NW][32];                               // 1 / Σ_q w'(p,q), 0 if none
  float cs[NW][32][K1 + 1];                         // EDGE: 1 / suffix (left) or prefix (right) column sums
  float g[GH * GWS];                                // guide tile (padded image values, see kGuideFlag)
  uint32_t cwb[NW][2][AggGeom<R>::CWS];             // classification words: current / next d-block
  short2 rng[AggGeom<R>::TY][kTX];                  // RANGED: the tile's per-pixel suggested ranges
  int rlo, rhi;                                     // RANGED: their union
};

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

// Denominator form of one warp sub-tile (origin sx, sy; 4 x PY pixels) for d-block
// b, exact and conservative: EDGE if the frame edge cuts taps off, GENERAL if the
// other image has an undefined block anywhere in the shifted range.  The range
// spans at most 16 rows x 4 mask words (slot 4 row + word), two per lane: cw_load fetches them into
// shared memory (cp.async, one d-block ahead), cw_classify consumes them.
// Sub-tiles are anchored at multiples of (4, PY) in frame coordinates, so the
// form a pixel gets never depends on the row band being computed.
template <int R>
struct CwRange {
  int qy0, lo, hi, edge, nw, rows, w0;
  __device__ __forceinline__ CwRange(const AggArgs& a, int side, int sx, int sy, int b) {
    qy0 = max(sy - R, 1);
    const int qy1 = min(sy + AggGeom<R>::PY - 1 + R, a.H - 2);
    const int qx0 = max(sx - R, 1), qx1 = min(sx + kPX - 1 + R, a.W - 2);
    const int d_lo = a.d_min + b * kDB, d_hi = min(d_lo + kDB - 1, a.d_max);
    if (side == 0) { lo = qx0 - d_hi; hi = qx1 - d_lo; edge = lo < 1; lo = max(lo, 1); }
    else { lo = qx0 + d_lo; hi = qx1 + d_hi; edge = hi > a.W - 2; hi = min(hi, a.W - 2); }
    rows = (qy0 <= qy1 && qx0 <= qx1 && lo <= hi) ? qy1 - qy0 + 1 : 0;
    w0 = lo >> 5;
    nw = rows ? (hi >> 5) - w0 + 1 : 0;
  }
};
template <int R>
__device__ __forceinline__ void cw_load(const AggArgs& a, int side, int sx, int sy, int b, int lane,
                                        uint32_t* cwb) {
  const CwRange<R> g(a, side, sx, sy, b);
  const uint32_t* bits = side == 0 ? a.bitsR : a.bitsL;
#pragma unroll
  for (int k = 0; k < AggGeom<R>::CWS / 32; ++k) {  // slot i = 4 row + word (no division)
    const int i = lane + 32 * k, row = i >> 2, wd = i & 3;
    if (row < g.rows && wd < g.nw) cp_async4(cwb + i, bits + (size_t)(g.qy0 + row) * a.Wb + g.w0 + wd);
  }
}
template <int R>
__device__ __forceinline__ int cw_classify(const AggArgs& a, int side, int sx, int sy, int b, int lane,
                                           const uint32_t* cwb) {
  const CwRange<R> g(a, side, sx, sy, b);
  bool tex = false;
#pragma unroll
  for (int k = 0; k < AggGeom<R>::CWS / 32; ++k) {
    const int i = lane + 32 * k, row = i >> 2, wd = i & 3;
    if (row < g.rows && wd < g.nw) {
      const int wi = g.w0 + wd;
      uint32_t m = 0xffffffffu;
      if (wi == g.w0) m &= 0xffffffffu << (g.lo & 31);
      if (wi == (g.hi >> 5)) m &= 0xffffffffu >> (31 - (g.hi & 31));
      tex |= (~cwb[i] & m) != 0u;
    }
  }
  if (__any_sync(0xffffffffu, tex)) return kGeneral;
  return g.edge ? kEdge : kFast;
}

// EMPTY (a special case of GENERAL, tested only there): no block of the other
// image in range is defined, so every cost any window of the sub-tile reads at
// this d-block is undefined and every aggregated cost is SENT, exactly.  (Kept
// out of cw_classify: folding it in changed the code generated for the FAST
// stream and cost 5 % at Teddy.)
template <int R>
__device__ __forceinline__ bool cw_empty(const AggArgs& a, int side, int sx, int sy, int b, int lane,
                                         const uint32_t* cwb) {
  const CwRange<R> g(a, side, sx, sy, b);
  bool def = false;
#pragma unroll
  for (int k = 0; k < AggGeom<R>::CWS / 32; ++k) {
    const int i = lane + 32 * k, row = i >> 2, wd = i & 3;
    if (row < g.rows && wd < g.nw) {
      const int wi = g.w0 + wd;
      uint32_t m = 0xffffffffu;
      if (wi == g.w0) m &= 0xffffffffu << (g.lo & 31);
      if (wi == (g.hi >> 5)) m &= 0xffffffffu >> (31 - (g.hi & 31));
      def |= (cwb[i] & m) != 0u;
    }
  }
  return g.rows > 0 && !__any_sync(0xffffffffu, def);
}

// 1/x for x > 0: MUFU reciprocal + one Newton step (<= 1 ulp; no slow path)
__device__ __forceinline__ float rcp_nr(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return __fmul_rn(r, __fmaf_rn(-x, r, 2.0f));
}

// Weights w' = 2^(cd + nkr Δ²) (Eq.(7)(8); Δ² exact, one MUFU.EX2 per tap) of the two
// adjacent taps (dy, dx), (dy, dx+1) of a prologue row, their arithmetic as f32x2 (the
// same per-element roundings as the scalar form, half the issue slots), and the taps'
// column sums advanced as one pair.
__device__ __forceinline__ void tap_pair(float g0, float g1, float gp, float nkr, float cd0, float cd1,
                                         float& w0, float& w1, float& col0, float& col1) {
  unsigned long long G, P, D2, NK, CD, C, CL, WP;
  asm("mov.b64 %0, {%1, %2};" : "=l"(G) : "f"(g0), "f"(g1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(P) : "f"(-gp));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(D2) : "l"(G), "l"(P));
  asm("mul.rn.f32x2 %0, %0, %0;" : "+l"(D2));
  asm("mov.b64 %0, {%1, %1};" : "=l"(NK) : "f"(nkr));
  asm("mov.b64 %0, {%1, %2};" : "=l"(CD) : "f"(cd0), "f"(cd1));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(C) : "l"(D2), "l"(NK), "l"(CD));
  float c0, c1;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(C));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(w0) : "f"(c0));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(w1) : "f"(c1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(CL) : "f"(col0), "f"(col1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(WP) : "f"(w0), "f"(w1));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(CL) : "l"(WP));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(col0), "=f"(col1) : "l"(CL));
}
__device__ __forceinline__ float tap_one(float g, float gp, float nkr, float cd, float& col) {
  const float dd = __fsub_rn(g, gp);
  float w;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(w) : "f"(__fmaf_rn(__fmul_rn(dd, dd), nkr, cd)));
  col = __fadd_rn(col, w);
  return w;
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

// Cost rows of the stream.  The first kPX columns of row r+1 (all that its first
// dx step needs) are loaded while row r is consumed; the rest of a row is loaded
// at its start (registers allow no more).
template <int R, int r, int NR, int NPY>
struct Rows4 {
  static __device__ __forceinline__ void run(const float* __restrict__ vb, size_t rowstride,
                                             const float* __restrict__ wsm, float4 (&head)[kPX],
                                             float2 (&num)[NPY][kPX][2]) {
    constexpr int NC = kPX + 2 * R;
    float4 c[NC];
    const float* rp = vb + (size_t)r * rowstride;
#pragma unroll
    for (int j = 0; j < kPX; ++j) c[j] = head[j];
#pragma unroll
    for (int j = kPX; j < NC; ++j) c[j] = __ldg(reinterpret_cast<const float4*>(rp + j * kDB));
    if constexpr (r + 1 < NR) {
#pragma unroll
      for (int j = 0; j < kPX; ++j) head[j] = __ldg(reinterpret_cast<const float4*>(rp + rowstride + j * kDB));
    }
    row_fma4<R, NPY, r>(c, wsm, num);
    Rows4<R, r + 1, NR, NPY>::run(vb, rowstride, wsm, head, num);
  }
};
template <int R, int NR, int NPY>
struct Rows4<R, NR, NR, NPY> {
  static __device__ __forceinline__ void run(const float*, size_t, const float*, float4 (&)[kPX],
                                             float2 (&)[NPY][kPX][2]) {}
};

// Numerator for the half-warp's 4 x NPY pixels (undefined c = -0.0 adds nothing).
template <int R, int NPY>
__device__ __forceinline__ void agg_num4(const float* __restrict__ vb, size_t rowstride,
                                         const float* __restrict__ wsm, float2 (&num)[NPY][kPX][2]) {
#pragma unroll
  for (int py = 0; py < NPY; ++py)
#pragma unroll
    for (int px = 0; px < kPX; ++px) num[py][px][0] = num[py][px][1] = make_float2(0.f, 0.f);
  if constexpr (AggGeom<R>::kRolled) {
    static_assert(NPY == 1, "the rolled stream feeds one output row per cost row");
    constexpr int K1 = 2 * R + 1, NC = kPX + 2 * R;
#pragma unroll 1
    for (int r = 0; r < K1; ++r) {  // cost row r = window row dy (same order as the unrolled form)
      const float* rp = vb + (size_t)r * rowstride;
      float4 c[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) c[j] = __ldg(reinterpret_cast<const float4*>(rp + j * kDB));
      const float* wr = wsm + r * K1 * kPX;
#pragma unroll
      for (int dx = 0; dx < K1; ++dx) {
        const float4 w = reinterpret_cast<const float4*>(wr)[dx];
        const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int px = 0; px < kPX; ++px) {
          const float4 cc = c[dx + px];
          ffma2(num[0][px][0], wv[px], make_float2(cc.x, cc.y));
          ffma2(num[0][px][1], wv[px], make_float2(cc.z, cc.w));
        }
      }
    }
    return;
  }
  float4 head[kPX];
#pragma unroll
  for (int j = 0; j < kPX; ++j) head[j] = __ldg(reinterpret_cast<const float4*>(vb + j * kDB));
  Rows4<R, 0, NPY + 2 * R, NPY>::run(vb, rowstride, wsm, head, num);
}

// GENERAL: explicit num and den of one output row (wrow = its weights),
// cost rows 0..2R of that row's window, compact runtime loop.
template <int R>
__device__ __forceinline__ void agg_num_den_row4(const float* __restrict__ vb, size_t rowstride,
                                                 const float* __restrict__ wrow, float2 (&num)[kPX][2],
                                                 float2 (&den)[kPX][2]) {
  constexpr int K1 = 2 * R + 1;
  constexpr int NC = kPX + 2 * R;
#pragma unroll
  for (int px = 0; px < kPX; ++px) num[px][0] = num[px][1] = den[px][0] = den[px][1] = make_float2(0.f, 0.f);
#pragma unroll 1
  for (int dy = 0; dy < K1; ++dy) {
    float4 c[NC];
    const float* rp = vb + (size_t)dy * rowstride;
#pragma unroll
    for (int j = 0; j < NC; ++j) c[j] = __ldg(reinterpret_cast<const float4*>(rp + j * kDB));
#pragma unroll
    for (int dx = 0; dx < K1; ++dx) {
      const float4 w = reinterpret_cast<const float4*>(wrow + dy * K1 * kPX)[dx];
      const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int px = 0; px < kPX; ++px) {
        const float4 cc = c[dx + px];
        const float4 vv = make_float4(is_undef(cc.x) ? 0.f : 1.f, is_undef(cc.y) ? 0.f : 1.f,
                                      is_undef(cc.z) ? 0.f : 1.f, is_undef(cc.w) ? 0.f : 1.f);
        ffma2(num[px][0], wv[px], make_float2(cc.x, cc.y));
        ffma2(num[px][1], wv[px], make_float2(cc.z, cc.w));
        ffma2(den[px][0], wv[px], make_float2(vv.x, vv.y));
        ffma2(den[px][1], wv[px], make_float2(vv.z, vv.w));
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

// grid: (ceil(W/kTX), tile rows, 2 sides); block AggGeom<R>::THREADS (warps of 4 x PY sub-tiles).
// EMPTY: whether GENERAL units test for the EMPTY special case (the production
// instantiation does: KITTI +22.5 %, Teddy -0.6 %).  Bit-identical
// results either way.
// EXPORT: the debug export of the right aggregated volume is compiled in (its
// store loop alone costs the production kernel ~1 %).
// KEYS: disparity-range split (fbs_compute_keys); RANGED: sparse search range
// (fbs_compute_ranged).
template <int R, bool EMPTY, bool EXPORT, bool KEYS = false, bool RANGED = false>
__global__ void __launch_bounds__(AggGeom<R>::THREADS, AggGeom<R>::MINB) k_agg(const AggArgs a) {
  constexpr int kPY = AggGeom<R>::PY;
  constexpr int kTY = AggGeom<R>::TY;
  constexpr int kThreads = AggGeom<R>::THREADS;
  extern __shared__ __align__(16) unsigned char smraw[];
  AggSmem<R>& sm = *reinterpret_cast<AggSmem<R>*>(smraw);
  constexpr int K1 = 2 * R + 1;
  constexpr int GW = AggSmem<R>::GW, GH = AggSmem<R>::GH, GWS = AggSmem<R>::GWS;
  // Dispatch order (blocks start in linear-index order): the tiles wholly inside the
  // frame first, both sides, then the partial tiles of the last tile column and row.
  // Warps of a partial tile that lie wholly outside the frame skip their work, so the
  // last wave is made of cheap CTAs instead of full ones.
  int tx, ty, side;  // side 0: left volume / left guide, 1: right
  {
    const int ntx = gridDim.x, nty = gridDim.y;
    const int lin = blockIdx.x + ntx * (blockIdx.y + nty * blockIdx.z);
    const int fx = a.W / kTX;                                // tile columns wholly inside
    const int fy = min(nty, max(0, a.H / kTY - a.ty0));      // tile rows wholly inside
    const int nfull = fx * fy, npart = ntx * nty - nfull;
    if (lin < 2 * nfull) {
      side = lin / nfull;
      const int t = lin - side * nfull;
      tx = t % fx;
      ty = t / fx;
    } else {
      const int l2 = lin - 2 * nfull;
      side = l2 / npart;
      int t = l2 - side * npart;
      const int ncol = fx < ntx ? fy : 0;  // the last column's tiles within the full rows
      if (t < ncol) {
        tx = fx;
        ty = t;
      } else {
        t -= ncol;
        tx = t % ntx;
        ty = fy + t / ntx;
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = tx * kTX, y0 = (a.ty0 + ty) * kTY;
  const int wx = (warp % kNWX) * kPX, wy = (warp / kNWX) * kPY;
  const int sx = x0 + wx, sy = y0 + wy;

  pdl_trigger();
  pdl_wait();  // everything below reads k_cost's outputs

  // RANGED: the union of the tile's suggested ranges decides which d-blocks run
  int b_lo = 0, b_hi = a.nblk - 1;
  if constexpr (RANGED) {
    if (threadIdx.x == 0) { sm.rlo = 0x7fffffff; sm.rhi = -0x7fffffff; }
    __syncthreads();
    for (int i = threadIdx.x; i < kTY * kTX; i += kThreads) {
      const int px = i % kTX, py = i / kTX, x = x0 + px, y = y0 + py;
      short2 r = make_short2(32767, -32768);  // outside the frame: no candidates
      if (x < a.W && y < a.H) {
        r = a.ranges[side][(size_t)y * a.W + x];
        r.x = (short)max((int)r.x, a.d_min);
        r.y = (short)min((int)r.y, a.d_max);
        if (r.x <= r.y) { atomicMin(&sm.rlo, (int)r.x); atomicMax(&sm.rhi, (int)r.y); }
      }
      sm.rng[py][px] = r;
    }
    __syncthreads();
    if (sm.rlo <= sm.rhi) {
      b_lo = (sm.rlo - a.d_min) / kDB;
      b_hi = (sm.rhi - a.d_min) / kDB;
    } else {
      b_lo = 0; b_hi = -1;  // no candidate disparity in the tile
    }
  }
  {  // guide tile (padded rows y0.., columns x0..: 16-B aligned) and the first
     // d-block's classification words, all in flight at once
    const float* src = (side == 0 ? a.gpadL : a.gpadR) + (size_t)y0 * a.Wg + x0;
    for (int c = threadIdx.x; c < GH * (GW / 4); c += kThreads) {
      const int row = c / (GW / 4), q = c % (GW / 4);
      cp_async16(&sm.g[row * GWS + 4 * q], src + (size_t)row * a.Wg + 4 * q);
    }
    if (b_lo <= b_hi) cw_load<R>(a, side, sx, sy, b_lo, lane, sm.cwb[warp][b_lo & 1]);
    cp_async_commit();
    cp_async_wait_all();
  }
  __syncthreads();

  // ---- weights w'(p,q) = def_self(q) · ω_d(q-p) · ω_r(|i(q) - i(p)|), Eq.(6)-(8),
  //      their sum, and the window's column sums (EDGE denominators) ----
  const bool live = sx < a.W && sy < a.H;  // warp-uniform: the sub-tile has a pixel in the frame
  if (live && lane < kPX * kPY) {
    const int py = lane / kPX, px = lane % kPX;
    // pixels outside the frame read the margin (kGuideUndef): their outputs are discarded
    float* wsm = sm.w[warp];
    const float* gq = sm.g + (wy + py) * GWS + (wx + px);
    const float gc = gq[R * GWS + R];                     // i(p) (+ kGuideFlag if undefined)
    const float gp = gc >= kGuideFlag ? __fsub_rn(gc, kGuideFlag) : gc;
    float wsum = 0.f;
    float col[K1];
#pragma unroll
    for (int dx = 0; dx < K1; ++dx) col[dx] = 0.f;
    // Loads of a chunk of CH tap rows are issued before any store of that chunk:
    // the weight stores may alias the guide/LUT loads as far as ptxas can tell,
    // so interleaving them would serialise every LDS -> LDS -> STS chain.
    constexpr int CH = (K1 * K1 <= 64) ? K1 : (64 / K1 > 0 ? 64 / K1 : 1);
    constexpr int kChunkUnroll = AggGeom<R>::kRolled ? 1 : 16;  // ρ >= 7: chunks in a loop (code size)
#pragma unroll kChunkUnroll
    for (int dy0 = 0; dy0 < K1; dy0 += CH) {
      constexpr int NB = CH * K1;
      float gv[NB];
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int dy = dy0 + t / K1, dx = t % K1;
        gv[t] = dy < K1 ? gq[dy * GWS + dx] : 0.f;
      }
      // ω_d ω_r = 2^(cd(dx,dy) + nkr Δ²), adjacent taps of a row in pairs
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int dy = dy0 + t / K1, dx = t % K1;
        if (dy >= K1 || (dx & 1)) continue;
        float* wr = wsm + ((py * K1 + dy) * K1 + dx) * kPX + px;
        if (dx + 1 < K1) {
          float w0, w1;
          tap_pair(gv[t], gv[t + 1], gp, a.nkr, a.cd[dy * K1 + dx], a.cd[dy * K1 + dx + 1], w0, w1, col[dx],
                   col[dx + 1]);
          wr[0] = w0;
          wr[kPX] = w1;
        } else {
          wr[0] = tap_one(gv[t], gp, a.nkr, a.cd[dy * K1 + dx], col[dx]);
        }
      }
    }
#pragma unroll
    for (int dx = 0; dx < K1; ++dx) wsum = __fadd_rn(wsum, col[dx]);  // Σ w', column-major
    sm.rinv[warp][lane] = wsum > 0.f ? rcp_nr(wsum) : 0.f;
    // EDGE tables hold reciprocals: left pass, taps with dx >= m defined -> 1 / suffix sum;
    // right pass, dx < m -> 1 / prefix sum (0 when no tap is defined)
    float* cs = sm.cs[warp][lane];
    float acc = 0.f;
    if (side == 0) {
      cs[K1] = 0.f;
#pragma unroll
      for (int dx = K1 - 1; dx >= 0; --dx) {
        acc = __fadd_rn(acc, col[dx]);
        cs[dx] = acc > 0.f ? rcp_nr(acc) : 0.f;
      }
    } else {
      cs[0] = 0.f;
#pragma unroll
      for (int dx = 0; dx < K1; ++dx) {
        acc = __fadd_rn(acc, col[dx]);
        cs[dx + 1] = acc > 0.f ? rcp_nr(acc) : 0.f;
      }
    }
  }
  __syncwarp();

  const float* vol = side == 0 ? a.volL : a.volR;
  const size_t rowstride = (size_t)a.nblk * a.Wv * kDB;
  constexpr int HPY = AggGeom<R>::HPY;
  constexpr int RS = K1 * K1 * kPX;                 // weights per output row
  const int half = lane >> 4, dq = lane & 15;       // half-warp, disparity quad within the block
  const int py0 = half * HPY;                       // first output row of this half in the sub-tile
  const float* wsm = sm.w[warp] + py0 * RS;
  // on-chip aggregated costs of half-row pyl (compact mode): [px][64]
  auto vrow = [&](int pyl) -> float* {
    return AggSmem<R>::kAlias ? sm.w[warp] + (py0 + pyl) * RS : sm.val[warp] + (py0 + pyl) * kPX * kDB;
  };
  unsigned long long best = 0ull;  // running best key of slot (lane & 15) of this half
  for (int b = b_lo; b <= b_hi; ++b) {
    // volume row (sy + py0 - R + r) + R = sy + py0 + r; column (sx - R + j) + R = sx + j
    const float* vb = vol + vol_at(sy + py0 - a.vbase, b, sx, a.nblk, a.Wv) + 4 * dq;
    if (b > b_lo) {  // this d-block's words (issued one d-block ahead)
      cp_async_wait_all();
      // one CTA barrier per d-block keeps the warps in lockstep: warps that drift
      // apart run different parts of the unrolled FMA stream, which is larger than
      // the instruction cache (measured: MB2014 aggregation 14.3 -> 13.0 ms)
      __syncthreads();
    }
    if (!live) continue;  // (still meets the per-d-block barriers)
    const int cls = cw_classify<R>(a, side, sx, sy, b, lane, sm.cwb[warp][b & 1]);
    __syncwarp();
    if (b + 1 <= b_hi) {
      cw_load<R>(a, side, sx, sy, b + 1, lane, sm.cwb[warp][(b + 1) & 1]);
      cp_async_commit();
    }
    if (a.tile_stats && lane == 0 && cls != kGeneral) atomicAdd(a.tile_stats + cls, 1ull);  // [4]: FAST EDGE GENERAL EMPTY
    unsigned long long k[16];
#pragma unroll
    for (int s2 = kPX * HPY; s2 < 16; ++s2) k[s2] = 0ull;
    const int di0 = b * kDB + 4 * dq;
    // padded disparity slots of the last block never win: their values get -inf
    float pad[4], cpad[4];  // cpad (KEYS): disparities outside [c_lo, c_hi] do not compete
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      pad[t] = di0 + t < a.D ? 0.f : -INFINITY;
      cpad[t] = KEYS ? (di0 + t >= a.c_lo && di0 + t <= a.c_hi ? 0.f : -INFINITY) : 0.f;
    }
    // aggregated costs (d = di0 .. di0+3) of half-row pixel (pyl, px) -> key, left store, export
    // (FAST / EDGE pass the padded values themselves, PADDED = true)
    auto emit = [&](int pyl, int px, float4 agg, bool padded) {
      const int y = sy + py0 + pyl, x = sx + px;
      float v0 = padded ? agg.x : agg.x + pad[0], v1 = padded ? agg.y : agg.y + pad[1],
            v2 = padded ? agg.z : agg.z + pad[2], v3 = padded ? agg.w : agg.w + pad[3];
      if constexpr (KEYS) {
        v0 += cpad[0]; v1 += cpad[1]; v2 += cpad[2]; v3 += cpad[3];
      }
      if constexpr (RANGED) {  // only the pixel's suggested range competes (R#32)
        const short2 r = sm.rng[wy + py0 + pyl][wx + px];
        const int d0 = a.d_min + di0;
        v0 += (d0 >= r.x && d0 <= r.y) ? 0.f : -INFINITY;
        v1 += (d0 + 1 >= r.x && d0 + 1 <= r.y) ? 0.f : -INFINITY;
        v2 += (d0 + 2 >= r.x && d0 + 2 <= r.y) ? 0.f : -INFINITY;
        v3 += (d0 + 3 >= r.x && d0 + 3 <= r.y) ? 0.f : -INFINITY;
      }
      const bool h01 = v1 > v0, h23 = v3 > v2;     // equal values keep the smaller d
      const float b01 = h01 ? v1 : v0, b23 = h23 ? v3 : v2;
      const bool h = b23 > b01;
      const int t = h ? 2 + h23 : h01;
      k[pyl * kPX + px] = ((unsigned long long)fkey(h ? b23 : b01) << 32) | (unsigned)(0xffff - (di0 + t));
      if (side == 0) {
        if (a.agg3)  // its weight row is dead: the stream of half-row pyl is done
          *reinterpret_cast<float4*>(vrow(pyl) + px * kDB + 4 * dq) = agg;
        else if (x < a.W && y < a.H)
          *reinterpret_cast<float4*>(a.aggL + (((size_t)(y - a.abase) * a.nblk + b) * a.W + x) * kDB + 4 * dq) = agg;
      } else if ((EXPORT ? a.exportR : nullptr) && x < a.W && y >= a.r0 && y < a.r1) {
        float* er = (EXPORT ? a.exportR : nullptr) + ((size_t)y * a.W + x) * a.D;
        const float av[4] = {agg.x, agg.y, agg.z, agg.w};
#pragma unroll
        for (int tt = 0; tt < 4; ++tt)
          if (di0 + tt < a.D) er[di0 + tt] = av[tt];
      }
    };
    if (cls != kGeneral) {
      float2 num[HPY][kPX][2];
      agg_num4<R, HPY>(vb, rowstride, wsm, num);
      if (a.agg3) __syncwarp();  // every lane is done with the weights before they are overwritten
#pragma unroll
      for (int pyl = 0; pyl < HPY; ++pyl)
#pragma unroll
        for (int px = 0; px < kPX; ++px) {
          const int pix = (py0 + pyl) * kPX + px;
          float ri[4];  // 1 / denominator per disparity
          if (cls == kFast) {
            const float r0 = sm.rinv[warp][pix];
            ri[0] = ri[1] = ri[2] = ri[3] = r0;
          } else {
            // EDGE: defined taps are those with dx >= d + 1 + R - x (left) or dx < W-1-d+R-x (right)
            const int x = sx + px;
            const int d0 = a.d_min + di0;
            const float* cs = sm.cs[warp][pix];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int m = side == 0 ? d0 + t + 1 + R - x : a.W - 1 - (d0 + t) + R - x;
              ri[t] = cs[min(max(m, 0), K1)];
            }
          }
          const float2 n0 = num[pyl][px][0], n1 = num[pyl][px][1];
          // num / den = num * (1/den) + 0, the padding (-inf) or, without any
          // defined tap (1/den stored as 0), the sentinel folded into the addend
          float off[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) off[t] = ri[t] > 0.f ? pad[t] : kSent;
          emit(pyl, px, make_float4(__fmaf_rn(n0.x, ri[0], off[0]), __fmaf_rn(n0.y, ri[1], off[1]),
                                    __fmaf_rn(n1.x, ri[2], off[2]), __fmaf_rn(n1.y, ri[3], off[3])), true);
        }
    } else if (EMPTY && cw_empty<R>(a, side, sx, sy, b, lane, sm.cwb[warp][b & 1])) {
      if (a.tile_stats && lane == 0) atomicAdd(a.tile_stats + kEmpty, 1ull);
      // every aggregated cost of the unit is SENT, which never wins the WTA (an
      // all-SENT pixel stays INVALID whatever key it keeps): only the full left
      // store and the debug export need the values
      if (side == 0 && !a.agg3) {
#pragma unroll 1
        for (int s2 = 0; s2 < kPX * HPY; ++s2) {
          const int y = sy + py0 + s2 / kPX, x = sx + s2 % kPX;
          if (x < a.W && y < a.H)
            *reinterpret_cast<float4*>(a.aggL + (((size_t)(y - a.abase) * a.nblk + b) * a.W + x) * kDB + 4 * dq) =
                make_float4(kSent, kSent, kSent, kSent);
        }
      } else if (side == 1 && (EXPORT ? a.exportR : nullptr)) {
#pragma unroll 1
        for (int s2 = 0; s2 < kPX * HPY; ++s2) {
          const int y = sy + py0 + s2 / kPX, x = sx + s2 % kPX;
          if (x < a.W && y >= a.r0 && y < a.r1)
            for (int tt = 0; tt < 4; ++tt)
              if (di0 + tt < a.D) (EXPORT ? a.exportR : nullptr)[((size_t)y * a.W + x) * a.D + di0 + tt] = kSent;
        }
      }
      // no keys: zero keys leave the running best unchanged
#pragma unroll
      for (int s2 = 0; s2 < kPX * HPY; ++s2) k[s2] = 0ull;
    } else {
      if (a.tile_stats && lane == 0) atomicAdd(a.tile_stats + kGeneral, 1ull);
#pragma unroll
      for (int pyl = 0; pyl < HPY; ++pyl) {
        float2 num[kPX][2], den[kPX][2];
        agg_num_den_row4<R>(vb + (size_t)pyl * rowstride, rowstride, wsm + pyl * RS, num, den);
        if (a.agg3) __syncwarp();
#pragma unroll
        for (int px = 0; px < kPX; ++px) {
          const float2 n0 = num[px][0], n1 = num[px][1], e0 = den[px][0], e1 = den[px][1];
          emit(pyl, px, make_float4(e0.x > 0.f ? __fmul_rn(n0.x, rcp_nr(e0.x)) : kSent,
                                    e0.y > 0.f ? __fmul_rn(n0.y, rcp_nr(e0.y)) : kSent,
                                    e1.x > 0.f ? __fmul_rn(n1.x, rcp_nr(e1.x)) : kSent,
                                    e1.y > 0.f ? __fmul_rn(n1.y, rcp_nr(e1.y)) : kSent), false);
        }
      }
    }
    best = umax64(best, wta_butterfly16(k, lane));  // earlier blocks win ties (smaller d)
  }

  // ---- epilogue: lane l holds slot l & 15 of its half ----
  if (a.agg3) __syncwarp();  // the half's on-chip costs are complete
  {
    const int s2 = lane & 15;
    if (s2 < kPX * HPY) {
      const int x = sx + s2 % kPX, y = sy + py0 + s2 / kPX;
      if (x < a.W && y >= a.r0 && y < a.r1) {
        const bool ok = (unsigned)(best >> 32) > fkey(kSent);
        const int d_int = ok ? a.d_min + (0xffff - (int)(best & 0xffffu)) : -1;
        (side == 0 ? a.dL : a.dR)[(size_t)y * a.W + x] = d_int;
        if constexpr (KEYS)  // global-d key: (value bits << 32) | (0xFFFFFFFF - d); 0 = no defined cost
          a.keys_out[side][(size_t)y * a.W + x] =
              ok ? ((best >> 32) << 32) | (unsigned long long)(0xffffffffu - (unsigned)d_int) : 0ull;
        if (side == 0 && a.agg3 && ok) {  // the three costs Eq.(10) needs
          const float* vr = vrow(s2 / kPX) + (s2 % kPX) * kDB;
          const int di = d_int - a.d_min;
          bool in_m = di > 0, in_p = di + 1 < a.D;
          if constexpr (RANGED) {  // the range ends act like the ends of [d_min, d_max] (R#33)
            const short2 r = sm.rng[wy + py0 + s2 / kPX][wx + s2 % kPX];
            in_m = in_m && d_int - 1 >= r.x;
            in_p = in_p && d_int + 1 <= r.y;
          }
          a.agg3[(size_t)y * a.W + x] = make_float4(in_m ? vr[di - 1] : kSent, vr[di], in_p ? vr[di + 1] : kSent, 0.f);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Debug select path: WTA over a given [H][W][D] volume (same rules as k_agg);
// the left volume is also copied into the [H][nblk][W][64] layout k_finalize reads.
__global__ void k_select_wta(const float* __restrict__ agg, int W, int H, int D, int d_min, int nblk,
                             int32_t* __restrict__ disp, float* __restrict__ aggL) {
  const size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (p >= (size_t)W * H) return;
  const float* col = agg + p * D;
  float best = -INFINITY;
  int bi = 0;
  for (int k = 0; k < D; ++k) {
    const float v = col[k];
    if (v > best) { best = v; bi = k; }
    if (aggL) {
      const size_t y = p / W, x = p % W;
      aggL[((y * nblk + k / kDB) * W + x) * kDB + k % kDB] = v;
    }
  }
  disp[p] = best > kSent ? d_min + bi : -1;
}

#include "fbs_aggsd.cuh"  // k_aggsd: D <= 16

}  // namespace vol
}  // namespace fbs
