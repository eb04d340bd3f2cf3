// fbs_fused.cuh — the fused sm_100a path: block statistics once per image
// (k_prep), then ONE kernel per frame batch that computes the NCC costs of a
// tile into shared memory and aggregates them there (k_fbs): the cost volume
// never leaves the SM.
//
//   k_prep   per image and pixel: the packed 3-pixel column, the block
//            statistics S = Σ_3x3 i and r = V^{-1/2}, V = 9 Σ i² - S²
//            (Eq.(2)(3), "pre-calculated" P:L84), the guide value and
//            the bit-packed block-defined mask.  ~12 B per pixel and image.
//   k_fbs    persistent "walker": CTA c owns a contiguous run of (frame, side,
//            16-column strip, 12-row step) units and walks down its strips.
//            Per step and 64-disparity block:
//              1. TMA (cp.async.bulk.tensor) stages the 12 new rows of packed
//                 columns + statistics of the strip and of the other image's
//                 disparity range (issued one phase ahead, mbarrier-tracked);
//              2. the CTA computes the twin NCC costs of those rows (Eq.(1),
//                 exact integer N, DP4A column dots) into a ring of cost rows
//                 in shared memory (ρ-row halo kept from the previous step, so
//                 every cost row is computed once per strip and d-block);
//              3. the bilateral weights of the step's 192 pixels (Eq.(6)-(8))
//                 from the TMA-staged guide tile;
//              4. the FFMA2 aggregation stream of k_agg, fed by LDS from the
//                 ring instead of LDG from an HBM volume, then the WTA
//                 butterfly and the per-pixel record (best key + the three
//                 aggregated costs Eq.(10) needs, tracked across d-blocks).
//   k_finalize (fbs_kernels.cuh) then applies LRC (Eq.(9)) and the subpixel fit.
#pragma once
#include <cuda.h>

#include "fbs_kernels.cuh"

namespace fbs {

// ---------------------------------------------------------------------------
// k_prep: per-pixel statistics of both images of F frames.
struct PrepArgs {
  int W, H, Wp, Wg, Wb, R, y0, y1;  // rows [y0, y1)
  const uint8_t* img[2];             // left, right: [F][H][W]
  uint32_t* P[2];                    // packed columns [F][H][Wp]
  int2* SR[2];                       // (S, V^{-1/2} bits) [F][H][Wp]; r = 0: undefined block
  float* G[2];                       // padded guides [F][guide_rows][Wg] (interior written here)
  uint32_t* bits[2];                 // block-defined masks [F][H][Wb]
  size_t gfs;                        // guide frame stride (floats)
};

// grid (ceil(W/128), y1-y0, 2 F); block 128.  Position (x, y) of image z&1, frame z>>1.
__global__ void __launch_bounds__(128) k_prep(PrepArgs a) {
  pdl_trigger();
  pdl_wait();
  const int im = blockIdx.z & 1, f = blockIdx.z >> 1;
  const int x = blockIdx.x * 128 + threadIdx.x, y = a.y0 + blockIdx.y;
  const size_t fo = (size_t)f * a.H;
  const uint8_t* I = a.img[im] + fo * a.W;
  uint32_t Pc = 0u;
  int S = 0, Q = 0;
  float rs = 0.f;
  const bool inb = x >= 1 && x <= a.W - 2 && y >= 1 && y <= a.H - 2;
  if (x < a.W && y >= 1 && y <= a.H - 2) {
    const uint32_t u0 = I[(size_t)(y - 1) * a.W + x], u1 = I[(size_t)y * a.W + x], u2 = I[(size_t)(y + 1) * a.W + x];
    Pc = u0 | (u1 << 8) | (u2 << 16);
  }
  if (inb) {
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int v = I[(size_t)(y + dy) * a.W + x + dx];
        S += v;
        Q += v * v;
      }
    const int V = 9 * Q - S * S;  // exact: < 2^24 (R#5); V = 0 <=> σ < σ_floor (R#7)
    if (V > 0) {
      const float v = (float)V;
      float r;
      asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
      rs = __fmul_rn(r, __fmaf_rn(__fmul_rn(-0.5f * v, r), r, 1.5f));  // one Newton step (~1 ulp)
    }
  }
  const bool ok = rs != 0.f;
  const unsigned bits = __ballot_sync(0xffffffffu, ok);
  if (x < a.W) {
    const size_t p = (fo + y) * a.Wp + x;
    a.P[im][p] = Pc;
    a.SR[im][p] = make_int2(S, __float_as_int(rs));
    const float gi = (float)I[(size_t)y * a.W + x] + (ok ? 0.f : kGuideFlag);
    a.G[im][f * a.gfs + (size_t)(y + a.R) * a.Wg + x + a.R] = gi;
    if ((threadIdx.x & 31) == 0) a.bits[im][(fo + y) * a.Wb + x / 32] = bits;
  }
}

// ---------------------------------------------------------------------------
// TMA / mbarrier helpers (PTX; SASS UTMALDG / SYNCS)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
#ifndef FBS_SUSPEND_HINT
#define FBS_SUSPEND_HINT 0x989680
#endif
// try_wait with a suspend-time hint: the waiting warp sleeps in hardware until
// the phase completes (or the hint expires) instead of spinning on issue slots.
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(FBS_SUSPEND_HINT)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, unsigned long long* bar, int x, int y,
                                            int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Walker geometry.  Warps: 4 across x 2 down, sub-tile 4 x PY pixels (two
// half-warps of HPY rows); CTA step tile TX x TY; cost ring SR rows x SC cols
// x 64 disparities.  One CTA per SM (the ring + weights use ~220 KB).
template <int R>
struct WGeo {
  static constexpr int RR = R;
  static constexpr int K1 = 2 * R + 1;
  static constexpr int HPY = R <= 4 ? 3 : (R == 5 ? 2 : 1);
  static constexpr int PY = 2 * HPY;
  static constexpr int NWX = 4, NWY = 2, NW = 8, THREADS = 256;
  static constexpr int TX = kPX * NWX;  // 16
  static constexpr int TY = PY * NWY;
  static constexpr int SC = TX + 2 * R;  // ring columns: x0-R .. x0+TX+R-1
  static constexpr int SR = TY + 2 * R;  // ring rows
  static constexpr int NSLOT = SR;       // ring slots (a frame row's slot: row index mod NSLOT)
  static constexpr int CU = SC / 2;      // positions per cost unit (half a ring row)
  // staging (TMA boxes; inner extent x element size a multiple of 16 B).  A box
  // must also START at a 16-B aligned x (measured on this part: other starts
  // fault with an illegal instruction, tools/microbench/tma_probe.cu), so each
  // box starts at the aligned column at or below the first one needed and is
  // up to 3 words wider; walk_off() gives the offset of the first needed one.
  static constexpr int SROWS = ((TY > 2 * R ? TY : 2 * R) + 1) / 2 * 2;
  static constexpr int SPC = (SC + 2 + 3 + 3) / 4 * 4;   // self packed columns  x0-R-1 ..
  static constexpr int SSC = (SC + 1 + 1) / 2 * 2;       // self statistics      x0-R ..  (pairs)
  static constexpr int OPC = (SC + 65 + 3 + 3) / 4 * 4;  // other packed columns obase-1 ..
  static constexpr int OSC = (SC + 63 + 1 + 1) / 2 * 2;  // other statistics     obase .. (pairs)
  static constexpr int GW = (SC + 3) / 4 * 4;
  static constexpr int GWS = GW % 32 == 24 ? GW + 4 : GW;  // guide tile row stride (bank spread)
  static constexpr int GH = SR;
  static constexpr int WPW = PY * K1 * K1 * kPX;         // weights per warp
  static constexpr bool kAlias = K1 * K1 >= kDB;         // dead weight rows hold the left costs
};

// Timing ablations (experiment builds only, tools/build_variants.py): bit 1 skips
// the cost phase, bit 2 the FMA stream, bit 4 the weight prologue, bit 8 (k_fbs_ws)
// the TMA loads.  Results are
// wrong in those builds; 0 in the product.
#ifndef FBS_ABL
#define FBS_ABL 0
#endif

template <int R>
struct WSmem {
  using G = WGeo<R>;
  alignas(128) float ring[G::SR][G::SC][kDB];
  alignas(128) uint32_t Ps[G::SROWS * G::SPC];
  alignas(128) uint32_t Po[G::SROWS * G::OPC];
  alignas(128) int2 Ss[G::SROWS * G::SSC];
  alignas(128) int2 So[G::SROWS * G::OSC];
  alignas(128) float g[2][(G::GH * G::GWS + 31) / 32 * 32];  // each buffer a 128-B aligned TMA destination
  float w[G::NW][G::WPW];  // [warp][py][dy][dx][px]
  float val[G::NW][G::kAlias ? 4 : G::PY * kPX * kDB];
  float rinv[G::NW][32];
  float cs[G::NW][32][G::K1 + 1];
  uint32_t cwb[G::NW][64];
  unsigned long long bar;
};

struct WalkArgs {
  CUtensorMap tmPs[2], tmPo[2], tmSs[2], tmSo[2], tmG[2];  // [image]: 0 left, 1 right
  int W, H, D, d_min, d_max, nblk;
  int Wb;
  const uint32_t* bits[2];  // [F][H][Wb]
  int32_t* dmap[2];         // dL, dR [F][H][W]
  float4* agg3;             // left (c(d*-1), c(d*), c(d*+1), c(last d of block)) [F][H][W]
  unsigned long long* keys; // [2][F][H][W] running best keys (nblk > 1)
  int r0, r1;               // output rows
  int ty0, nty, nstrips, nframes;
  long long total;          // walker steps
  float* expC[2];           // EXPORT: cost volumes [F=1][H][W][D], FBS_SENTINEL = undefined
  float* expA[2];           // EXPORT: aggregated volumes
  unsigned long long* tile_stats;
  unsigned long long* trace;  // FBS_TRACE builds only: clock64 stamps of CTA 0 (else null)
  float nkr;
  float cd[(2 * kMaxRadius + 1) * (2 * kMaxRadius + 1)];
};

// Staging offsets of the first needed column in each box (boxes start at the
// 16-B aligned column at or below it; & 3 is the floor modulus).
struct WOff {
  int ps, ss, po, so;  // packed-column words / statistics pairs
  __device__ __forceinline__ WOff(int R, int x0, int side, int dlo) {
    const int obase = side == 0 ? x0 - R - dlo - 63 : x0 - R + dlo;
    ps = (x0 - R - 1) & 3;
    ss = (x0 - R) & 1;
    po = (obase - 1) & 3;
    so = obase & 1;
  }
};

// Denominator form of one warp sub-tile and d-block (forms: fbs_kernels.cuh),
// exact and conservative: EDGE if the frame edge cuts taps off, GENERAL if the
// other image has an undefined block anywhere in the shifted range (<= 16 rows
// x 4 mask words, two per lane).
template <class G>
struct WCw {
  int qy0, lo, hi, edge, nw, rows, w0;
  __device__ __forceinline__ WCw(int W, int H, int d_min, int d_max, int side, int sx, int sy, int b) {
    constexpr int R = G::RR;
    qy0 = max(sy - R, 1);
    const int qy1 = min(sy + G::PY - 1 + R, H - 2);
    const int qx0 = max(sx - R, 1), qx1 = min(sx + kPX - 1 + R, W - 2);
    const int d_lo = d_min + b * kDB, d_hi = min(d_lo + kDB - 1, d_max);
    if (side == 0) { lo = qx0 - d_hi; hi = qx1 - d_lo; edge = lo < 1; lo = max(lo, 1); }
    else { lo = qx0 + d_lo; hi = qx1 + d_hi; edge = hi > W - 2; hi = min(hi, W - 2); }
    rows = (qy0 <= qy1 && qx0 <= qx1 && lo <= hi) ? qy1 - qy0 + 1 : 0;
    w0 = lo >> 5;
    nw = rows ? (hi >> 5) - w0 + 1 : 0;
  }
  __device__ __forceinline__ uint32_t mask(int wi) const {
    uint32_t m = 0xffffffffu;
    if (wi == w0) m &= 0xffffffffu << (lo & 31);
    if (wi == (hi >> 5)) m &= 0xffffffffu >> (31 - (hi & 31));
    return m;
  }
};

// Cost rows -> ring.  Rows [yc, yc + n) of frame f, strip x0, disparity block
// starting at dlo; staging row t holds frame row yc + t.  Unit = (row, half):
// lane <-> disparity pair (2 lane, 2 lane + 1), CU positions per unit; the 3x3
// dot product is the sum of three DP4A column dots shared along the unit.
// Both sides evaluate N · (r_self · r_other) with the same exact integer N and
// a commutative product, so right(u-d,v,d) == left(u,v,d) bit-exactly.
// Geometry-generic form: staging buffers Ps/Po/Ss/So, ring [G::NSLOT][G::SC][64];
// row yc + t goes to ring slot (slot0 + t) mod NSLOT; units (row, half) u =
// u0, u0 + us, ... (the calling warps).
template <class G, int SIDE, bool EXPORT>
__device__ __forceinline__ void walk_cost_g(const WalkArgs& a, float (*ring)[G::SC][kDB], const uint32_t* Ps,
                                            const uint32_t* Po, const int2* Ss, const int2* So, int yc, int n,
                                            int slot0, int x0, int dlo, int u0, int us) {
  constexpr int R = G::RR;
  constexpr int CU = G::CU;
  const int lane = threadIdx.x & 31;
  const int k0 = 2 * lane;
  const bool pad0 = dlo + k0 > a.d_max, pad1 = dlo + k0 + 1 > a.d_max;
  const WOff off(R, x0, SIDE, dlo);
  for (int u = u0; u < 2 * n; u += us) {
    const int yy = u >> 1, i0 = (u & 1) * CU;
    const int y = yc + yy;
    int slot = slot0 + yy;
    if (slot >= G::NSLOT) slot -= G::NSLOT;
    float* dst = &ring[slot][i0][k0];
    // self packed columns of positions i0-1 .. i0+CU (staging col ip = i + 1)
    const uint32_t* ps = Ps + yy * G::SPC + off.ps + i0;
    // other packed columns: side 0 jp = i - k + 64 (k0: i0-1+m - k0 + 64); side 1 jp = i + k + 1
    const uint32_t* pob = Po + yy * G::OPC + off.po + (SIDE == 0 ? i0 + 63 - k0 - 1 : i0 + k0);
    uint32_t po[CU + 3];
#pragma unroll
    for (int m = 0; m < CU + 3; ++m) po[m] = pob[m];
    int cd0[CU + 2], cd1[CU + 2];
#pragma unroll
    for (int m = 0; m < CU + 2; ++m) {
      const uint32_t s = ps[m];
      cd0[m] = (int)__dp4a(s, SIDE == 0 ? po[m + 1] : po[m], 0u);
      cd1[m] = (int)__dp4a(s, SIDE == 0 ? po[m] : po[m + 1], 0u);
    }
    // statistics: self position i -> Ss[i]; other: side 0 j = i - k + 63, side 1 j = i + k
    const int2* ss = Ss + yy * G::SSC + off.ss + i0;
    const int2* sob = So + yy * G::OSC + off.so + (SIDE == 0 ? i0 + 63 - k0 - 1 : i0 + k0);
    int2 so[CU + 1];
#pragma unroll
    for (int m = 0; m < CU + 1; ++m) so[m] = sob[m];
#pragma unroll
    for (int q = 0; q < CU; ++q) {
      const int2 sv = ss[q];
      const float rsf = __int_as_float(sv.y);
      float o[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        // side 0: k0 -> so[q + 1], k1 -> so[q]; side 1: k0 -> so[q], k1 -> so[q + 1]
        const int2 ov = SIDE == 0 ? so[q + 1 - k] : so[q + k];
        const int dot = k == 0 ? cd0[q] + cd0[q + 1] + cd0[q + 2] : cd1[q] + cd1[q + 1] + cd1[q + 2];
        const int N = 9 * dot - sv.x * ov.x;  // exact (|N| < 2^24, R#5)
        const float Pp = __fmul_rn(rsf, __int_as_float(ov.y));
        const float c = fminf(1.0f, fmaxf(-1.0f, __fmul_rn((float)N, Pp)));  // clamp (R#8)
        o[k] = Pp != 0.f ? c : kUndef;
      }
      if (pad0) o[0] = kUndef;
      if (pad1) o[1] = kUndef;
      *reinterpret_cast<float2*>(dst + q * kDB) = make_float2(o[0], o[1]);
      if constexpr (EXPORT) {
        const int x = x0 - R + i0 + q;
        if (x >= x0 && x < x0 + G::TX && x < a.W && y >= 0 && y < a.H && a.expC[SIDE]) {
          float* e = a.expC[SIDE] + ((size_t)y * a.W + x) * a.D + (dlo - a.d_min);
#pragma unroll
          for (int k = 0; k < 2; ++k)
            if (dlo + k0 + k <= a.d_max) e[k0 + k] = is_undef(o[k]) ? kSent : o[k];
        }
      }
    }
  }
}

template <int R, int SIDE, bool EXPORT>
__device__ __forceinline__ void walk_cost(const WalkArgs& a, WSmem<R>& sm, int yc, int n, int yb, int x0, int dlo,
                                          int f) {
  using G = WGeo<R>;
  walk_cost_g<G, SIDE, EXPORT>(a, sm.ring, sm.Ps, sm.Po, sm.Ss, sm.So, yc, n, (yc - yb) % G::SR, x0, dlo,
                               threadIdx.x >> 5, G::NW);
}

// Numerator stream over the ring (FAST / EDGE): as Rows4 in k_agg, cost row r of
// the half-warp lives in ring slot (base + r) mod SR.
template <class G, int r, int NR, int NPY>
struct RingRows {
  static __device__ __forceinline__ void run(const float* __restrict__ col, int base, const float* __restrict__ wsm,
                                             float4 (&head)[kPX], float2 (&num)[NPY][kPX][2]) {
    constexpr int R = G::RR;
    constexpr int NC = kPX + 2 * R;
    constexpr int RS = G::SC * kDB;
    float4 c[NC];
#pragma unroll
    for (int j = 0; j < kPX; ++j) c[j] = head[j];
    int s = base + r;
    if (s >= G::NSLOT) s -= G::NSLOT;
    const float* rp = col + s * RS;
#pragma unroll
    for (int j = kPX; j < NC; ++j) c[j] = *reinterpret_cast<const float4*>(rp + j * kDB);
    if constexpr (r + 1 < NR) {
      int s1 = s + 1;
      if (s1 >= G::NSLOT) s1 -= G::NSLOT;
      const float* rn = col + s1 * RS;
#pragma unroll
      for (int j = 0; j < kPX; ++j) head[j] = *reinterpret_cast<const float4*>(rn + j * kDB);
    }
    row_fma4<R, NPY, r>(c, wsm, num);
    RingRows<G, r + 1, NR, NPY>::run(col, base, wsm, head, num);
  }
};
template <class G, int NR, int NPY>
struct RingRows<G, NR, NR, NPY> {
  static __device__ __forceinline__ void run(const float*, int, const float*, float4 (&)[kPX],
                                             float2 (&)[NPY][kPX][2]) {}
};

// Compact form of the stream (the warp-specialised walker: producer and
// consumer warps share the SM's instruction caches, so the stream must be
// small).  Rows that feed only some of the NPY output rows (the first NPY-1
// and the last NPY-1 cost rows) are unrolled at compile time; the cost rows
// that feed all NPY output rows run in a loop whose body is one cost row
// (NC LDS.128 + NPY*K1 weight LDS.128 + NPY*K1*8 FFMA2).  Per accumulator the
// summation order is the same as RingRows (dy ascending, then dx).
template <class G, int r, int NPY>
__device__ __forceinline__ void ring_row_ct(const float* __restrict__ col, int base, const float* __restrict__ wsm,
                                            float2 (&num)[NPY][kPX][2]) {
  constexpr int R = G::RR;
  constexpr int NC = kPX + 2 * R;
  int s = base + r;
  if (s >= G::NSLOT) s -= G::NSLOT;
  const float* rp = col + s * (G::SC * kDB);
  float4 c[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) c[j] = *reinterpret_cast<const float4*>(rp + j * kDB);
  row_fma4<R, NPY, r>(c, wsm, num);
}
template <class G, int r, int rend, int NPY>
struct RowsCT {
  static __device__ __forceinline__ void run(const float* __restrict__ col, int base, const float* __restrict__ wsm,
                                             float2 (&num)[NPY][kPX][2]) {
    ring_row_ct<G, r, NPY>(col, base, wsm, num);
    RowsCT<G, r + 1, rend, NPY>::run(col, base, wsm, num);
  }
};
template <class G, int rend, int NPY>
struct RowsCT<G, rend, rend, NPY> {
  static __device__ __forceinline__ void run(const float*, int, const float*, float2 (&)[NPY][kPX][2]) {}
};
template <class G, int NPY>
__device__ __forceinline__ void ring_stream(const float* __restrict__ col, int base, const float* __restrict__ wsm,
                                            float2 (&num)[NPY][kPX][2]) {
  constexpr int R = G::RR, K1 = 2 * R + 1;
  constexpr int NC = kPX + 2 * R;
  constexpr int NR = NPY + 2 * R;
  if constexpr (2 * R < NPY - 1) {
    RowsCT<G, 0, NR, NPY>::run(col, base, wsm, num);
  } else {
    RowsCT<G, 0, NPY - 1, NPY>::run(col, base, wsm, num);  // head rows
    int s = base + NPY - 1;
    if (s >= G::NSLOT) s -= G::NSLOT;
    float4 head[kPX];  // the first kPX columns of the loop's next row, loaded one row ahead
    {
      const float* rp = col + s * (G::SC * kDB);
#pragma unroll
      for (int j = 0; j < kPX; ++j) head[j] = *reinterpret_cast<const float4*>(rp + j * kDB);
    }
#pragma unroll 1
    for (int r = NPY - 1; r <= 2 * R; ++r) {  // full rows: every output row pyl, dy = r - pyl
      const float* rp = col + s * (G::SC * kDB);
      if (++s >= G::NSLOT) s -= G::NSLOT;
      float4 c[NC];
#pragma unroll
      for (int j = 0; j < kPX; ++j) c[j] = head[j];
#pragma unroll
      for (int j = kPX; j < NC; ++j) c[j] = *reinterpret_cast<const float4*>(rp + j * kDB);
      {  // next row's head (the row after the loop is a tail row or, for ρ's last row, harmless)
        const float* rn = col + s * (G::SC * kDB);
#pragma unroll
        for (int j = 0; j < kPX; ++j) head[j] = *reinterpret_cast<const float4*>(rn + j * kDB);
      }
      const float* wr = wsm + r * K1 * kPX;  // (pyl, dy = r - pyl) -> wr + pyl (K1 - 1) K1 kPX
#pragma unroll
      for (int dx = 0; dx < K1; ++dx) {
#pragma unroll
        for (int pyl = 0; pyl < NPY; ++pyl) {
          const float4 w = reinterpret_cast<const float4*>(wr + pyl * (K1 - 1) * K1 * kPX)[dx];
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
    RowsCT<G, 2 * R + 1, NR, NPY>::run(col, base, wsm, num);  // tail rows
  }
}

// GENERAL: explicit numerator and denominator of one output row.
template <class G>
__device__ __forceinline__ void ring_num_den_row(const float* __restrict__ col, int base, const float* __restrict__ wrow,
                                                 float2 (&num)[kPX][2], float2 (&den)[kPX][2]) {
  constexpr int R = G::RR;
  constexpr int K1 = 2 * R + 1;
  constexpr int NC = kPX + 2 * R;
  constexpr int RS = G::SC * kDB;
#pragma unroll
  for (int px = 0; px < kPX; ++px) num[px][0] = num[px][1] = den[px][0] = den[px][1] = make_float2(0.f, 0.f);
#pragma unroll 1
  for (int dy = 0; dy < K1; ++dy) {
    int s = base + dy;
    if (s >= G::NSLOT) s -= G::NSLOT;
    const float* rp = col + s * RS;
    float4 c[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) c[j] = *reinterpret_cast<const float4*>(rp + j * kDB);
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

// Issue the TMA loads of one walker phase (one thread): rows [yc, yc + G::SROWS)
// of the strip's packed columns / statistics and of the other image's range;
// with gdst also the guide tile of output rows [y0, y0 + G::GH - 2R).
// Completion: bar (one phase, expect_tx).
template <class G>
__device__ __forceinline__ void walk_issue_g(const WalkArgs& a, uint32_t* Ps, int2* Ss, uint32_t* Po, int2* So,
                                             float* gdst, unsigned long long* bar, int f, int side, int strip, int b,
                                             int yc, int y0) {
  constexpr int R = G::RR;
  constexpr unsigned kStageBytes = G::SROWS * (G::SPC * 4 + G::SSC * 8 + G::OPC * 4 + G::OSC * 8);
  constexpr unsigned kGuideBytes = G::GH * G::GWS * 4;
  const int x0 = strip * G::TX;
  const int dlo = a.d_min + b * kDB;
  const int obase = side == 0 ? x0 - R - dlo - 63 : x0 - R + dlo;
  fence_proxy_async();
  mbar_expect_tx(bar, kStageBytes + (gdst ? kGuideBytes : 0u));
  tma_load_3d(Ps, &a.tmPs[side], bar, (x0 - R - 1) & ~3, yc, f);
  tma_load_3d(Ss, &a.tmSs[side], bar, (2 * (x0 - R)) & ~3, yc, f);  // (S, r) word pairs
  tma_load_3d(Po, &a.tmPo[1 - side], bar, (obase - 1) & ~3, yc, f);
  tma_load_3d(So, &a.tmSo[1 - side], bar, (2 * obase) & ~3, yc, f);
  if (gdst) tma_load_3d(gdst, &a.tmG[side], bar, x0, y0, f);  // padded coordinates: frame (x0-R, y0-R)
}
template <int R>
__device__ __forceinline__ void walk_issue(const WalkArgs& a, WSmem<R>& sm, int f, int side, int strip, int b, int yc,
                                           int y0, bool step, int gb) {
  walk_issue_g<WGeo<R>>(a, sm.Ps, sm.Ss, sm.Po, sm.So, step ? sm.g[gb] : nullptr, &sm.bar, f, side, strip, b, yc, y0);
}

// grid: min(total steps, #SMs) CTAs; block 256; one CTA per SM.
template <int R, bool EXPORT>
__global__ void __launch_bounds__(256, 1) k_fbs(const __grid_constant__ WalkArgs a) {
  using G = WGeo<R>;
  constexpr int K1 = 2 * R + 1;
  constexpr int kPY = G::PY, HPY = G::HPY, GWS = G::GWS;
  constexpr int RS = K1 * K1 * kPX;  // weights per output row
  extern __shared__ __align__(128) unsigned char smraw[];
  // TMA destinations need 128-B alignment: align the dynamic base (+128 B requested)
  WSmem<R>& sm = *reinterpret_cast<WSmem<R>*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wx = (warp % G::NWX) * kPX, wy = (warp / G::NWX) * kPY;
  const long long T = a.total;
  const long long s_begin = blockIdx.x * T / gridDim.x, s_end = (blockIdx.x + 1) * T / gridDim.x;
  if (s_begin >= s_end) return;

  auto decomp = [&](long long s, int& f, int& side, int& strip, int& j) {
    j = (int)(s % a.nty);
    long long q = s / a.nty;
    strip = (int)(q % a.nstrips);
    q /= a.nstrips;
    side = (int)(q & 1);
    f = (int)(q >> 1);
  };
  // walks: maximal runs of steps of one (frame, side, strip) inside [s_begin, s_end)
  auto walk_end = [&](long long s) {
    const long long e = s - s % a.nty + a.nty;
    return e < s_end ? e : s_end;
  };
  // first phase of a walk-block: the fill (R > 0) or its first step
  auto issue_first = [&](long long s, int b, int gb) {
    int f, side, strip, j;
    decomp(s, f, side, strip, j);
    const int y0 = (a.ty0 + j) * G::TY;
    if (R > 0) walk_issue<R>(a, sm, f, side, strip, b, y0 - R, y0, false, 0);
    else walk_issue<R>(a, sm, f, side, strip, b, y0 + R, y0, true, gb);
  };

  if (threadIdx.x == 0) {
    mbar_init(&sm.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      tma_prefetch_desc(&a.tmPs[i]); tma_prefetch_desc(&a.tmPo[i]);
      tma_prefetch_desc(&a.tmSs[i]); tma_prefetch_desc(&a.tmSo[i]); tma_prefetch_desc(&a.tmG[i]);
    }
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();  // k_prep's outputs are complete and visible
  if (threadIdx.x == 0) issue_first(s_begin, 0, 0);

  const int half = lane >> 4, dq = lane & 15;
  const int py0 = half * HPY;
  unsigned par = 0;
  int nstep = 0;  // steps executed by this CTA (guide buffer parity)

  for (long long s = s_begin; s < s_end;) {
    const long long we = walk_end(s);
    int f, side, strip, j0;
    decomp(s, f, side, strip, j0);
    const int x0 = strip * G::TX;
    const int ya = (a.ty0 + j0) * G::TY;
    const int yb = ya - R;  // frame row of ring slot 0
    const int sx = x0 + wx;
    const uint32_t* obits = a.bits[1 - side] + (size_t)f * a.H * a.Wb;
    for (int b = 0; b < a.nblk; ++b) {
      const int dlo = a.d_min + b * kDB;
      if (R > 0) {  // fill: cost rows [ya - R, ya + R)
        mbar_wait(&sm.bar, par);
        par ^= 1;
        if (!(FBS_ABL & 1)) {
          if (side == 0) walk_cost<R, 0, EXPORT>(a, sm, ya - R, 2 * R, yb, x0, dlo, f);
          else walk_cost<R, 1, EXPORT>(a, sm, ya - R, 2 * R, yb, x0, dlo, f);
        }
        __syncthreads();
        if (threadIdx.x == 0) walk_issue<R>(a, sm, f, side, strip, b, ya + R, ya, true, nstep & 1);
      }
      for (long long t = s; t < we; ++t) {
        const int j = j0 + (int)(t - s);
        const int y0 = (a.ty0 + j) * G::TY;
        const int sy = y0 + wy;
        const int gb = nstep & 1;
        // classification words of this (sub-tile, d-block), in flight during the cost phase
        const WCw<G> cw(a.W, a.H, a.d_min, a.d_max, side, sx, sy, b);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int i = lane + 32 * k, row = i >> 2, wd = i & 3;
          if (row < cw.rows && wd < cw.nw) cp_async4(sm.cwb[warp] + i, obits + (size_t)(cw.qy0 + row) * a.Wb + cw.w0 + wd);
        }
        cp_async_commit();
        mbar_wait(&sm.bar, par);
        par ^= 1;
        // ---- cost rows [y0 + R, y0 + TY + R) -> ring ----
        if (!(FBS_ABL & 1)) {
          if (side == 0) walk_cost<R, 0, EXPORT>(a, sm, y0 + R, G::TY, yb, x0, dlo, f);
          else walk_cost<R, 1, EXPORT>(a, sm, y0 + R, G::TY, yb, x0, dlo, f);
        }
        // ---- weights w'(p,q) of the warp's pixels, Eq.(6)-(8) (see k_agg) ----
        if (!(FBS_ABL & 4) && lane < kPX * kPY) {
          const int py = lane / kPX, px = lane % kPX;
          float* wsm = sm.w[warp];
          const float* gq = sm.g[gb] + (wy + py) * GWS + (wx + px);
          const float gc = gq[R * GWS + R];
          const float gp = gc >= kGuideFlag ? __fsub_rn(gc, kGuideFlag) : gc;
          float wsum = 0.f;
          float col[K1];
#pragma unroll
          for (int dx = 0; dx < K1; ++dx) col[dx] = 0.f;
          constexpr int CH = (K1 * K1 <= 64) ? K1 : (64 / K1 > 0 ? 64 / K1 : 1);
#pragma unroll
          for (int dy0 = 0; dy0 < K1; dy0 += CH) {
            constexpr int NB = CH * K1;
            float gv[NB];
#pragma unroll
            for (int tt = 0; tt < NB; ++tt) {
              const int dy = dy0 + tt / K1, dx = tt % K1;
              gv[tt] = dy < K1 ? gq[dy * GWS + dx] : 0.f;
            }
#pragma unroll
            for (int tt = 0; tt < NB; ++tt) {
              const int dy = dy0 + tt / K1, dx = tt % K1;
              if (dy < K1) {
                const float dd = __fsub_rn(gv[tt], gp);
                float w;
                asm("ex2.approx.ftz.f32 %0, %1;"
                    : "=f"(w)
                    : "f"(__fmaf_rn(__fmul_rn(dd, dd), a.nkr, a.cd[dy * K1 + dx])));
                col[dx] = __fadd_rn(col[dx], w);
                wsm[((py * K1 + dy) * K1 + dx) * kPX + px] = w;
              }
            }
          }
#pragma unroll
          for (int dx = 0; dx < K1; ++dx) wsum = __fadd_rn(wsum, col[dx]);
          sm.rinv[warp][lane] = wsum > 0.f ? rcp_nr(wsum) : 0.f;
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
        cp_async_wait_all();
        __syncwarp();
        bool tex = false, def = false;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int i = lane + 32 * k, row = i >> 2, wd = i & 3;
          if (row < cw.rows && wd < cw.nw) {
            const uint32_t m = cw.mask(cw.w0 + wd), v = sm.cwb[warp][i];
            tex |= (~v & m) != 0u;
            def |= (v & m) != 0u;
          }
        }
        const int cls = __any_sync(0xffffffffu, tex) ? kGeneral : (cw.edge ? kEdge : kFast);
        const bool empty = cls == kGeneral && cw.rows > 0 && !__any_sync(0xffffffffu, def);
        __syncthreads();  // (A) ring rows and weights complete; staging consumed
        if (threadIdx.x == 0) {  // next phase's staging, in flight during this step's stream
          const bool more = t + 1 < we;
          if (more) walk_issue<R>(a, sm, f, side, strip, b, y0 + G::TY + R, y0 + G::TY, true, (nstep + 1) & 1);
          else if (b + 1 < a.nblk) issue_first(s, b + 1, (nstep + 1) & 1);
          else if (we < s_end) issue_first(we, 0, (nstep + 1) & 1);
        }
        if (a.tile_stats && lane == 0) atomicAdd(a.tile_stats + (empty ? kEmpty : cls), 1ull);

        // ---- aggregation stream, emit, WTA ----
        const float* col = &sm.ring[0][wx][4 * dq];
        int base = sy + py0 - R - yb;
        base %= G::SR;
        const float* wsm = sm.w[warp] + py0 * RS;
        auto vrow = [&](int pyl) -> float* {
          return G::kAlias ? sm.w[warp] + (py0 + pyl) * RS : sm.val[warp] + (py0 + pyl) * kPX * kDB;
        };
        unsigned long long k[16];
#pragma unroll
        for (int s2 = kPX * HPY; s2 < 16; ++s2) k[s2] = 0ull;
        const int di0 = b * kDB + 4 * dq;
        float pad[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) pad[q] = di0 + q < a.D ? 0.f : -INFINITY;
        auto emit = [&](int pyl, int px, float4 agg, bool padded) {
          const float v0 = padded ? agg.x : agg.x + pad[0], v1 = padded ? agg.y : agg.y + pad[1],
                      v2 = padded ? agg.z : agg.z + pad[2], v3 = padded ? agg.w : agg.w + pad[3];
          const bool h01 = v1 > v0, h23 = v3 > v2;  // equal values keep the smaller d
          const float b01 = h01 ? v1 : v0, b23 = h23 ? v3 : v2;
          const bool h = b23 > b01;
          const int q = h ? 2 + h23 : h01;
          k[pyl * kPX + px] = ((unsigned long long)fkey(h ? b23 : b01) << 32) | (unsigned)(0xffff - (di0 + q));
          if (side == 0) *reinterpret_cast<float4*>(vrow(pyl) + px * kDB + 4 * dq) = agg;
          if constexpr (EXPORT) {
            const int y = sy + py0 + pyl, x = sx + px;
            if (a.expA[side] && x < a.W && y >= a.r0 && y < a.r1) {
              float* er = a.expA[side] + ((size_t)y * a.W + x) * a.D;
              const float av[4] = {agg.x, agg.y, agg.z, agg.w};
#pragma unroll
              for (int q2 = 0; q2 < 4; ++q2)
                if (di0 + q2 < a.D) er[di0 + q2] = av[q2];
            }
          }
        };
        if (cls != kGeneral) {
          float2 num[HPY][kPX][2];
#pragma unroll
          for (int py = 0; py < HPY; ++py)
#pragma unroll
            for (int px = 0; px < kPX; ++px) num[py][px][0] = num[py][px][1] = make_float2(0.f, 0.f);
          float4 head[kPX];
          {
            const float* rp = col + base * (G::SC * kDB);
#pragma unroll
            for (int jj = 0; jj < kPX; ++jj) head[jj] = *reinterpret_cast<const float4*>(rp + jj * kDB);
          }
          if (!(FBS_ABL & 2)) RingRows<G, 0, HPY + 2 * R, HPY>::run(col, base, wsm, head, num);
          __syncwarp();  // every lane is done with the weights before the dead rows are overwritten
#pragma unroll
          for (int pyl = 0; pyl < HPY; ++pyl)
#pragma unroll
            for (int px = 0; px < kPX; ++px) {
              const int pix = (py0 + pyl) * kPX + px;
              float ri[4];
              if (cls == kFast) {
                const float r0 = sm.rinv[warp][pix];
                ri[0] = ri[1] = ri[2] = ri[3] = r0;
              } else {
                const int x = sx + px;
                const int d0 = a.d_min + di0;
                const float* cs = sm.cs[warp][pix];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const int m = side == 0 ? d0 + q + 1 + R - x : a.W - 1 - (d0 + q) + R - x;
                  ri[q] = cs[min(max(m, 0), K1)];
                }
              }
              const float2 n0 = num[pyl][px][0], n1 = num[pyl][px][1];
              float off[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) off[q] = ri[q] > 0.f ? pad[q] : kSent;
              emit(pyl, px, make_float4(__fmaf_rn(n0.x, ri[0], off[0]), __fmaf_rn(n0.y, ri[1], off[1]),
                                        __fmaf_rn(n1.x, ri[2], off[2]), __fmaf_rn(n1.y, ri[3], off[3])), true);
            }
        } else if (empty) {
          // every cost of the unit is undefined: all aggregated costs are SENT (no arithmetic)
#pragma unroll
          for (int pyl = 0; pyl < HPY; ++pyl)
#pragma unroll
            for (int px = 0; px < kPX; ++px) emit(pyl, px, make_float4(kSent, kSent, kSent, kSent), false);
#pragma unroll
          for (int s2 = 0; s2 < kPX * HPY; ++s2) k[s2] = 0ull;  // zero keys never win
        } else {
#pragma unroll
          for (int pyl = 0; pyl < HPY; ++pyl) {
            float2 num[kPX][2], den[kPX][2];
            int bb = base + pyl;
            if (bb >= G::SR) bb -= G::SR;
            ring_num_den_row<G>(col, bb, wsm + pyl * RS, num, den);
            __syncwarp();
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
        const unsigned long long kb = wta_butterfly16(k, lane);  // lane l: slot l & 15 of its half
        __syncwarp();  // the half's aggregated costs (left) are in vrow
        // ---- per-pixel record across d-blocks; maps at the last block ----
        {
          const int s2 = lane & 15;
          const int x = sx + s2 % kPX, y = sy + py0 + s2 / kPX;
          if (s2 < kPX * HPY && x < a.W && y < a.H) {
            const size_t p = ((size_t)f * a.H + y) * a.W + x;
            const bool last = b + 1 == a.nblk;
            unsigned long long kp = 0ull;
            if (b > 0) kp = a.keys[(size_t)side * a.nframes * a.H * a.W + p];
            const unsigned long long kn = kb > kp ? kb : kp;
            if (side == 0) {
              const float* vr = vrow(s2 / kPX) + (s2 % kPX) * kDB;
              float4 rec = b > 0 ? a.agg3[p] : make_float4(kSent, kSent, kSent, kSent);
              if (kb > kp) {
                const int di = 0xffff - (int)(kb & 0xffffu);
                const int l = di - b * kDB;
                rec.x = l > 0 ? vr[l - 1] : rec.w;
                rec.y = vr[l];
                rec.z = di + 1 < a.D ? (l + 1 < kDB ? vr[l + 1] : __int_as_float(0x7fc00001)) : kSent;
              } else if (__float_as_uint(rec.z) == 0x7fc00001u) {
                rec.z = vr[0];  // the best so far was the previous block's last disparity
              }
              rec.w = vr[kDB - 1];
              a.agg3[p] = rec;
            }
            if (!last) a.keys[(size_t)side * a.nframes * a.H * a.W + p] = kn;
            else if (y >= a.r0 && y < a.r1) {
              const bool ok = (unsigned)(kn >> 32) > fkey(kSent);
              a.dmap[side][p] = ok ? a.d_min + (0xffff - (int)(kn & 0xffffu)) : -1;
            }
          }
        }
        __syncthreads();  // (B) the ring rows of this step are dead; weights free
        ++nstep;
      }
    }
    s = we;
  }
}

// LRC (Eq.(9)) + subpixel (Eq.(10)) of rows [r0, r1) of frame blockIdx.z, from
// the walker's maps and per-pixel record (c(d*-1), c(d*), c(d*+1)).
template <bool SCATTER>
__global__ void k_final(const int32_t* __restrict__ dl, const int32_t* __restrict__ dr,
                        const float4* __restrict__ agg3, int W, int H, int r0, int r1, int d_min, int d_max,
                        float* __restrict__ out, const OutSet os) {
  pdl_wait();  // the walker's maps
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = r0 + blockIdx.y;
  if (x >= W || y >= r1) return;
  const size_t p = ((size_t)blockIdx.z * H + y) * W + x;
  const int d = dl[p];
  int e = -1;
  if (d >= 0 && x - d >= 0) e = dr[p - d];
  float c0 = kSent, cm = kSent, cp = kSent;
  if (d >= 0) {
    const float4 v = agg3[p];
    cm = v.x; c0 = v.y; cp = v.z;
  }
  const float v = finalize_pixel(d, e, c0, cm, cp, d_min, d_max);
  if constexpr (!SCATTER) {
    out[((size_t)blockIdx.z * (r1 - r0) + (y - r0)) * W + x] = v;
  } else {
    for (int k = 0; k < os.n; ++k) os.p[k][(size_t)y * W + x] = v;  // band scatter (one frame)
  }
}

}  // namespace fbs
