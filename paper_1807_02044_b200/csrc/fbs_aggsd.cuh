// fbs_aggsd.cuh — k_aggsd: the volume path's bilateral aggregation + WTA for small
// disparity ranges (D <= 16, radii 1..5: the Tsukuba-shaped BASELINE config), included
// by fbs_volume.cuh inside namespace fbs::vol.  Same arithmetic as k_agg (Eq.(6)-(8),
// P:L118-132; WTA P:L140), a lane mapping without disparity padding:
//
//   k_agg   half-warp (16 lanes x 4 disparities = a 64-disparity block) per 4x3 pixels:
//           at D = 16, 75 % of every FFMA2 is padding
//   k_aggsd 8-lane group (8 lanes x 2 disparities = 16) per 4x3 pixels, four groups
//           per warp (a 2x2 arrangement: the warp covers 8x6 pixels, the CTA of four
//           warps the same 16x12 tile as k_agg)
//
// Per lane the accumulators are 12 pixels x 2 disparities.  A broadcast weight float4
// (4 pixels, four groups' addresses in disjoint banks: 2 wavefronts,
// profiles/r02_lds_wavefronts_microbench.txt) now feeds 4 FFMA2 instead of 8, and a
// cost load is 8 B per lane: 0.77 L1 wavefronts per FFMA2 instead of 0.52
// (profiles/r02_agg_lsu_budget.txt), for a quarter of the FFMA2s.  The weights of 48
// pixels per warp limit the SM to three 4-warp CTAs (12 warps).
//
// Per pixel the numerator is summed in k_agg's order (cost row, then tap column) and the
// FAST / EDGE denominators come from k_agg's prologue arithmetic.
#pragma once

namespace sd {
constexpr int kGP = 4;      // group tile width (pixels)
constexpr int kGY = 3;      // group tile height
constexpr int kWX = 8, kWY = 6;   // warp tile (2 x 2 group tiles)
constexpr int kNW = 4;      // warps per CTA (2 x 2 warp tiles): CTA tile 16 x 12 (= k_agg's)
constexpr int kThreads = 32 * kNW;
constexpr int kD = 16;      // disparities per group (8 lanes x 2)
constexpr int kCWS = 64;    // classification words per warp (<= 16 rows x 4)
constexpr int kNPX = 48;    // pixels per warp
}  // namespace sd
constexpr bool aggsd_ok(int R, int D) { return R >= 1 && R <= 5 && D <= sd::kD; }

template <int R>
struct AggSdSmem {
  static constexpr int K1 = 2 * R + 1;
  // weights of one pixel row (pyl) of the four group tiles: [dy][dx][group][px], later
  // that row's aggregated costs [group][px][16]; the +8 spreads the rows over banks
  static constexpr int PYS = (K1 * K1 * 16 > 256 ? K1 * K1 * 16 : 256) + 8;
  static constexpr int WPW = sd::kGY * PYS;
  static constexpr int GW = (16 + 2 * R + 3) / 4 * 4, GH = 12 + 2 * R;
  static constexpr int GWS = GW % 32 == 24 ? GW + 4 : GW;
  float w[sd::kNW][WPW];
  float rinv[sd::kNW][sd::kNPX];          // pixel id = group*12 + pyl*4 + px
  float cs[sd::kNW][sd::kNPX][K1 + 1];
  float g[GH * GWS];
  uint32_t cwb[sd::kNW][sd::kCWS];
};

// Denominator form of one 8x6 warp tile (origin sx, sy): k_agg's rules over the warp
// tile's window and the whole (single, <= 16) disparity range.
template <int R>
struct CwSdRange {
  int qy0, lo, hi, edge, nw, rows, w0;
  __device__ __forceinline__ CwSdRange(const AggArgs& a, int side, int sx, int sy) {
    qy0 = max(sy - R, 1);
    const int qy1 = min(sy + sd::kWY - 1 + R, a.H - 2);
    const int qx0 = max(sx - R, 1), qx1 = min(sx + sd::kWX - 1 + R, a.W - 2);
    const int d_lo = a.d_min, d_hi = a.d_max;
    if (side == 0) { lo = qx0 - d_hi; hi = qx1 - d_lo; edge = lo < 1; lo = max(lo, 1); }
    else { lo = qx0 + d_lo; hi = qx1 + d_hi; edge = hi > a.W - 2; hi = min(hi, a.W - 2); }
    rows = (qy0 <= qy1 && qx0 <= qx1 && lo <= hi) ? qy1 - qy0 + 1 : 0;
    w0 = lo >> 5;
    nw = rows ? (hi >> 5) - w0 + 1 : 0;
  }
};
// mode 0: any undefined block in range (-> GENERAL); mode 1: any defined block (EMPTY test)
template <int R, int MODE>
__device__ __forceinline__ bool cwsd_any(const AggArgs& a, int side, int sx, int sy, int lane,
                                         const uint32_t* cwb, int& rows) {
  const CwSdRange<R> g(a, side, sx, sy);
  bool hit = false;
#pragma unroll
  for (int k = 0; k < sd::kCWS / 32; ++k) {
    const int i = lane + 32 * k, row = i >> 2, wd = i & 3;
    if (row < g.rows && wd < g.nw) {
      const int wi = g.w0 + wd;
      uint32_t m = 0xffffffffu;
      if (wi == g.w0) m &= 0xffffffffu << (g.lo & 31);
      if (wi == (g.hi >> 5)) m &= 0xffffffffu >> (31 - (g.hi & 31));
      hit |= ((MODE == 0 ? ~cwb[i] : cwb[i]) & m) != 0u;
    }
  }
  rows = g.rows;
  return __any_sync(0xffffffffu, hit);
}

// num[pyl][px] += Σ_dx w(pyl, r - pyl, dx, px) · c[px + dx]  for cost row r
template <int R, int r>
__device__ __forceinline__ void row_fma_sd(const float2* c, const float* __restrict__ wg,
                                           float2 (&num)[sd::kGY][sd::kGP]) {
  constexpr int K1 = 2 * R + 1;
#pragma unroll
  for (int dx = 0; dx < K1; ++dx) {
#pragma unroll
    for (int pyl = 0; pyl < sd::kGY; ++pyl) {
      const int dy = r - pyl;
      if (dy >= 0 && dy <= 2 * R) {
        const float4 w = *reinterpret_cast<const float4*>(wg + pyl * AggSdSmem<R>::PYS + (dy * K1 + dx) * 16);
        const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int px = 0; px < sd::kGP; ++px) ffma2(num[pyl][px], wv[px], c[dx + px]);
      }
    }
  }
}
// Cost rows of the stream (k_agg's Rows4 with 2 disparities per lane): the first
// kGP columns of row r+1 are in flight while row r is consumed.
template <int R, int r, int NR>
struct RowsSd {
  static __device__ __forceinline__ void run(const float* __restrict__ vb, size_t rowstride,
                                             const float* __restrict__ wg, float2 (&head)[sd::kGP],
                                             float2 (&num)[sd::kGY][sd::kGP]) {
    constexpr int NC = sd::kGP + 2 * R;
    float2 c[NC];
    const float* rp = vb + (size_t)r * rowstride;
#pragma unroll
    for (int j = 0; j < sd::kGP; ++j) c[j] = head[j];
#pragma unroll
    for (int j = sd::kGP; j < NC; ++j) c[j] = __ldg(reinterpret_cast<const float2*>(rp + j * kDB));
    if constexpr (r + 1 < NR) {
#pragma unroll
      for (int j = 0; j < sd::kGP; ++j) head[j] = __ldg(reinterpret_cast<const float2*>(rp + rowstride + j * kDB));
    }
    row_fma_sd<R, r>(c, wg, num);
    RowsSd<R, r + 1, NR>::run(vb, rowstride, wg, head, num);
  }
};
template <int R, int NR>
struct RowsSd<R, NR, NR> {
  static __device__ __forceinline__ void run(const float*, size_t, const float*, float2 (&)[sd::kGP],
                                             float2 (&)[sd::kGY][sd::kGP]) {}
};

// Argmax of a group's 16 slots over its 8 lanes: transposing butterfly, 8+4+2 u64
// exchanges; lane dq then holds slots 2dq (k[0]) and 2dq+1 (k[1]).
__device__ __forceinline__ void wta_butterfly_g8(unsigned long long (&k)[16], int lane) {
#pragma unroll
  for (int lvl = 0; lvl < 3; ++lvl) {
    const int n = 8 >> lvl;
    const int m = 4 >> lvl;
    const bool up = lane & m;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const unsigned long long keep = up ? k[n + i] : k[i];
      const unsigned long long send = up ? k[i] : k[n + i];
      k[i] = umax64(keep, shfl_xor64(send, m));
    }
  }
}

// grid: (ceil(W/16), tile rows, 2 sides); block 128 = 4 warps of 8x6 pixels.
// EMPTY / EXPORT as for k_agg.  One d-block (D <= 16).
template <int R, bool EMPTY, bool EXPORT>
__global__ void __launch_bounds__(sd::kThreads, 3) k_aggsd(const AggArgs a) {
  using SM = AggSdSmem<R>;
  constexpr int K1 = 2 * R + 1, NC = sd::kGP + 2 * R;
  constexpr int GW = SM::GW, GH = SM::GH, GWS = SM::GWS, PYS = SM::PYS;
  extern __shared__ __align__(16) unsigned char smraw[];
  SM& sm = *reinterpret_cast<SM*>(smraw);
  const int side = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane >> 3, dq = lane & 7;
  const int x0 = blockIdx.x * 16, y0 = (a.ty0 + blockIdx.y) * 12;
  const int wx = (warp & 1) * sd::kWX, wy = (warp >> 1) * sd::kWY;
  const int sx = x0 + wx, sy = y0 + wy;
  const int gx = sx + (grp & 1) * sd::kGP, gy = sy + (grp >> 1) * sd::kGY;

  pdl_trigger();
  pdl_wait();  // everything below reads k_cost's outputs

  {  // guide tile and the classification words, in flight together
    const float* src = (side == 0 ? a.gpadL : a.gpadR) + (size_t)y0 * a.Wg + x0;
    for (int c = threadIdx.x; c < GH * (GW / 4); c += sd::kThreads) {
      const int row = c / (GW / 4), q = c % (GW / 4);
      cp_async16(&sm.g[row * GWS + 4 * q], src + (size_t)row * a.Wg + 4 * q);
    }
    const CwSdRange<R> g(a, side, sx, sy);
    const uint32_t* bits = side == 0 ? a.bitsR : a.bitsL;
#pragma unroll
    for (int k = 0; k < sd::kCWS / 32; ++k) {
      const int i = lane + 32 * k, row = i >> 2, wd = i & 3;
      if (row < g.rows && wd < g.nw) cp_async4(sm.cwb[warp] + i, bits + (size_t)(g.qy0 + row) * a.Wb + g.w0 + wd);
    }
    cp_async_commit();
    cp_async_wait_all();
  }
  __syncthreads();

  // ---- weights (k_agg's arithmetic): lane l takes pixels l and l+32 (< 48) ----
  float* wsm = sm.w[warp];
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int pid = lane + 32 * h;
    if (pid >= sd::kNPX) break;
    const int pg = pid / 12, pyl = (pid % 12) >> 2, px = pid & 3;
    const float* gq = sm.g + (wy + (pg >> 1) * sd::kGY + pyl) * GWS + (wx + (pg & 1) * sd::kGP + px);
    const float gc = gq[R * GWS + R];
    const float gp = gc >= kGuideFlag ? __fsub_rn(gc, kGuideFlag) : gc;
    float col[K1];
#pragma unroll
    for (int dx = 0; dx < K1; ++dx) col[dx] = 0.f;
    float* wp = wsm + pyl * PYS + pg * 4 + px;
    constexpr int CH = (K1 * K1 <= 64) ? K1 : (64 / K1 > 0 ? 64 / K1 : 1);
#pragma unroll
    for (int dy0 = 0; dy0 < K1; dy0 += CH) {
      constexpr int NB = CH * K1;
      float gv[NB];
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int dy = dy0 + t / K1, dx = t % K1;
        gv[t] = dy < K1 ? gq[dy * GWS + dx] : 0.f;
      }
#pragma unroll
      for (int t = 0; t < NB; ++t) {  // adjacent taps of a row in pairs (k_agg's tap_pair)
        const int dy = dy0 + t / K1, dx = t % K1;
        if (dy >= K1 || (dx & 1)) continue;
        if (dx + 1 < K1) {
          float w0, w1;
          tap_pair(gv[t], gv[t + 1], gp, a.nkr, a.cd[dy * K1 + dx], a.cd[dy * K1 + dx + 1], w0, w1, col[dx],
                   col[dx + 1]);
          wp[(dy * K1 + dx) * 16] = w0;
          wp[(dy * K1 + dx + 1) * 16] = w1;
        } else {
          wp[(dy * K1 + dx) * 16] = tap_one(gv[t], gp, a.nkr, a.cd[dy * K1 + dx], col[dx]);
        }
      }
    }
    float wsum = 0.f;
#pragma unroll
    for (int dx = 0; dx < K1; ++dx) wsum = __fadd_rn(wsum, col[dx]);
    sm.rinv[warp][pid] = wsum > 0.f ? rcp_nr(wsum) : 0.f;
    float* cs = sm.cs[warp][pid];
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
  const float* wg = wsm + grp * 4;
  // on-chip aggregated costs of slot s (pixel row s >> 2) in that row's dead weights
  auto vrow = [&](int s) -> float* { return wsm + (s >> 2) * PYS + (grp * sd::kGP + (s & 3)) * sd::kD; };
  // volume row (gy - R + r) + R = gy + r; column (gx - R + j) + R = gx + j
  const float* vb = vol + vol_at(gy - a.vbase, 0, gx, a.nblk, a.Wv) + 2 * dq;
  int rows;
  const bool general = cwsd_any<R, 0>(a, side, sx, sy, lane, sm.cwb[warp], rows);
  const int cls = general ? kGeneral : (CwSdRange<R>(a, side, sx, sy).edge ? kEdge : kFast);
  if (a.tile_stats && lane == 0 && cls != kGeneral) atomicAdd(a.tile_stats + cls, 1ull);
  unsigned long long k[16];
#pragma unroll
  for (int s = sd::kGY * sd::kGP; s < 16; ++s) k[s] = 0ull;
  const int di0 = 2 * dq;
  float pad[2];  // disparities beyond D never win
#pragma unroll
  for (int t = 0; t < 2; ++t) pad[t] = di0 + t < a.D ? 0.f : -INFINITY;
  // aggregated costs (d = di0, di0+1) of slot s -> key, stores
  auto emit = [&](int s, float v0, float v1) {
    const int y = gy + (s >> 2), x = gx + (s & 3);
    const bool h1 = v1 > v0;  // equal values keep the smaller d
    k[s] = ((unsigned long long)fkey(h1 ? v1 : v0) << 32) | (unsigned)(0xffff - (di0 + h1));
    if (side == 0) {
      if (a.agg3) {
        *reinterpret_cast<float2*>(vrow(s) + di0) = make_float2(v0, v1);
      } else if (x < a.W && y < a.H) {
        *reinterpret_cast<float2*>(a.aggL + ((size_t)(y - a.abase) * a.nblk * a.W + x) * kDB + di0) =
            make_float2(v0, v1);
      }
    } else if ((EXPORT ? a.exportR : nullptr) && x < a.W && y >= a.r0 && y < a.r1) {
      float* er = (EXPORT ? a.exportR : nullptr) + ((size_t)y * a.W + x) * a.D;
      if (di0 < a.D) er[di0] = v0;
      if (di0 + 1 < a.D) er[di0 + 1] = v1;
    }
  };
  if (cls != kGeneral) {
    float2 num[sd::kGY][sd::kGP];
#pragma unroll
    for (int i = 0; i < sd::kGY; ++i)
#pragma unroll
      for (int j = 0; j < sd::kGP; ++j) num[i][j] = make_float2(0.f, 0.f);
    {
      float2 head[sd::kGP];
#pragma unroll
      for (int j = 0; j < sd::kGP; ++j) head[j] = __ldg(reinterpret_cast<const float2*>(vb + j * kDB));
      RowsSd<R, 0, sd::kGY + 2 * R>::run(vb, rowstride, wg, head, num);
    }
    if (a.agg3) __syncwarp();  // every lane is done with the weights before they are overwritten
#pragma unroll
    for (int pyl = 0; pyl < sd::kGY; ++pyl)
#pragma unroll
      for (int px = 0; px < sd::kGP; ++px) {
        const int pid = grp * 12 + pyl * 4 + px;
        float ri[2];
        if (cls == kFast) {
          ri[0] = ri[1] = sm.rinv[warp][pid];
        } else {  // EDGE: defined taps are dx >= d + 1 + R - x (left) or dx < W-1-d+R-x (right)
          const int x = gx + px;
          const int d0 = a.d_min + di0;
          const float* cs = sm.cs[warp][pid];
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int m = side == 0 ? d0 + t + 1 + R - x : a.W - 1 - (d0 + t) + R - x;
            ri[t] = cs[min(max(m, 0), K1)];
          }
        }
        const float2 n = num[pyl][px];
        emit(pyl * 4 + px, __fmaf_rn(n.x, ri[0], ri[0] > 0.f ? pad[0] : kSent),
             __fmaf_rn(n.y, ri[1], ri[1] > 0.f ? pad[1] : kSent));
      }
  } else {
    int er = 0;
    if (EMPTY && !cwsd_any<R, 1>(a, side, sx, sy, lane, sm.cwb[warp], er) && er > 0) {
      if (a.tile_stats && lane == 0) atomicAdd(a.tile_stats + kEmpty, 1ull);
      // every aggregated cost of the unit is SENT and never wins
      if (side == 0 && !a.agg3) {
#pragma unroll 1
        for (int s = 0; s < sd::kGY * sd::kGP; ++s) {
          const int y = gy + (s >> 2), x = gx + (s & 3);
          if (x < a.W && y < a.H)
            *reinterpret_cast<float2*>(a.aggL + ((size_t)(y - a.abase) * a.nblk * a.W + x) * kDB + di0) =
                make_float2(kSent, kSent);
        }
      } else if (side == 1 && (EXPORT ? a.exportR : nullptr)) {
#pragma unroll 1
        for (int s = 0; s < sd::kGY * sd::kGP; ++s) {
          const int y = gy + (s >> 2), x = gx + (s & 3);
          if (x < a.W && y >= a.r0 && y < a.r1)
            for (int t = 0; t < 2; ++t)
              if (di0 + t < a.D) (EXPORT ? a.exportR : nullptr)[((size_t)y * a.W + x) * a.D + di0 + t] = kSent;
        }
      }
#pragma unroll
      for (int s = 0; s < sd::kGY * sd::kGP; ++s) k[s] = 0ull;
    } else {
      if (a.tile_stats && lane == 0) atomicAdd(a.tile_stats + kGeneral, 1ull);
      // explicit numerator and denominator, one pixel row at a time
#pragma unroll
      for (int pyl = 0; pyl < sd::kGY; ++pyl) {
        float2 num[sd::kGP], den[sd::kGP];
#pragma unroll
        for (int px = 0; px < sd::kGP; ++px) num[px] = den[px] = make_float2(0.f, 0.f);
#pragma unroll 1
        for (int dy = 0; dy < K1; ++dy) {
          const float* rp = vb + (size_t)(pyl + dy) * rowstride;
          float2 c[NC];
#pragma unroll
          for (int j = 0; j < NC; ++j) c[j] = __ldg(reinterpret_cast<const float2*>(rp + j * kDB));
#pragma unroll
          for (int dx = 0; dx < K1; ++dx) {
            const float4 w = *reinterpret_cast<const float4*>(wg + pyl * PYS + (dy * K1 + dx) * 16);
            const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int px = 0; px < sd::kGP; ++px) {
              const float2 cc = c[dx + px];
              ffma2(num[px], wv[px], cc);
              ffma2(den[px], wv[px], make_float2(is_undef(cc.x) ? 0.f : 1.f, is_undef(cc.y) ? 0.f : 1.f));
            }
          }
        }
        if (a.agg3) __syncwarp();  // row pyl's weights are dead in every lane
#pragma unroll
        for (int px = 0; px < sd::kGP; ++px) {
          const float2 n = num[px], e = den[px];
          emit(pyl * 4 + px, (e.x > 0.f ? __fmul_rn(n.x, rcp_nr(e.x)) : kSent) + pad[0],
               (e.y > 0.f ? __fmul_rn(n.y, rcp_nr(e.y)) : kSent) + pad[1]);
        }
      }
    }
  }
  wta_butterfly_g8(k, lane);

  // ---- epilogue: lane dq holds slots 2dq, 2dq+1 of its group ----
  if (a.agg3) __syncwarp();  // the group's on-chip costs are complete
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int s = 2 * dq + i;
    if (s >= sd::kGY * sd::kGP) continue;
    const int x = gx + (s & 3), y = gy + (s >> 2);
    if (x < a.W && y >= a.r0 && y < a.r1) {
      const bool ok = (unsigned)(k[i] >> 32) > fkey(kSent);
      const int d_int = ok ? a.d_min + (0xffff - (int)(k[i] & 0xffffu)) : -1;
      (side == 0 ? a.dL : a.dR)[(size_t)y * a.W + x] = d_int;
      if (side == 0 && a.agg3 && ok) {  // the three costs Eq.(10) needs
        const float* vr = vrow(s);
        const int di = d_int - a.d_min;
        a.agg3[(size_t)y * a.W + x] =
            make_float4(di > 0 ? vr[di - 1] : kSent, vr[di], di + 1 < a.D ? vr[di + 1] : kSent, 0.f);
      }
    }
  }
  (void)GW;
}
