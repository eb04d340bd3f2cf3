// fbs_agg8.cuh — k_agg8: the volume path's bilateral aggregation + WTA for radii
// 1..4 (every BASELINE configuration), included by fbs_volume.cuh inside
// namespace fbs::vol.  Same arithmetic as k_agg (Eq.(6)-(8); WTA P:L140,
// P:L201), a different lane tile:
//
//   k_agg   lane = 4 disparities x (4 x 3 pixels), two pixel groups per warp
//   k_agg8  lane = 8 disparities x (4 x 4 pixels), four pixel groups per warp
//
// Why (profiles/r02_agg_lsu_budget.txt): the FFMA2 stream is bounded by the SM's
// L1 data pipe, not by the FMA pipe.  A lane receives at most 8 B per wavefront
// (profiles/r02_lds_wavefronts_microbench.txt), so a broadcast weight costs 1/Dl
// wavefronts per FFMA2 (Dl = disparities per lane) and the per-lane cost operands
// 2/n_p (n_p = pixels of the lane tile that use a loaded cost column).  4x3 x 4
// needs 0.25 + 0.27 = 0.52 wavefronts per FFMA2 — with the rest of the kernel 0.69,
// i.e. a 72 % FP32 ceiling; 4x4 x 8 needs 0.125 + 0.22 = 0.35.  The price is 128
// accumulator registers per lane, hence 8 warps per SM (two 4-warp CTAs), each
// streaming with 64 independent FFMA2 chains and cost columns prefetched a few tap
// steps ahead (a loop over cost rows: the unrolled stream does not fit the
// instruction cache).
//
// Per pixel the numerator is summed in the same order as k_agg (cost row, then tap
// column), and the FAST / EDGE denominators come from the same prologue arithmetic,
// so both kernels give identical bits wherever they pick the same denominator form.
#pragma once

namespace a8 {
constexpr int kGP = 4;      // group tile: kGP x kGP pixels
constexpr int kNG = 4;      // pixel groups per warp (8 lanes each), 2 x 2 group tiles
constexpr int kWT = 8;      // warp tile: 8 x 8 pixels
constexpr int kNW = 4;      // warps per CTA (2 x 2 warp tiles)
constexpr int kT = 16;      // CTA tile: 16 x 16 pixels
constexpr int kThreads = 32 * kNW;
constexpr int kCWS = 64;    // classification words per warp (16 rows x 4)
}  // namespace a8
#ifdef FBS_NO_AGG8  // A/B experiment builds: k_agg for every radius
constexpr bool agg8_radius(int) { return false; }
#else
constexpr bool agg8_radius(int R) { return R >= 1 && R <= 4; }
#endif

template <int R>
struct Agg8Smem {
  static constexpr int K1 = 2 * R + 1;
  // weights of one pixel row (pyl) of the four group tiles: [dy][dx][group][px], later
  // that row's aggregated costs [group][px][64] (hence >= 1024); the +8 keeps the four
  // pyl rows of a lane's prologue stores in distinct banks
  static constexpr int PYS = (K1 * K1 * 16 > 1024 ? K1 * K1 * 16 : 1024) + 8;
  static constexpr int WPW = 4 * PYS;  // per warp
  static constexpr int GW = (a8::kT + 2 * R + 3) / 4 * 4, GH = a8::kT + 2 * R;
  static constexpr int GWS = GW % 32 == 24 ? GW + 4 : GW;
  float w[a8::kNW][WPW];        // weights; after the stream of a one-d-block frame: aggregated costs [64 px][64]
  float rinv[a8::kNW][64];      // 1 / Σ_q w'(p,q), 0 if none  (pixel id = group*16 + pyl*4 + px)
  float cs[a8::kNW][64][K1 + 1];  // EDGE: 1 / suffix (left) or prefix (right) column sums
  float g[GH * GWS];            // guide tile
  uint32_t cwb[a8::kNW][2][a8::kCWS];
};

// Denominator form of one 8x8 warp tile (origin sx, sy) for d-block b: the k_agg
// rules (CwRange) over the warp tile's window.
template <int R>
struct Cw8Range {
  int qy0, lo, hi, edge, nw, rows, w0;
  __device__ __forceinline__ Cw8Range(const AggArgs& a, int side, int sx, int sy, int b) {
    qy0 = max(sy - R, 1);
    const int qy1 = min(sy + a8::kWT - 1 + R, a.H - 2);
    const int qx0 = max(sx - R, 1), qx1 = min(sx + a8::kWT - 1 + R, a.W - 2);
    const int d_lo = a.d_min + b * kDB, d_hi = min(d_lo + kDB - 1, a.d_max);
    if (side == 0) { lo = qx0 - d_hi; hi = qx1 - d_lo; edge = lo < 1; lo = max(lo, 1); }
    else { lo = qx0 + d_lo; hi = qx1 + d_hi; edge = hi > a.W - 2; hi = min(hi, a.W - 2); }
    rows = (qy0 <= qy1 && qx0 <= qx1 && lo <= hi) ? qy1 - qy0 + 1 : 0;
    w0 = lo >> 5;
    nw = rows ? (hi >> 5) - w0 + 1 : 0;
  }
};
template <int R>
__device__ __forceinline__ void cw8_load(const AggArgs& a, int side, int sx, int sy, int b, int lane,
                                         uint32_t* cwb) {
  const Cw8Range<R> g(a, side, sx, sy, b);
  const uint32_t* bits = side == 0 ? a.bitsR : a.bitsL;
#pragma unroll
  for (int k = 0; k < a8::kCWS / 32; ++k) {
    const int i = lane + 32 * k, row = i >> 2, wd = i & 3;
    if (row < g.rows && wd < g.nw) cp_async4(cwb + i, bits + (size_t)(g.qy0 + row) * a.Wb + g.w0 + wd);
  }
}
// mode 0: any undefined block in range (-> GENERAL); mode 1: any defined block (EMPTY test)
template <int R, int MODE>
__device__ __forceinline__ bool cw8_any(const AggArgs& a, int side, int sx, int sy, int b, int lane,
                                        const uint32_t* cwb, int& rows) {
  const Cw8Range<R> g(a, side, sx, sy, b);
  bool hit = false;
#pragma unroll
  for (int k = 0; k < a8::kCWS / 32; ++k) {
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

// ---- the FFMA2 stream over the group's NR = 4 + 2R cost rows, as a loop over cost
// rows (the unrolled form, 5,184 FFMA2 per lane at R = 4, overflows the instruction
// cache: ncu no_instruction 3.1 stalls per issue).  Step (r, dx) uses cost columns
// dx .. dx+3 of row r; columns live in a ring of Q = 4 + PF slots indexed by column
// (Q divides NC, so the slot of a column is the same in every row), column dx+3+PF
// (wrapping into row r+1) requested at step dx.
template <int R>
struct Loop8 {
  static constexpr int K1 = 2 * R + 1, NC = a8::kGP + 2 * R, NR = a8::kGP + 2 * R;
  static constexpr int Q = (NC % 2 == 0 && NC / 2 >= 5) ? NC / 2 : NC;
  static constexpr int PF = Q - a8::kGP;
};
template <int R>
__device__ __forceinline__ void stream8(const float* __restrict__ vb, size_t rowstride,
                                        const float* __restrict__ wg, float2 (&num)[a8::kGP][a8::kGP][4]) {
  using G = Loop8<R>;
  constexpr int K1 = G::K1, NC = G::NC, Q = G::Q, PF = G::PF;
  constexpr int PYS = Agg8Smem<R>::PYS;
  float4 ring[Q][2];
  auto ld = [&](const float* rp, int j) {  // column j of row rp (j >= NC: row rp + 1)
    const float* p = j < NC ? rp + j * kDB : rp + rowstride + (j - NC) * kDB;
    ring[j % Q][0] = __ldg(reinterpret_cast<const float4*>(p));
    ring[j % Q][1] = __ldg(reinterpret_cast<const float4*>(p + 4));
  };
#pragma unroll
  for (int j = 0; j < PF; ++j) ld(vb, j);
#pragma unroll 1
  for (int r = 0; r < G::NR; ++r) {
    const float* rp = vb + (size_t)r * rowstride;
#pragma unroll
    for (int dx = 0; dx < K1; ++dx) {
      if (dx == 0) {
#pragma unroll
        for (int j = PF; j < PF + a8::kGP; ++j) ld(rp, j);
      } else {
        ld(rp, dx + a8::kGP - 1 + PF);
      }
#pragma unroll
      for (int pyl = 0; pyl < a8::kGP; ++pyl) {
        const int dy = r - pyl;
        if (dy >= 0 && dy <= 2 * R) {
          const float4 w = *reinterpret_cast<const float4*>(wg + pyl * PYS + (dy * K1 + dx) * 16);
          const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int px = 0; px < a8::kGP; ++px) {
            const float4 c0 = ring[(dx + px) % Q][0], c1 = ring[(dx + px) % Q][1];
            ffma2(num[pyl][px][0], wv[px], make_float2(c0.x, c0.y));
            ffma2(num[pyl][px][1], wv[px], make_float2(c0.z, c0.w));
            ffma2(num[pyl][px][2], wv[px], make_float2(c1.x, c1.y));
            ffma2(num[pyl][px][3], wv[px], make_float2(c1.z, c1.w));
          }
        }
      }
    }
  }
}

// Argmax of a group's 16 pixel slots over its 8 lanes (k[s] = this lane's best key of
// slot s): transposing butterfly, 8+4+2 u64 exchanges; lane dq then holds slots
// 2dq (k[0]) and 2dq+1 (k[1]).
__device__ __forceinline__ void wta_butterfly8(unsigned long long (&k)[16], int lane) {
#pragma unroll
  for (int lvl = 0; lvl < 3; ++lvl) {
    const int n = 8 >> lvl;      // slots kept after this level
    const int m = 4 >> lvl;      // partner lane distance
    const bool up = lane & m;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const unsigned long long keep = up ? k[n + i] : k[i];
      const unsigned long long send = up ? k[i] : k[n + i];
      k[i] = umax64(keep, shfl_xor64(send, m));
    }
  }
}

// grid: (ceil(W/16), tile rows, 2 sides); block 128 = 4 warps of 8x8 pixels.
// EMPTY / EXPORT as for k_agg.
template <int R, bool EMPTY, bool EXPORT>
__global__ void __launch_bounds__(a8::kThreads, 2) k_agg8(const AggArgs a) {
  using SM = Agg8Smem<R>;
  constexpr int K1 = 2 * R + 1, NC = a8::kGP + 2 * R;
  constexpr int GW = SM::GW, GH = SM::GH, GWS = SM::GWS, PYS = SM::PYS;
  extern __shared__ __align__(16) unsigned char smraw[];
  SM& sm = *reinterpret_cast<SM*>(smraw);
  const int side = blockIdx.z;  // 0: left volume / left guide, 1: right
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane >> 3, dq = lane & 7;
  const int x0 = blockIdx.x * a8::kT, y0 = (a.ty0 + blockIdx.y) * a8::kT;
  const int wx = (warp & 1) * a8::kWT, wy = (warp >> 1) * a8::kWT;   // warp tile in the CTA tile
  const int sx = x0 + wx, sy = y0 + wy;                              // warp tile in the frame
  const int gx = sx + (grp & 1) * a8::kGP, gy = sy + (grp >> 1) * a8::kGP;  // group tile

  pdl_trigger();
  pdl_wait();  // everything below reads k_cost's outputs

  {  // guide tile and the first d-block's classification words
    const float* src = (side == 0 ? a.gpadL : a.gpadR) + (size_t)y0 * a.Wg + x0;
    for (int c = threadIdx.x; c < GH * (GW / 4); c += a8::kThreads) {
      const int row = c / (GW / 4), q = c % (GW / 4);
      cp_async16(&sm.g[row * GWS + 4 * q], src + (size_t)row * a.Wg + 4 * q);
    }
    cw8_load<R>(a, side, sx, sy, 0, lane, sm.cwb[warp][0]);
    cp_async_commit();
    cp_async_wait_all();
  }
  __syncthreads();

  // ---- weights w'(p,q) (Eq.(6)-(8)), their sum and the EDGE column sums: lane l
  // takes pixels l and l+32 of the warp (pixel id = group*16 + pyl*4 + px), with
  // k_agg's arithmetic (same expression, same summation order) ----
  float* wsm = sm.w[warp];
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int pid = lane + 32 * h;
    const int pg = pid >> 4, pyl = (pid >> 2) & 3, px = pid & 3;
    const float* gq = sm.g + (wy + (pg >> 1) * a8::kGP + pyl) * GWS + (wx + (pg & 1) * a8::kGP + px);
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
      for (int t = 0; t < NB; ++t) {
        const int dy = dy0 + t / K1, dx = t % K1;
        if (dy < K1) {
          const float dd = __fsub_rn(gv[t], gp);
          float w;
          asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(w) : "f"(__fmaf_rn(__fmul_rn(dd, dd), a.nkr, a.cd[dy * K1 + dx])));
          col[dx] = __fadd_rn(col[dx], w);
          wp[(dy * K1 + dx) * 16] = w;
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
  // one-d-block frames: the aggregated costs of pixel row pyl go into that row's weights
  // once they are dead ([group][px][64] in the PYS floats of row pyl)
  auto vrow = [&](int s) -> float* { return wsm + (s >> 2) * PYS + (grp * a8::kGP + (s & 3)) * kDB; };
  unsigned long long best[2] = {0ull, 0ull};  // running best keys of slots 2dq, 2dq+1
  for (int b = 0; b < a.nblk; ++b) {
    // volume row (gy - R + r) + R = gy + r; column (gx - R + j) + R = gx + j
    const float* vb = vol + vol_at(gy - a.vbase, b, gx, a.nblk, a.Wv) + 8 * dq;
    if (b > 0) {
      cp_async_wait_all();
      __syncthreads();  // lockstep per d-block (k_agg)
    }
    int rows;
    const bool general = cw8_any<R, 0>(a, side, sx, sy, b, lane, sm.cwb[warp][b & 1], rows);
    const int cls = general ? kGeneral : (Cw8Range<R>(a, side, sx, sy, b).edge ? kEdge : kFast);
    __syncwarp();
    if (b + 1 < a.nblk) {
      cw8_load<R>(a, side, sx, sy, b + 1, lane, sm.cwb[warp][(b + 1) & 1]);
      cp_async_commit();
    }
    if (a.tile_stats && lane == 0 && cls != kGeneral) atomicAdd(a.tile_stats + cls, 1ull);
    unsigned long long k[16];
    const int di0 = b * kDB + 8 * dq;
    float pad[8];  // padded disparity slots of the last block never win
#pragma unroll
    for (int t = 0; t < 8; ++t) pad[t] = di0 + t < a.D ? 0.f : -INFINITY;
    // aggregated costs v[0..7] (d = di0 .. di0+7) of slot s -> key, stores
    auto emit = [&](int s, const float (&v)[8]) {
      const int y = gy + (s >> 2), x = gx + (s & 3);
      float bv = v[0];
      int bt = 0;
#pragma unroll
      for (int t = 1; t < 8; ++t)
        if (v[t] > bv) { bv = v[t]; bt = t; }  // equal values keep the smaller d
      k[s] = ((unsigned long long)fkey(bv) << 32) | (unsigned)(0xffff - (di0 + bt));
      const float4 lo4 = make_float4(v[0], v[1], v[2], v[3]), hi4 = make_float4(v[4], v[5], v[6], v[7]);
      if (side == 0) {
        if (a.agg3) {
          float* vr = vrow(s) + 8 * dq;
          *reinterpret_cast<float4*>(vr) = lo4;
          *reinterpret_cast<float4*>(vr + 4) = hi4;
        } else if (x < a.W && y < a.H) {
          float* ap = a.aggL + (((size_t)(y - a.abase) * a.nblk + b) * a.W + x) * kDB + 8 * dq;
          *reinterpret_cast<float4*>(ap) = lo4;
          *reinterpret_cast<float4*>(ap + 4) = hi4;
        }
      } else if ((EXPORT ? a.exportR : nullptr) && x < a.W && y >= a.r0 && y < a.r1) {
        float* er = (EXPORT ? a.exportR : nullptr) + ((size_t)y * a.W + x) * a.D;
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (di0 + t < a.D) er[di0 + t] = v[t];
      }
    };
    if (cls != kGeneral) {
      float2 num[a8::kGP][a8::kGP][4];
#pragma unroll
      for (int i = 0; i < a8::kGP; ++i)
#pragma unroll
        for (int j = 0; j < a8::kGP; ++j)
#pragma unroll
          for (int t = 0; t < 4; ++t) num[i][j][t] = make_float2(0.f, 0.f);
      stream8<R>(vb, rowstride, wg, num);
      if (a.agg3) __syncwarp();  // every lane is done with the weights before they are overwritten
#pragma unroll
      for (int pyl = 0; pyl < a8::kGP; ++pyl)
#pragma unroll
        for (int px = 0; px < a8::kGP; ++px) {
          const int pid = grp * 16 + pyl * 4 + px;
          float ri[8];
          if (cls == kFast) {
            const float r0 = sm.rinv[warp][pid];
#pragma unroll
            for (int t = 0; t < 8; ++t) ri[t] = r0;
          } else {  // EDGE: defined taps are dx >= d + 1 + R - x (left) or dx < W-1-d+R-x (right)
            const int x = gx + px;
            const int d0 = a.d_min + di0;
            const float* cs = sm.cs[warp][pid];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const int m = side == 0 ? d0 + t + 1 + R - x : a.W - 1 - (d0 + t) + R - x;
              ri[t] = cs[min(max(m, 0), K1)];
            }
          }
          float v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const float n = (t & 1) ? num[pyl][px][t >> 1].y : num[pyl][px][t >> 1].x;
            v[t] = __fmaf_rn(n, ri[t], ri[t] > 0.f ? pad[t] : kSent);
          }
          emit(pyl * 4 + px, v);
        }
    } else {
      int er = 0;
      if (EMPTY && !cw8_any<R, 1>(a, side, sx, sy, b, lane, sm.cwb[warp][b & 1], er) && er > 0) {
        if (a.tile_stats && lane == 0) atomicAdd(a.tile_stats + kEmpty, 1ull);
        // every aggregated cost of the unit is SENT and never wins: only the full left
        // store and the debug export need the values
        if (side == 0 && !a.agg3) {
#pragma unroll 1
          for (int s = 0; s < 16; ++s) {
            const int y = gy + (s >> 2), x = gx + (s & 3);
            if (x < a.W && y < a.H) {
              float* ap = a.aggL + (((size_t)(y - a.abase) * a.nblk + b) * a.W + x) * kDB + 8 * dq;
              *reinterpret_cast<float4*>(ap) = make_float4(kSent, kSent, kSent, kSent);
              *reinterpret_cast<float4*>(ap + 4) = make_float4(kSent, kSent, kSent, kSent);
            }
          }
        } else if (side == 1 && (EXPORT ? a.exportR : nullptr)) {
#pragma unroll 1
          for (int s = 0; s < 16; ++s) {
            const int y = gy + (s >> 2), x = gx + (s & 3);
            if (x < a.W && y >= a.r0 && y < a.r1)
              for (int t = 0; t < 8; ++t)
                if (di0 + t < a.D) (EXPORT ? a.exportR : nullptr)[((size_t)y * a.W + x) * a.D + di0 + t] = kSent;
          }
        }
#pragma unroll
        for (int s = 0; s < 16; ++s) k[s] = 0ull;
      } else {
        if (a.tile_stats && lane == 0) atomicAdd(a.tile_stats + kGeneral, 1ull);
        // explicit numerator and denominator, one pixel row at a time (unrolled: the
        // keys k[] stay in registers)
#pragma unroll
        for (int pyl = 0; pyl < a8::kGP; ++pyl) {
          float2 num[a8::kGP][4], den[a8::kGP][4];
#pragma unroll
          for (int px = 0; px < a8::kGP; ++px)
#pragma unroll
            for (int t = 0; t < 4; ++t) num[px][t] = den[px][t] = make_float2(0.f, 0.f);
#pragma unroll 1
          for (int dy = 0; dy < K1; ++dy) {
            const float* rp = vb + (size_t)(pyl + dy) * rowstride;
            float4 c[NC][2];
#pragma unroll
            for (int j = 0; j < NC; ++j) {
              c[j][0] = __ldg(reinterpret_cast<const float4*>(rp + j * kDB));
              c[j][1] = __ldg(reinterpret_cast<const float4*>(rp + j * kDB + 4));
            }
#pragma unroll
            for (int dx = 0; dx < K1; ++dx) {
              const float4 w = *reinterpret_cast<const float4*>(wg + pyl * PYS + (dy * K1 + dx) * 16);
              const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
              for (int px = 0; px < a8::kGP; ++px) {
                const float cc[8] = {c[dx + px][0].x, c[dx + px][0].y, c[dx + px][0].z, c[dx + px][0].w,
                                     c[dx + px][1].x, c[dx + px][1].y, c[dx + px][1].z, c[dx + px][1].w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                  ffma2(num[px][t], wv[px], make_float2(cc[2 * t], cc[2 * t + 1]));
                  ffma2(den[px][t], wv[px], make_float2(is_undef(cc[2 * t]) ? 0.f : 1.f,
                                                        is_undef(cc[2 * t + 1]) ? 0.f : 1.f));
                }
              }
            }
          }
          if (a.agg3) __syncwarp();  // row pyl's weights are dead in every lane before its costs overwrite them
#pragma unroll
          for (int px = 0; px < a8::kGP; ++px) {
            float v[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const float n = (t & 1) ? num[px][t >> 1].y : num[px][t >> 1].x;
              const float e = (t & 1) ? den[px][t >> 1].y : den[px][t >> 1].x;
              v[t] = e > 0.f ? __fmul_rn(n, rcp_nr(e)) + pad[t] : kSent;
            }
            emit(pyl * 4 + px, v);
          }
        }
      }
    }
    wta_butterfly8(k, lane);
    best[0] = umax64(best[0], k[0]);  // earlier blocks win ties (smaller d)
    best[1] = umax64(best[1], k[1]);
  }
  (void)GW;
  // ---- epilogue: lane dq holds slots 2dq, 2dq+1 of its group ----
  if (a.agg3) __syncwarp();  // the group's on-chip costs are complete
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int s = 2 * dq + i;
    const int x = gx + (s & 3), y = gy + (s >> 2);
    if (x < a.W && y >= a.r0 && y < a.r1) {
      const bool ok = (unsigned)(best[i] >> 32) > fkey(kSent);
      const int d_int = ok ? a.d_min + (0xffff - (int)(best[i] & 0xffffu)) : -1;
      (side == 0 ? a.dL : a.dR)[(size_t)y * a.W + x] = d_int;
      if (side == 0 && a.agg3 && ok) {  // the three costs Eq.(10) needs
        const float* vr = vrow(s);
        const int di = d_int - a.d_min;
        a.agg3[(size_t)y * a.W + x] =
            make_float4(di > 0 ? vr[di - 1] : kSent, vr[di], di + 1 < a.D ? vr[di + 1] : kSent, 0.f);
      }
    }
  }
}
