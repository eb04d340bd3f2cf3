// fbs_ws.cuh — warp-specialised form of the fused walker (k_fbs_ws, ρ <= 4).
//
// The synchronous walker (k_fbs, fbs_fused.cuh) runs its phases one after the
// other in every warp — TMA wait, NCC costs into the ring, weight prologue,
// FFMA2 stream, WTA — with two warps per scheduler and a CTA barrier between
// them, so the FMA pipe idles through every phase but the stream.  Here the 12
// warps of the CTA split the work:
//   producers (warps 8-11)  wait for the TMA-staged rows, compute the twin NCC
//                           cost rows (Eq.(1)) into the shared-memory ring
//                           and issue the next phase's TMA loads;
//   consumers (warps 0-7)   two groups of four; group g takes chunks g, g+2, ...
//                           of CY = 4 output rows x 16 columns: weights
//                           (Eq.(6)-(8)), the FFMA2 stream from the ring, emit,
//                           WTA butterfly, per-pixel record.
// The ring holds NS = 3 CY + 2ρ rows, so while the two consumer groups work on
// chunks c and c+1 the producers already write chunk c+2.  Hand-over: mbarriers
// full[c mod 4] (producers -> group) and empty_ring / empty_w[c mod 4] (group ->
// producers), each arrived on by every thread of the signalling side; TMA
// completion on tbar[phase mod 3].
//
// Ordering rules (c = chunk counter of the CTA, the same in every warp):
//   * chunk c's new cost rows overwrite the rows of chunk c-3's window, so the
//     producers wait empty(c-3) before writing them;
//   * the first phase of a walk (a new strip, side or d-block) writes 2ρ + CY rows
//     of a new window: the producers wait until no chunk is in flight
//     (empty(c-1), empty(c-2));
//   * guide tile buffer c mod 4 is refilled by the TMA for chunk c+4, issued
//     after empty(c) (same chain as above).
#pragma once
#include "fbs_fused.cuh"

namespace fbs {

template <int R>
struct SGeo {
  static constexpr int RR = R;
  static constexpr int K1 = 2 * R + 1;
  static constexpr int HPY = 2;                 // rows per half-warp
  static constexpr int PY = 2 * HPY;            // rows per consumer warp sub-tile
  static constexpr int CY = PY;                 // chunk rows
  static constexpr int TY = CY;                 // (anchoring unit of the row bands)
  static constexpr int NCW = 8, NPW = 8, NW = 16, THREADS = 32 * NW;
  static constexpr int TX = kPX * 4;            // 16
  static constexpr int SC = TX + 2 * R;
  static constexpr int CU = SC / 2;
  static constexpr int NSLOT = 3 * CY + 2 * R;  // ring slots
  static constexpr int SROWS = CY;              // staged rows per producer phase
  static constexpr int NFILL = (2 * R + CY - 1) / CY;
  static constexpr int SPC = (SC + 2 + 3 + 3) / 4 * 4;
  static constexpr int SSC = (SC + 1 + 1) / 2 * 2;
  static constexpr int OPC = (SC + 65 + 3 + 3) / 4 * 4;
  static constexpr int OSC = (SC + 63 + 1 + 1) / 2 * 2;
  static constexpr int GW = (SC + 3) / 4 * 4;
  static constexpr int GWS = GW % 32 == 24 ? GW + 4 : GW;
  static constexpr int GH = CY + 2 * R;
  static constexpr int GSZ = (GH * GWS + 31) / 32 * 32;
  static constexpr int WPW = PY * K1 * K1 * kPX;
  static constexpr bool kAlias = K1 * K1 >= kDB;
  static constexpr unsigned kStageBytes = SROWS * (SPC * 4 + SSC * 8 + OPC * 4 + OSC * 8);
  // staging buffer strides, rounded to 128 B (TMA destinations are 128-B aligned)
  static constexpr int PSZ = (SROWS * SPC + 31) / 32 * 32, POZ = (SROWS * OPC + 31) / 32 * 32;
  static constexpr int SSZ = (SROWS * SSC + 15) / 16 * 16, SOZ = (SROWS * OSC + 15) / 16 * 16;
};

template <int R>
struct SSmem {
  using G = SGeo<R>;
  alignas(128) float ring[G::NSLOT][G::SC][kDB];
  alignas(128) uint32_t Ps[3][G::PSZ];
  alignas(128) uint32_t Po[3][G::POZ];
  alignas(128) int2 Ss[3][G::SSZ];
  alignas(128) int2 So[3][G::SOZ];
  alignas(128) float g[3][G::GSZ];
  // per chunk (3 buffers, chunk c -> c mod 3) and consumer warp of the group
  alignas(16) float w[3][4][G::WPW];  // [py][dy][dx][px]; after the stream: the left aggregated costs
  float rinv[3][4][16];
  float cs[3][4][16][G::K1 + 1];
  int cls[3][4];                      // denominator form (kFast / kEdge / kGeneral / kEmpty)
  float val[G::NCW][G::kAlias ? 4 : G::PY * kPX * kDB];
  uint32_t cwb[4][64];
  unsigned long long tbar[3], full[4], empty_ring[4], empty_w[4];
};

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// The CTA's work, in order: walks (maximal runs of chunks of one (frame, side,
// strip) inside [s_begin, s_end)), per walk the d-blocks, per d-block NFILL fill
// phases then one phase per chunk.  Producers and consumers walk the same list.
// Only the first walk needs a division; later walks start at chunk 0 of the
// next strip.
struct WsSeq {
  long long s, s_end;            // CTA step index of the walk's first chunk; end of the CTA's range
  int nty, nstrips, nblk, nfill;
  int f, side, strip, j0, len;   // the current walk
  int b, k;                      // d-block; phase within (walk, d-block): < nfill fill, else chunk k - nfill
  __device__ __forceinline__ void init(long long s0, long long s1, int nty_, int nstrips_, int nblk_, int nfill_) {
    s = s0; s_end = s1; nty = nty_; nstrips = nstrips_; nblk = nblk_; nfill = nfill_;
    b = 0; k = 0;
    j0 = (int)(s % nty);
    long long q = s / nty;
    strip = (int)(q % nstrips);
    q /= nstrips;
    side = (int)(q & 1);
    f = (int)(q >> 1);
    len = (int)min((long long)(nty - j0), s_end - s);
  }
  __device__ __forceinline__ bool valid() const { return s < s_end; }
  __device__ __forceinline__ bool is_chunk() const { return k >= nfill; }
  __device__ __forceinline__ void advance() {
    if (++k < nfill + len) return;
    k = 0;
    if (++b < nblk) return;
    b = 0;
    s += len;
    j0 = 0;
    if (++strip == nstrips) {
      strip = 0;
      if (++side == 2) { side = 0; ++f; }
    }
    len = (int)min((long long)nty, s_end - s);
  }
};

// Weights w'(p,q) of half a consumer sub-tile (8 pixels: rows 2 pr, 2 pr + 1 of
// the 4x4 sub-tile; Eq.(6)-(8)) by one warp: lane = (tap-row part, pixel), the
// K1 tap rows split in 4 parts; column sums combined across the parts.  Also
// Σ w' (FAST) and the prefix / suffix column-sum reciprocals (EDGE).
template <int R>
__device__ __forceinline__ void ws_weights(const WalkArgs& a, const float* gtile, int wx, int pr, int side, float* wsm,
                                           float* rinv, float (*cs)[2 * R + 2]) {
  using G = SGeo<R>;
  constexpr int K1 = G::K1, GWS = G::GWS;
  const int lane = threadIdx.x & 31;
  const int pix = 8 * pr + (lane & 7), part = lane >> 3;
  const int py = pix / kPX, px = pix % kPX;
  const float* gq = gtile + py * GWS + (wx + px);
  const float gc = gq[R * GWS + R];
  const float gp = gc >= kGuideFlag ? __fsub_rn(gc, kGuideFlag) : gc;
  constexpr int DYP = (K1 + 3) / 4;  // tap rows per part
  float col[K1];
#pragma unroll
  for (int dx = 0; dx < K1; ++dx) col[dx] = 0.f;
#pragma unroll 1
  for (int dyy = 0; dyy < DYP; ++dyy) {
    const int dy = part * DYP + dyy;
    if (dy < K1) {
      float gv[K1];
#pragma unroll
      for (int dx = 0; dx < K1; ++dx) gv[dx] = gq[dy * GWS + dx];
#pragma unroll
      for (int dx = 0; dx < K1; ++dx) {
        const float dd = __fsub_rn(gv[dx], gp);
        float w;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(w) : "f"(__fmaf_rn(__fmul_rn(dd, dd), a.nkr, a.cd[dy * K1 + dx])));
        col[dx] = __fadd_rn(col[dx], w);
        wsm[((py * K1 + dy) * K1 + dx) * kPX + px] = w;
      }
    }
  }
#pragma unroll
  for (int dx = 0; dx < K1; ++dx) {
    col[dx] = __fadd_rn(col[dx], __shfl_xor_sync(0xffffffffu, col[dx], 8));
    col[dx] = __fadd_rn(col[dx], __shfl_xor_sync(0xffffffffu, col[dx], 16));
  }
  if (part == 0) {
    float wsum = 0.f;
#pragma unroll
    for (int dx = 0; dx < K1; ++dx) wsum = __fadd_rn(wsum, col[dx]);
    rinv[pix] = wsum > 0.f ? rcp_nr(wsum) : 0.f;
    float* c = cs[pix];
    float acc = 0.f;
    if (side == 0) {
      c[K1] = 0.f;
#pragma unroll
      for (int dx = K1 - 1; dx >= 0; --dx) {
        acc = __fadd_rn(acc, col[dx]);
        c[dx] = acc > 0.f ? rcp_nr(acc) : 0.f;
      }
    } else {
      c[0] = 0.f;
#pragma unroll
      for (int dx = 0; dx < K1; ++dx) {
        acc = __fadd_rn(acc, col[dx]);
        c[dx + 1] = acc > 0.f ? rcp_nr(acc) : 0.f;
      }
    }
  }
}

// grid: min(total chunks, #SMs) CTAs; block 512 (8 consumer + 8 producer warps); one CTA per SM.
template <int R, bool EXPORT>
__global__ void __launch_bounds__(SGeo<R>::THREADS, 1) k_fbs_ws(const __grid_constant__ WalkArgs a) {
  using G = SGeo<R>;
  constexpr int K1 = G::K1, HPY = G::HPY, CY = G::CY, NS = G::NSLOT;
  constexpr int RS = K1 * K1 * kPX;  // weights per output row
  extern __shared__ __align__(128) unsigned char smraw[];
  SSmem<R>& sm = *reinterpret_cast<SSmem<R>*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long T = a.total;
  const long long s_begin = blockIdx.x * T / gridDim.x, s_end = (blockIdx.x + 1) * T / gridDim.x;
  if (s_begin >= s_end) return;

  if (threadIdx.x == 0) {
    mbar_init(&sm.tbar[0], 1);
    mbar_init(&sm.tbar[1], 1);
    mbar_init(&sm.tbar[2], 1);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      // every thread that wrote (or read) the hand-over data arrives itself, so the
      // release -> acquire edge is direct for each of them (no reliance on a
      // named barrier or __syncwarp in between; racecheck-clean)
      mbar_init(&sm.full[i], G::NPW * 32);
      mbar_init(&sm.empty_ring[i], 4 * 32);
      mbar_init(&sm.empty_w[i], 4 * 32);
    }
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

  WsSeq seq;
  seq.init(s_begin, s_end, a.nty, a.nstrips, a.nblk, G::NFILL);
  auto wait_chunk = [&](unsigned long long* bars, long long j) {
    mbar_wait(&bars[j & 3], (unsigned)((j >> 2) & 1));
  };

  if (warp >= G::NCW) {
    // =========================== producers ===========================
    const int pw = warp - G::NCW;
    const int st = pw & 3, pr = pw >> 2;  // weights: sub-tile st, pixel rows 2 pr .. 2 pr + 1
    const bool leader = threadIdx.x == G::NCW * 32;
    // phase descriptor: frame rows [yc, yc + n) of (f, side, strip, b); chunk output rows from y0
    auto phase = [&](const WsSeq& q, int& yc, int& n, int& y0) {
      const int ya = (a.ty0 + q.j0) * CY;
      if (!q.is_chunk()) {
        yc = ya - R + q.k * CY;
        n = min(CY, 2 * R - q.k * CY);
        y0 = 0;
      } else {
        y0 = ya + (q.k - q.nfill) * CY;
        yc = y0 + R;
        n = CY;
      }
    };
    // TMA three stages deep: phase p's loads are issued at the start of phase p-2
    auto issue = [&](const WsSeq& q, int sb) {
      int yc, n, y0;
      phase(q, yc, n, y0);
      walk_issue_g<G>(a, sm.Ps[sb], sm.Ss[sb], sm.Po[sb], sm.So[sb], q.is_chunk() ? sm.g[sb] : nullptr,
                      &sm.tbar[sb], q.f, q.side, q.strip, q.b, yc, y0);
    };
    WsSeq nx = seq;
    nx.advance();
    if (leader && !(FBS_ABL & 8)) {
      issue(seq, 0);
      if (nx.valid()) issue(nx, 1);
    }
    long long c = 0;  // chunks produced
    int p = 0;        // phases
    int sb = 0;       // p mod 3: staging / guide buffer and TMA barrier of this phase
    unsigned tpar = 0;  // (p / 3) & 1
    int wb = 0;       // c mod 3: weight buffer
    int qrow = 0;     // ring row sequence number of the next produced row
    while (seq.valid()) {
      WsSeq nx2 = nx;
      if (nx2.valid()) nx2.advance();
      const bool chunk = seq.is_chunk();
      unsigned long long* tr = (a.trace && blockIdx.x == 0 && leader && p < 1000) ? a.trace + 4 * p : nullptr;
      if (tr) tr[0] = clock64();
      if (seq.k == 0) {  // a new window: no chunk may still read the ring or its weights
        if (c >= 1) { wait_chunk(sm.empty_ring, c - 1); wait_chunk(sm.empty_w, c - 1); }
        if (c >= 2) { wait_chunk(sm.empty_ring, c - 2); wait_chunk(sm.empty_w, c - 2); }
      } else if (chunk && c >= 3) {
        wait_chunk(sm.empty_ring, c - 3);  // ring rows of chunk c-3's window
        wait_chunk(sm.empty_w, c - 3);     // weight buffer c mod 3
      }
      if (tr) tr[1] = clock64();
      if (leader && nx2.valid() && !(FBS_ABL & 8)) issue(nx2, sb >= 1 ? sb - 1 : 2);  // (p + 2) mod 3
      int yc, n, y0;
      phase(seq, yc, n, y0);
      const int f = seq.f, side = seq.side;
      const int x0 = seq.strip * G::TX;
      const int b = seq.b;
      const int dlo = a.d_min + b * kDB;
      WCw<G> cw(a.W, a.H, a.d_min, a.d_max, side, x0 + st * kPX, y0, b);
      const bool classify = chunk && pr == 1;  // (warp 8, the TMA leader, has pr == 0)
      if (classify) {  // classification words of sub-tile st (global, in flight during the TMA wait)
        const uint32_t* obits = a.bits[1 - side] + (size_t)f * a.H * a.Wb;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int i = lane + 32 * k, row = i >> 2, wd = i & 3;
          if (row < cw.rows && wd < cw.nw) cp_async4(sm.cwb[st] + i, obits + (size_t)(cw.qy0 + row) * a.Wb + cw.w0 + wd);
        }
        cp_async_commit();
      }
      if (!(FBS_ABL & 8)) mbar_wait(&sm.tbar[sb], tpar);
      if (tr) tr[2] = clock64();
      if (!(FBS_ABL & 1)) {
        if (side == 0)
          walk_cost_g<G, 0, EXPORT>(a, sm.ring, sm.Ps[sb], sm.Po[sb], sm.Ss[sb], sm.So[sb], yc, n, qrow % NS, x0, dlo,
                                    pw, G::NPW);
        else
          walk_cost_g<G, 1, EXPORT>(a, sm.ring, sm.Ps[sb], sm.Po[sb], sm.Ss[sb], sm.So[sb], yc, n, qrow % NS, x0, dlo,
                                    pw, G::NPW);
      }
      qrow += n;
      if (chunk && !(FBS_ABL & 4))
        ws_weights<R>(a, sm.g[sb], st * kPX, pr, side, sm.w[wb][st], sm.rinv[wb][st], sm.cs[wb][st]);
      if (classify) {
        cp_async_wait_all();
        __syncwarp();
        bool tex = false, def = false;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int i = lane + 32 * k, row = i >> 2, wd = i & 3;
          if (row < cw.rows && wd < cw.nw) {
            const uint32_t m = cw.mask(cw.w0 + wd), v = sm.cwb[st][i];
            tex |= (~v & m) != 0u;
            def |= (v & m) != 0u;
          }
        }
        const int cl = __any_sync(0xffffffffu, tex) ? kGeneral : (cw.edge ? kEdge : kFast);
        const bool empty = cl == kGeneral && cw.rows > 0 && !__any_sync(0xffffffffu, def);
        if (lane == 0) {
          sm.cls[wb][st] = empty ? kEmpty : cl;
          if (a.tile_stats) atomicAdd(a.tile_stats + (empty ? kEmpty : cl), 1ull);
        }
      }
      named_sync(1, G::NPW * 32);  // the phase's rows / weights are written; its staging buffer is free
      if (tr) tr[3] = clock64() | ((unsigned long long)chunk << 63);
      if (chunk) {
        mbar_arrive(&sm.full[c & 3]);
        ++c;
        if (++wb == 3) wb = 0;
      }
      ++p;
      if (++sb == 3) { sb = 0; tpar ^= 1u; }
      seq = nx;
      nx = nx2;
    }
    return;
  }

  // =========================== consumers ===========================
  const int grp = warp >> 2;  // chunks grp, grp + 2, ...
  const int wq = warp & 3;    // sub-tile within the chunk
  const int wx = wq * kPX;
  const int half = lane >> 4, dq = lane & 15;
  const int py0 = half * HPY;
  long long c = 0;
  int c3 = 0;     // c mod 3 (weight buffer of the next chunk)
  int qrow = 0;   // ring row sequence number: same bookkeeping as the producers
  int qwin = 0;   // sequence number of the current walk window's first row
  for (; seq.valid(); seq.advance()) {
    if (seq.k == 0) qwin = qrow;
    if (!seq.is_chunk()) {
      qrow += min(CY, 2 * R - seq.k * CY);
      continue;
    }
    const int kc = seq.k - seq.nfill;  // chunk index within the walk
    qrow += CY;
    const long long cc = c++;
    const int wb = c3;
    if (++c3 == 3) c3 = 0;
    if ((int)(cc & 1) != grp) continue;
    const int f = seq.f, side = seq.side;
    const int b = seq.b;
    const int x0 = seq.strip * G::TX;
    const int y0 = (a.ty0 + seq.j0 + kc) * CY;
    const int sx = x0 + wx, sy = y0;
    unsigned long long* tr =
        (a.trace && blockIdx.x == 0 && wq == 0 && lane == 0 && cc < 1000) ? a.trace + 4096 + 4 * cc : nullptr;
    if (tr) tr[0] = clock64();
    wait_chunk(sm.full, cc);
    if (tr) tr[1] = clock64();
    const int cls = sm.cls[wb][wq];

    // ---- aggregation stream, emit, WTA ----
    const float* col = &sm.ring[0][wx][4 * dq];
    const int base = (qwin + kc * CY + py0) % NS;  // ring slot of the half's first cost row
    float* wbuf = sm.w[wb][wq];
    const float* wsm = wbuf + py0 * RS;
    auto vrow = [&](int pyl) -> float* {
      return G::kAlias ? wbuf + (py0 + pyl) * RS : sm.val[warp] + (py0 + pyl) * kPX * kDB;
    };
    unsigned long long k[kPX * HPY];
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
        if (a.expA[side] && x < a.W && y < a.H && y >= a.r0 && y < a.r1) {
          float* er = a.expA[side] + ((size_t)y * a.W + x) * a.D;
          const float av[4] = {agg.x, agg.y, agg.z, agg.w};
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2)
            if (di0 + q2 < a.D) er[di0 + q2] = av[q2];
        }
      }
    };
    if (cls == kFast || cls == kEdge) {
      float2 num[HPY][kPX][2];
#pragma unroll
      for (int py = 0; py < HPY; ++py)
#pragma unroll
        for (int px = 0; px < kPX; ++px) num[py][px][0] = num[py][px][1] = make_float2(0.f, 0.f);
      if (!(FBS_ABL & 2)) ring_stream<G, HPY>(col, base, wsm, num);
      __syncwarp();  // every lane is done with the ring and the weights
      mbar_arrive(&sm.empty_ring[cc & 3]);
#pragma unroll
      for (int pyl = 0; pyl < HPY; ++pyl)
#pragma unroll
        for (int px = 0; px < kPX; ++px) {
          const int pix = (py0 + pyl) * kPX + px;
          float ri[4];
          if (cls == kFast) {
            const float r0 = sm.rinv[wb][wq][pix];
            ri[0] = ri[1] = ri[2] = ri[3] = r0;
          } else {
            const int x = sx + px;
            const int d0 = a.d_min + di0;
            const float* cs = sm.cs[wb][wq][pix];
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
    } else if (cls == kEmpty) {
      mbar_arrive(&sm.empty_ring[cc & 3]);
#pragma unroll
      for (int pyl = 0; pyl < HPY; ++pyl)
#pragma unroll
        for (int px = 0; px < kPX; ++px) emit(pyl, px, make_float4(kSent, kSent, kSent, kSent), false);
#pragma unroll
      for (int s2 = 0; s2 < kPX * HPY; ++s2) k[s2] = 0ull;  // zero keys never win
    } else {
      float2 num[HPY][kPX][2], den[HPY][kPX][2];
#pragma unroll
      for (int pyl = 0; pyl < HPY; ++pyl) {
        int bb = base + pyl;
        if (bb >= NS) bb -= NS;
        ring_num_den_row<G>(col, bb, wsm + pyl * RS, num[pyl], den[pyl]);
      }
      __syncwarp();
      mbar_arrive(&sm.empty_ring[cc & 3]);
#pragma unroll
      for (int pyl = 0; pyl < HPY; ++pyl)
#pragma unroll
        for (int px = 0; px < kPX; ++px) {
          const float2 n0 = num[pyl][px][0], n1 = num[pyl][px][1], e0 = den[pyl][px][0], e1 = den[pyl][px][1];
          emit(pyl, px, make_float4(e0.x > 0.f ? __fmul_rn(n0.x, rcp_nr(e0.x)) : kSent,
                                    e0.y > 0.f ? __fmul_rn(n0.y, rcp_nr(e0.y)) : kSent,
                                    e1.x > 0.f ? __fmul_rn(n1.x, rcp_nr(e1.x)) : kSent,
                                    e1.y > 0.f ? __fmul_rn(n1.y, rcp_nr(e1.y)) : kSent), false);
        }
    }
    if (tr) tr[2] = clock64();
    const unsigned long long kb = wta_butterfly8(k, lane);  // lanes l, l ^ 8: slot l & 7 of their half
    __syncwarp();  // the half's aggregated costs (left) are in vrow
    // ---- per-pixel record across d-blocks; maps at the last block ----
    {
      const int s2 = lane & 15;
      const int x = sx + (s2 & 7) % kPX, y = sy + py0 + (s2 & 7) / kPX;
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
    __syncwarp();  // vrow (the weight buffer) is read before it is handed back
    mbar_arrive(&sm.empty_w[cc & 3]);
    if (tr) tr[3] = clock64();
  }
}

}  // namespace fbs
