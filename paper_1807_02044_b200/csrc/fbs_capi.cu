// fbs_capi.cu — C ABI of libfbs.so (declared in include/fbs.h).
//
// Host side: parameter validation, the ω_d / ω_r exponent constants (Eq.(7)(8),
// built in double and rounded once to fp32, "pre-calculated"), scratch
// allocation, TMA descriptors, and the launch sequence.  Two paths compute the
// same function:
//   FBS_PATH_VOLUME (default, fbs_volume.cuh): k_cost -> L2/HBM cost volumes ->
//                    k_agg -> k_finalize, one frame per launch sequence;
//   FBS_PATH_FUSED (fbs_fused.cuh, fbs_ws.cuh): 3 launches per batch of frames,
//                    programmatic dependent launch between them:
//   k_prep   block statistics, packed columns, guides, masks   Eq.(2)(3)
//   k_fbs    twin NCC costs in shared memory + aggregation    Eq.(1); Eq.(6)-(8)
//            + WTA, both sides, all frames of the batch
//   k_final  LRC + subpixel -> disp_out                        Eq.(9)(10)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <type_traits>
#include <utility>

#include <cuda.h>

#include "../../include/fbs.h"
#include "fbs_ws.cuh"
#include "fbs_volume.cuh"

// Radii instantiated per kernel family.  FBS_EXP_ONLY_R4 (experiment builds of
// tools/build_variants.py only) compiles radius 4 alone; other radii then fail
// with cudaErrorInvalidValue at launch.
#ifdef FBS_EXP_ONLY_R4
#define FBS_VOL_RADII(M) M(4)
#define FBS_SD_RADII(M) M(4)
#define FBS_WS_RADII(M) M(4)
#define FBS_SYNC_RADII(M)
#else
#define FBS_VOL_RADII(M) M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10)
#define FBS_SD_RADII(M) M(1) M(2) M(3) M(4) M(5)
#define FBS_WS_RADII(M) M(0) M(1) M(2) M(3) M(4)
#define FBS_SYNC_RADII(M) M(5) M(6)
#endif

using namespace fbs;

struct fbs_ctx {
  WalkArgs wa;  // tensor maps, geometry and the Eq.(7)(8) constants (first: 64-B aligned)
  int path;     // FBS_PATH_VOLUME / FBS_PATH_FUSED
  int W, H, d_min, d_max, D, nblk, R;
  float sigma_s, sigma_r;
  int device, num_sms;
  int fcap;  // frames per launch (scratch is sized for fcap frames)
  int Wp, Wg, GR, Wb, TY, TX;
  size_t gfs;  // guide frame stride (floats)
  // scratch (fcap frames each)
  uint32_t* P[2];
  int2* SR[2];
  float* G[2];
  uint32_t* bits[2];
  int32_t* dmap[2];
  float4* agg3;
  unsigned long long* keys;
  // volume path scratch (fbs_volume.cuh): padded cost volumes [Hv][nblk][Wv][64] per side,
  // padded guides, block-defined masks, the left aggregated volume (multi-block frames)
  int Wv, Hv, vWb, vWg;
  int rb0, rb1;        // rows this handle serves (band handles: fbs_create_band), else [0, H)
  int vbase, abase;    // frame row of volume row R / of aggL row 0 (band handles), else 0
  int arows;           // rows of aggL
  float *volL, *volR, *gpadL, *gpadR, *aggL;
  uint32_t *vbitsL, *vbitsR;
  int* rtiles;  // fbs_suggest_ranges: (min, max) per 16x16 tile, left then right
  // host path (fbs_compute_host[_batch]): two frame slots each, created on first use
  bool staging_ready;
  uint8_t *hL, *hR;
  float* hOut;
  cudaStream_t cs_in, cs_out;
  cudaEvent_t ev_entry, ev_in[2], ev_done[2], ev_out[2];
  unsigned long long* tile_stats;  // device [4] FAST/EDGE/GENERAL/EMPTY, counting while profiling
  unsigned long long* trace;       // FBS_TRACE builds: kernel timeline of CTA 0
  int launches;
  OutSet scat;  // fbs_compute_rows_scatter: destinations of the current call (n = 0 otherwise)
  cudaEvent_t* prof_ev;  // live profiling (fbs_profile_enable): kEv events per call
  int prof_cap, prof_n;
};

static thread_local std::string g_err;
static constexpr int kEv = FBS_NSTAGES + 1;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
static int cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(FBS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return FBS_OK;
}

extern "C" const char* fbs_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------------------
// Geometry per radius (the walker's compile-time traits): ρ <= 4 runs the
// warp-specialised walker (SGeo, fbs_ws.cuh), ρ = 5, 6 the synchronous one (WGeo).
template <int R>
using Geo = typename std::conditional<(R <= kWsMaxRadius), SGeo<R>, WGeo<R>>::type;
template <int R>
static void geo_of(int& TX, int& TY, size_t& smem, int& threads) {
  TX = Geo<R>::TX;
  TY = Geo<R>::TY;
  threads = Geo<R>::THREADS;
  smem = (R <= kWsMaxRadius ? sizeof(SSmem<R <= kWsMaxRadius ? R : 0>) : sizeof(WSmem<R>)) + 128;  // + alignment slack
}
static void geometry(int R, int& TX, int& TY, size_t& smem, int& threads) {
  switch (R) {
#define FBS_GEO(RR) \
  case RR: geo_of<RR>(TX, TY, smem, threads); break;
    FBS_GEO(0) FBS_GEO(1) FBS_GEO(2) FBS_GEO(3) FBS_GEO(4) FBS_GEO(5) FBS_GEO(6)
#undef FBS_GEO
  }
}

// ---------------------------------------------------------------------------
// TMA descriptors (driver entry point, no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}

// 3-D map over [F][rows][cols] elements of esize bytes (row pitch `pitch` elements);
// out-of-range elements read as zero (an undefined block / no packed column).
static bool make_map(CUtensorMap* m, void* base, CUtensorMapDataType dt, int esize, int cols, int rows, int pitch,
                     int frames, int box_cols, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)frames};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch * esize, (cuuint64_t)pitch * esize * rows};
  const cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(m, dt, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int R>
static bool make_maps(fbs_ctx* h) {
  using G = Geo<R>;
  bool ok = true;
  for (int im = 0; im < 2; ++im) {
    ok &= make_map(&h->wa.tmPs[im], h->P[im], CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, h->W, h->H, h->Wp, h->fcap, G::SPC,
                   G::SROWS);
    ok &= make_map(&h->wa.tmPo[im], h->P[im], CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, h->W, h->H, h->Wp, h->fcap, G::OPC,
                   G::SROWS);
    // (S, r) pairs as 32-bit words: x coordinates are doubled
    ok &= make_map(&h->wa.tmSs[im], h->SR[im], CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, 2 * h->W, h->H, 2 * h->Wp, h->fcap,
                   2 * G::SSC, G::SROWS);
    ok &= make_map(&h->wa.tmSo[im], h->SR[im], CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, 2 * h->W, h->H, 2 * h->Wp, h->fcap,
                   2 * G::OSC, G::SROWS);
    ok &= make_map(&h->wa.tmG[im], h->G[im], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, h->Wg, h->GR, h->Wg, h->fcap, G::GWS,
                   G::GH);
  }
  return ok;
}
static bool build_maps(fbs_ctx* h) {
  switch (h->R) {
#define FBS_MAPS(RR) \
  case RR: return make_maps<RR>(h);
    FBS_MAPS(0) FBS_MAPS(1) FBS_MAPS(2) FBS_MAPS(3) FBS_MAPS(4) FBS_MAPS(5) FBS_MAPS(6)
#undef FBS_MAPS
  }
  return false;
}

// ---------------------------------------------------------------------------
static void free_host_path(fbs_ctx* h) {
  if (h->cs_in) cudaStreamDestroy(h->cs_in);
  if (h->cs_out) cudaStreamDestroy(h->cs_out);
  cudaEvent_t evs[] = {h->ev_entry, h->ev_in[0], h->ev_in[1], h->ev_done[0], h->ev_done[1], h->ev_out[0], h->ev_out[1]};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  void* ptrs[] = {h->hL, h->hR, h->hOut};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  h->cs_in = h->cs_out = nullptr;
  h->ev_entry = h->ev_in[0] = h->ev_in[1] = h->ev_done[0] = h->ev_done[1] = h->ev_out[0] = h->ev_out[1] = nullptr;
  h->hL = h->hR = nullptr;
  h->hOut = nullptr;
  h->staging_ready = false;
}

static void free_all(fbs_ctx* h) {
  free_host_path(h);
  void* ptrs[] = {h->P[0], h->P[1], h->SR[0], h->SR[1], h->G[0], h->G[1], h->bits[0], h->bits[1],
                  h->dmap[0], h->dmap[1], h->agg3, h->keys, h->tile_stats, h->trace,
                  h->volL, h->volR, h->gpadL, h->gpadR, h->aggL, h->vbitsL, h->vbitsR, h->rtiles};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}

static size_t frame_bytes(const fbs_ctx* h) {
  const size_t npix = (size_t)h->W * h->H;
  return 2 * ((size_t)h->H * h->Wp * 12 + (size_t)h->GR * h->Wg * 4 + (size_t)h->H * h->Wb * 4 + npix * 4) +
         npix * 16 + (h->nblk > 1 ? 2 * npix * 8 : 0);
}

static fbs_ctx* create_volume(fbs_ctx* h);
static fbs_ctx* create_impl(int W, int H, int d_min, int d_max, int radius, float sigma_s, float sigma_r, int path,
                            int rb0, int rb1);

extern "C" fbs_ctx* fbs_create(int W, int H, int d_min, int d_max, int radius, float sigma_s, float sigma_r) {
  return fbs_create_ex(W, H, d_min, d_max, radius, sigma_s, sigma_r, FBS_PATH_VOLUME);
}

extern "C" fbs_ctx* fbs_create_ex(int W, int H, int d_min, int d_max, int radius, float sigma_s, float sigma_r,
                                  int path) {
  return create_impl(W, H, d_min, d_max, radius, sigma_s, sigma_r, path, 0, H);
}

extern "C" fbs_ctx* fbs_create_band(int W, int H, int d_min, int d_max, int radius, float sigma_s, float sigma_r,
                                    int path, int row_begin, int row_end) {
  if (row_begin < 0 || row_end > H || row_begin >= row_end) {
    g_err = "fbs_create_band: need 0 <= row_begin < row_end <= H";
    return nullptr;
  }
  return create_impl(W, H, d_min, d_max, radius, sigma_s, sigma_r, path, row_begin, row_end);
}

static fbs_ctx* create_impl(int W, int H, int d_min, int d_max, int radius, float sigma_s, float sigma_r, int path,
                            int rb0, int rb1) {
  g_err.clear();
  if (path != FBS_PATH_VOLUME && path != FBS_PATH_FUSED) {
    fail(FBS_E_PARAM, "fbs_create: path must be FBS_PATH_VOLUME or FBS_PATH_FUSED");
    return nullptr;
  }
  if (W < 3 || H < 3) {
    fail(FBS_E_DIM, "fbs_create: W and H must be >= 3 (one 3x3 NCC block)");
    return nullptr;
  }
  if (d_min < 0 || d_max <= d_min || radius < 0 || !std::isfinite(sigma_s) || !(sigma_s > 0) ||
      !std::isfinite(sigma_r) || !(sigma_r > 0)) {
    fail(FBS_E_PARAM, "fbs_create: need 0 <= d_min < d_max, radius >= 0, finite sigma_s, sigma_r > 0");
    return nullptr;
  }
  {  // R#13: every tap weight ω_d ω_r >= 2^-124 > FLT_MIN, so no defined tap flushes to 0 in fp32
    // (ρ = 0: the only tap is the centre, weight 1)
    const double e = radius == 0 ? 0.0
                                 : 1.4426950408889634 * (2.0 * radius * radius / ((double)sigma_s * sigma_s) +
                                                         65025.0 / ((double)sigma_r * sigma_r));
    if (!(e <= kMaxWeightExp2)) {
      fail(FBS_E_UNSUPPORTED, "fbs_create: the smallest tap weight exp(-2rho^2/sigma_s^2 - 255^2/sigma_r^2) is below "
                              "2^-124 (fp32 underflow); increase sigma_r or sigma_s");
      return nullptr;
    }
  }
  if (radius > kMaxRadius || (path == FBS_PATH_FUSED && radius > kFusedMaxRadius)) {
    fail(FBS_E_UNSUPPORTED, "fbs_create: radius > FBS_MAX_RADIUS (10; 6 on the fused path)");
    return nullptr;
  }
  if ((long long)d_max - d_min + 1 > 4096 || W > (1 << 20) || H > (1 << 20)) {
    fail(FBS_E_UNSUPPORTED, "fbs_create: more than 4096 disparities or a side above 2^20 pixels");
    return nullptr;
  }
  if (!encode_fn()) {
    fail(FBS_E_CUDA, "fbs_create: cuTensorMapEncodeTiled is not available from the driver");
    return nullptr;
  }
  fbs_ctx* h = new (std::nothrow) fbs_ctx();
  if (!h) {
    fail(FBS_E_OOM, "fbs_create: host allocation failed");
    return nullptr;
  }
  std::memset((void*)h, 0, sizeof(*h));
  h->path = path;
  h->rb0 = rb0; h->rb1 = rb1;
  h->W = W; h->H = H; h->d_min = d_min; h->d_max = d_max; h->D = d_max - d_min + 1;
  h->nblk = (h->D + kDB - 1) / kDB;
  h->R = radius;
  h->sigma_s = sigma_s; h->sigma_r = sigma_r;
  cudaGetDevice(&h->device);
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  size_t smem = 0;
  int threads = 0;
  geometry(radius, h->TX, h->TY, smem, threads);
  h->Wp = (W + 3) / 4 * 4;
  h->Wg = guide_pitch(W, radius);
  h->GR = guide_rows(H, radius);
  h->gfs = (size_t)h->GR * h->Wg;
  h->Wb = (W + 31) / 32 + 1;
  {  // frames per launch: up to 16, within ~256 MB of per-frame scratch
    const size_t fb = frame_bytes(h);
    size_t fc = (256u << 20) / (fb ? fb : 1);
    h->fcap = (int)(fc < 1 ? 1 : (fc > 16 ? 16 : fc));
  }
  // Eq.(7): ω_d(dx,dy) = exp(-(dx²+dy²)/γ_d²); Eq.(8): ω_r(Δ) = exp(-Δ²/γ_r²)  (R#10).
  // k_fbs evaluates the product as one power of two: ω_d ω_r = 2^(cd(dx,dy) + nkr Δ²),
  // cd = -log2(e)(dx²+dy²)/γ_d², nkr = -log2(e)/γ_r² (built in double, rounded once;
  // P:L199 "pre-calculated").
  const int K1 = 2 * radius + 1;
  const double gd = sigma_s, gr = sigma_r, l2e = 1.4426950408889634;
  for (int dy = -radius; dy <= radius; ++dy)
    for (int dx = -radius; dx <= radius; ++dx)
      h->wa.cd[(dy + radius) * K1 + (dx + radius)] = (float)(-l2e * (double)(dx * dx + dy * dy) / (gd * gd));
  // Taps of undefined blocks carry the guide offset kGuideFlag = 2^23 and must get
  // weight +0 (2^(nkr (2^23 - 255)^2) < 2^-126, flushed by ex2.approx.ftz): this needs
  // nkr <= -2e-12, i.e. gamma_r <= 8.5e5.  Larger gamma_r use nkr = -2e-12: every
  // range weight is then within 9e-8 (relative) of Eq.(8)'s, below the error of
  // ex2.approx itself (R#13).
  h->wa.nkr = (float)std::min(-l2e / (gr * gr), -2e-12);
  if (path == FBS_PATH_VOLUME) return create_volume(h);

  const size_t F = h->fcap, npix = (size_t)W * H;
  const size_t np = F * H * h->Wp;
  bool ok = true;
  for (int im = 0; im < 2; ++im) {
    ok &= cudaMalloc(&h->P[im], np * 4) == cudaSuccess;
    ok &= cudaMalloc(&h->SR[im], np * 8) == cudaSuccess;
    ok &= cudaMalloc(&h->G[im], F * h->gfs * 4) == cudaSuccess;
    ok &= cudaMalloc(&h->bits[im], F * H * h->Wb * 4) == cudaSuccess;
    ok &= cudaMalloc(&h->dmap[im], F * npix * 4) == cudaSuccess;
  }
  ok &= cudaMalloc(&h->agg3, F * npix * sizeof(float4)) == cudaSuccess;
  if (h->nblk > 1) ok &= cudaMalloc(&h->keys, 2 * F * npix * 8) == cudaSuccess;
  ok &= cudaMalloc(&h->tile_stats, 4 * sizeof(unsigned long long)) == cudaSuccess;
#ifdef FBS_TRACE
  ok &= cudaMalloc(&h->trace, 8192 * sizeof(unsigned long long)) == cudaSuccess;
#endif
  if (!ok) {
    cudaGetLastError();
    free_all(h);
    delete h;
    fail(FBS_E_OOM, "fbs_create: device allocation failed");
    return nullptr;
  }
  for (int im = 0; im < 2; ++im) {
    k_fill<<<256, 256>>>(h->G[im], F * h->gfs, kGuideUndef);  // margins: taps outside the frame
    cudaMemset(h->dmap[im], 0xff, F * npix * 4);
    cudaMemset(h->bits[im], 0, F * H * h->Wb * 4);
  }
  cudaMemset(h->tile_stats, 0, 4 * sizeof(unsigned long long));
  if (cuda_check(cudaDeviceSynchronize(), "fbs_create init") != FBS_OK) {
    free_all(h);
    delete h;
    return nullptr;
  }
  if (!build_maps(h)) {
    free_all(h);
    delete h;
    fail(FBS_E_CUDA, "fbs_create: cuTensorMapEncodeTiled rejected a descriptor");
    return nullptr;
  }
  // fixed per instantiation, so setting it per handle never lowers another handle's cap
  switch (radius) {
#define FBS_SMEM_WS(RR)                                                                                    \
  case RR:                                                                                                 \
    cudaFuncSetAttribute(k_fbs_ws<RR, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    cudaFuncSetAttribute(k_fbs_ws<RR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
    break;
#define FBS_SMEM_ATTR(RR)                                                                                  \
  case RR:                                                                                                 \
    cudaFuncSetAttribute(k_fbs<RR, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    cudaFuncSetAttribute(k_fbs<RR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
    break;
    FBS_WS_RADII(FBS_SMEM_WS) FBS_SYNC_RADII(FBS_SMEM_ATTR)
#undef FBS_SMEM_ATTR
#undef FBS_SMEM_WS
  }
  if (cuda_check(cudaGetLastError(), "fbs_create smem attributes") != FBS_OK) {
    free_all(h);
    delete h;
    return nullptr;
  }
  // constant part of the walker's arguments
  WalkArgs& a = h->wa;
  a.W = W; a.H = H; a.D = h->D; a.d_min = d_min; a.d_max = d_max; a.nblk = h->nblk;
  a.Wb = h->Wb;
  a.bits[0] = h->bits[0]; a.bits[1] = h->bits[1];
  a.dmap[0] = h->dmap[0]; a.dmap[1] = h->dmap[1];
  a.agg3 = h->agg3;
  a.keys = h->keys;
  a.nstrips = (W + h->TX - 1) / h->TX;
  return h;
}

// Production k_agg instantiation has the EMPTY denominator form (units whose costs are
// all undefined skip the stream): KITTI 1,295 -> 1,586 frames/s, Teddy -0.6 %,
// MB2014 -1.9 % (interleaved A/B).
static constexpr bool kVolEmpty = true;

// Volume path scratch (one frame): FBS_PATH_VOLUME.
static fbs_ctx* create_volume(fbs_ctx* h) {
  const int W = h->W, H = h->H, R = h->R;
  h->fcap = 1;
  h->TX = vol::kTX;
  h->TY = vol::agg_tile_h(R);
  h->Wv = (W + vol::kTX - 1) / vol::kTX * vol::kTX + 2 * R;
  {  // rows of the served band [rb0, rb1): cost rows [vbase, ..), tile rows [abase, ..)
    const int TY = h->TY, ty0 = h->rb0 / TY, ty1 = (h->rb1 + TY - 1) / TY;
    h->vbase = std::max(0, ty0 * TY - R);
    h->abase = ty0 * TY;
    h->Hv = ty1 * TY + 2 * R - h->vbase + vol::kTYMax;
    h->arows = std::min(H, ty1 * TY) - h->abase;
  }
  h->vWb = (W + vol::kCX - 1) / vol::kCX * (vol::kCX / 32);
  h->vWg = vol::guide_pitch(W, R);
  const size_t npix = (size_t)W * H;
  const size_t nvol = (size_t)h->Hv * h->Wv * h->nblk * kDB;
  const size_t ngp = (size_t)vol::guide_rows(H, R) * h->vWg;
  bool ok = true;
  ok &= cudaMalloc(&h->gpadL, ngp * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->gpadR, ngp * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->vbitsL, (size_t)H * h->vWb * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->vbitsR, (size_t)H * h->vWb * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->volL, nvol * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->volR, nvol * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->dmap[0], npix * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->dmap[1], npix * 4) == cudaSuccess;
  if (h->nblk > 1) ok &= cudaMalloc(&h->aggL, (size_t)h->arows * W * h->nblk * kDB * sizeof(float)) == cudaSuccess;
  ok &= cudaMalloc(&h->agg3, npix * sizeof(float4)) == cudaSuccess;
  ok &= cudaMalloc(&h->tile_stats, 4 * sizeof(unsigned long long)) == cudaSuccess;
  {
    const int T = vol::kRangeTile;
    ok &= cudaMalloc(&h->rtiles, 4 * (size_t)((W + T - 1) / T) * ((H + T - 1) / T) * sizeof(int)) == cudaSuccess;
  }
#ifdef FBS_TRACE
  ok &= cudaMalloc(&h->trace, 8192 * sizeof(unsigned long long)) == cudaSuccess;
#endif
  if (!ok) {
    cudaGetLastError();
    free_all(h);
    delete h;
    fail(FBS_E_OOM, "fbs_create: device allocation failed");
    return nullptr;
  }
  // margins (and never-written rows) of the volumes hold the undefined cost
  vol::k_fill<<<1184, 256>>>(h->volL, nvol, kUndef);
  vol::k_fill<<<1184, 256>>>(h->volR, nvol, kUndef);
  vol::k_fill<<<256, 256>>>(h->gpadL, ngp, kGuideUndef);  // margins: taps outside the frame
  vol::k_fill<<<256, 256>>>(h->gpadR, ngp, kGuideUndef);
  cudaMemset(h->tile_stats, 0, 4 * sizeof(unsigned long long));
  cudaMemset(h->dmap[0], 0xff, npix * 4);
  cudaMemset(h->dmap[1], 0xff, npix * 4);
  cudaMemset(h->vbitsL, 0, (size_t)H * h->vWb * 4);
  cudaMemset(h->vbitsR, 0, (size_t)H * h->vWb * 4);
  if (cuda_check(cudaDeviceSynchronize(), "fbs_create init") != FBS_OK) {
    free_all(h);
    delete h;
    return nullptr;
  }
  // fixed per instantiation (k_cost: the largest supported block count), so a later
  // handle never lowers another handle's cap
#define FBS_SMEM_ATTR(RR)                                                                                     \
  cudaFuncSetAttribute(vol::k_agg<RR, kVolEmpty, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                       sizeof(vol::AggSmem<RR>));                                                             \
  cudaFuncSetAttribute(vol::k_agg<RR, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                       sizeof(vol::AggSmem<RR>));                                                             \
  cudaFuncSetAttribute(vol::k_agg<RR, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                       sizeof(vol::AggSmem<RR>));                                                             \
  cudaFuncSetAttribute(vol::k_agg<RR, false, false, false, true>,                                             \
                       cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(vol::AggSmem<RR>));
  FBS_VOL_RADII(FBS_SMEM_ATTR)
#undef FBS_SMEM_ATTR
#define FBS_SMEM_ATTR_SD(RR)                                                                                  \
  cudaFuncSetAttribute(vol::k_aggsd<RR, kVolEmpty, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                       sizeof(vol::AggSdSmem<RR>));                                                           \
  cudaFuncSetAttribute(vol::k_aggsd<RR, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,            \
                       sizeof(vol::AggSdSmem<RR>));
  FBS_SD_RADII(FBS_SMEM_ATTR_SD)
#undef FBS_SMEM_ATTR_SD
  cudaFuncSetAttribute(vol::k_cost<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)vol::cost_smem_bytes(4096 / kDB));
  cudaFuncSetAttribute(vol::k_cost<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)vol::cost_smem_bytes(1, 4));
  if (cuda_check(cudaGetLastError(), "fbs_create smem attributes") != FBS_OK) {
    free_all(h);
    delete h;
    return nullptr;
  }
  return h;
}

static void prof_free(fbs_ctx* h) {
  if (h->prof_ev) {
    for (int i = 0; i < kEv * h->prof_cap; ++i) cudaEventDestroy(h->prof_ev[i]);
    delete[] h->prof_ev;
  }
  h->prof_ev = nullptr;
  h->prof_cap = h->prof_n = 0;
}

extern "C" void fbs_destroy(fbs_ctx* h) {
  if (!h) return;
  prof_free(h);
  free_all(h);
  delete h;
}

// ---------------------------------------------------------------------------
// Launch with programmatic stream serialization (PDL): the kernel may begin
// while its predecessor drains; it synchronises on it with pdl_wait().
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

static cudaError_t launch_walk(const fbs_ctx* h, const WalkArgs& a, bool exp, cudaStream_t s) {
  const long long g = a.total < h->num_sms ? a.total : h->num_sms;
  int tx, ty, threads;
  size_t smem;
  geometry(h->R, tx, ty, smem, threads);
  const dim3 grid((unsigned)g), block((unsigned)threads);
  switch (h->R) {
#define FBS_CASE_WS(RR)                                                                                   \
  case RR:                                                                                                \
    return exp ? launch_pdl(k_fbs_ws<RR, true>, grid, block, smem, s, a)                                  \
               : launch_pdl(k_fbs_ws<RR, false>, grid, block, smem, s, a);
#define FBS_CASE(RR)                                                                                      \
  case RR:                                                                                                \
    return exp ? launch_pdl(k_fbs<RR, true>, grid, block, smem, s, a)                                     \
               : launch_pdl(k_fbs<RR, false>, grid, block, smem, s, a);
    FBS_WS_RADII(FBS_CASE_WS) FBS_SYNC_RADII(FBS_CASE)
#undef FBS_CASE
#undef FBS_CASE_WS
  }
  return cudaErrorInvalidValue;
}

// Disparity-range split request (fbs_compute_keys): competing range [c_lo, c_hi]
// (handle-local indices) and the outputs replacing the final map.
struct KeysReq {
  int c_lo, c_hi;
  unsigned long long *keys_l, *keys_r;
  float4* rec_l;
};

// Volume path, one frame: output rows [r0, r1); exports when expC/expA are set.
static int run_volume(fbs_ctx* h, const uint8_t* L, const uint8_t* Rimg, int r0, int r1, float* out,
                      float* const* expC, float* const* expA, cudaStream_t s, const KeysReq* kq = nullptr,
                      const short2* const* ranges = nullptr) {
  const int W = h->W, H = h->H, R = h->R;
  // aggregation tiles are anchored at multiples of the tile height in frame rows, so a
  // pixel's denominator form never depends on the band; cost rows cover the
  // tiles' windows (the classification reads validity masks over them too)
  const int TY = vol::agg_tile_h(R);
  const int ty0 = r0 / TY, ty1 = (r1 + TY - 1) / TY;
  const int c0 = std::max(0, ty0 * TY - R), c1 = std::min(H, ty1 * TY + R);  // cost rows
  float* aggL_exp = expA ? expA[0] : nullptr;
  float* aggR_exp = expA ? expA[1] : nullptr;
  h->launches = 0;
  cudaEvent_t* ev = nullptr;
  if (h->prof_ev && h->prof_n < h->prof_cap) ev = h->prof_ev + kEv * h->prof_n++;
  if (ev) cudaEventRecord(ev[0], s);
  {
    vol::CostArgs ca;
    ca.W = W; ca.H = H; ca.D = h->D; ca.d_min = h->d_min; ca.nblk = h->nblk; ca.Wv = h->Wv; ca.R = R;
    ca.r0 = c0; ca.r1 = c1; ca.vbase = h->vbase;
    ca.L = L; ca.Rimg = Rimg; ca.volL = h->volL; ca.volR = h->volR;
    ca.bitsL = h->vbitsL; ca.bitsR = h->vbitsR; ca.Wb = h->vWb;
    ca.gpadL = h->gpadL; ca.gpadR = h->gpadR; ca.Wg = h->vWg;
    if (vol::cost_runs4(h->D)) {  // D <= 16: no padding slots computed
      const int cx = vol::kCX * 4;
      vol::k_cost<4><<<dim3((W + cx - 1) / cx, c1 - c0, 2), 256, vol::cost_smem_bytes(h->nblk, 4), s>>>(ca);
    } else {
      const dim3 grd((W + vol::kCX - 1) / vol::kCX, c1 - c0, 2);
      vol::k_cost<1><<<grd, 256, vol::cost_smem_bytes(h->nblk), s>>>(ca);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_check(e, "k_cost launch");  // nothing downstream runs on stale volumes
    h->launches += 1;
  }
  if (ev) cudaEventRecord(ev[1], s);
  vol::AggArgs a;
  a.W = W; a.H = H; a.D = h->D; a.d_min = h->d_min; a.d_max = h->d_max;
  a.nblk = h->nblk; a.Wv = h->Wv;
  std::memcpy(a.cd, h->wa.cd, sizeof(a.cd));
  a.nkr = h->wa.nkr;
  a.gpadL = h->gpadL; a.gpadR = h->gpadR; a.Wg = h->vWg;
  a.r0 = r0; a.r1 = r1; a.ty0 = ty0;
  a.vbase = h->vbase; a.abase = h->abase;
  a.volL = h->volL; a.volR = h->volR;
  a.bitsL = h->vbitsL; a.bitsR = h->vbitsR; a.Wb = h->vWb;
  a.dL = h->dmap[0]; a.dR = h->dmap[1]; a.aggL = h->aggL; a.exportR = aggR_exp;
  // one d-block: the left costs stay on chip and only Eq.(10)'s three are stored
  // (unless the debug export wants the whole left volume)
  float* aggL_tmp = nullptr;
  if (aggL_exp && !h->aggL) {  // single-block frame exporting its left volume: temporary store
    if (cudaMalloc(&aggL_tmp, (size_t)W * H * kDB * sizeof(float)) != cudaSuccess)
      return fail(FBS_E_OOM, "fbs_debug_volumes: scratch");
    a.aggL = aggL_tmp;
    a.abase = 0;
  }
  a.agg3 = (h->nblk == 1 && !aggL_exp) ? h->agg3 : nullptr;
  a.tile_stats = ev ? h->tile_stats : nullptr;
  a.c_lo = kq ? kq->c_lo : 0;
  a.c_hi = kq ? kq->c_hi : h->D - 1;
  a.keys_out[0] = kq ? kq->keys_l : nullptr;
  a.keys_out[1] = kq ? kq->keys_r : nullptr;
  a.ranges[0] = ranges ? ranges[0] : nullptr;
  a.ranges[1] = ranges ? ranges[1] : nullptr;
  {
    const dim3 grid((W + vol::kTX - 1) / vol::kTX, ty1 - ty0, 2);
    cudaError_t e = cudaErrorInvalidValue;
    // D <= 16 (Tsukuba-shaped): k_aggsd, 8-lane groups of 16 disparities, no padding;
    // the disparity-range split and the sparse search range keep k_agg's KEYS / RANGED
    const bool use_sd = vol::aggsd_ok(R, h->D) && !kq && !ranges;
    if (use_sd) switch (R) {
#define FBS_CASE_SD(RR)                                                                                       \
  case RR:                                                                                                    \
    e = aggR_exp ? launch_pdl(vol::k_aggsd<RR, false, true>, grid, dim3(vol::sd::kThreads),                   \
                              sizeof(vol::AggSdSmem<RR>), s, a)                                               \
                 : launch_pdl(vol::k_aggsd<RR, kVolEmpty, false>, grid, dim3(vol::sd::kThreads),              \
                              sizeof(vol::AggSdSmem<RR>), s, a);                                              \
    break;
      FBS_SD_RADII(FBS_CASE_SD)
#undef FBS_CASE_SD
    }
    else switch (R) {
#define FBS_CASE(RR)                                                                                          \
  case RR:                                                                                                    \
    e = aggR_exp ? launch_pdl(vol::k_agg<RR, false, true>, grid, dim3(vol::AggGeom<RR>::THREADS),             \
                              sizeof(vol::AggSmem<RR>), s, a)                                                 \
        : kq     ? launch_pdl(vol::k_agg<RR, false, false, true>, grid, dim3(vol::AggGeom<RR>::THREADS),      \
                              sizeof(vol::AggSmem<RR>), s, a)                                                 \
        : ranges ? launch_pdl(vol::k_agg<RR, false, false, false, true>, grid,                                \
                              dim3(vol::AggGeom<RR>::THREADS), sizeof(vol::AggSmem<RR>), s, a)                \
                 : launch_pdl(vol::k_agg<RR, kVolEmpty, false>, grid, dim3(vol::AggGeom<RR>::THREADS),        \
                              sizeof(vol::AggSmem<RR>), s, a);                                                \
    break;
      FBS_VOL_RADII(FBS_CASE)
#undef FBS_CASE
    }
    if (e != cudaSuccess) return cuda_check(e, "k_agg launch");
    h->launches += 1;
  }
  if (ev) cudaEventRecord(ev[2], s);
  if (kq) {  // disparity-range split: the records instead of the final map
    const dim3 grd((W + 127) / 128, r1 - r0);
    vol::k_records<<<grd, 128, 0, s>>>(h->dmap[0], a.aggL, a.agg3, h->nblk, W, r0, r1, h->d_min, h->d_max, a.abase,
                                       kq->rec_l);
    h->launches += 1;
    if (ev) cudaEventRecord(ev[3], s);
    return cuda_check(cudaGetLastError(), "fbs_compute_keys launch");
  }
  {
    const dim3 grd((W + 127) / 128, r1 - r0);
    const cudaError_t e = launch_pdl(h->scat.n ? vol::k_finalize<true> : vol::k_finalize<false>, grd, dim3(128), 0,
                                     s, (const int32_t*)h->dmap[0],
                                     (const int32_t*)h->dmap[1], (const float*)a.aggL, (const float4*)a.agg3,
                                     h->nblk, W, r0, r1, h->d_min, h->d_max, a.abase, out,
                                     (const short2*)(ranges ? ranges[0] : nullptr), h->scat);
    if (e != cudaSuccess) return cuda_check(e, "k_finalize launch");
    h->launches += 1;
  }
  if (ev) cudaEventRecord(ev[3], s);
  if (aggL_exp) vol::k_export_agg<<<1184, 256, 0, s>>>(a.aggL, W, H, h->D, h->nblk, aggL_exp);
  if (expC && expC[0]) vol::k_export_vol<<<1184, 256, 0, s>>>(h->volL, W, H, h->D, h->nblk, h->Wv, R, expC[0]);
  if (expC && expC[1]) vol::k_export_vol<<<1184, 256, 0, s>>>(h->volR, W, H, h->D, h->nblk, h->Wv, R, expC[1]);
  if (aggL_tmp) {
    cudaStreamSynchronize(s);
    cudaFree(aggL_tmp);
  }
  return cuda_check(cudaGetLastError(), "fbs launch");
}

// nf frames (left/right: nf x [H][W] device), output rows [r0, r1) of each into
// out (nf x [r1-r0][W]); exports (one frame) when expC/expA are set.
static int run(fbs_ctx* h, const uint8_t* L, const uint8_t* Rimg, int nf, int r0, int r1, float* out,
               float* const* expC, float* const* expA, cudaStream_t s) {
  if (h->path == FBS_PATH_VOLUME) {
    const size_t npix = (size_t)h->W * h->H, nout = (size_t)(r1 - r0) * h->W;
    int launches = 0;
    for (int i = 0; i < nf; ++i) {
      const int rc = run_volume(h, L + i * npix, Rimg + i * npix, r0, r1, out + i * nout, expC, expA, s);
      if (rc != FBS_OK) return rc;
      launches += h->launches;
    }
    h->launches = launches;
    return FBS_OK;
  }
  const int W = h->W, H = h->H, R = h->R, TY = h->TY;
  // walker steps are anchored at multiples of TY in frame rows, so a pixel's
  // denominator form never depends on the band; cost rows cover their windows
  const int ty0 = r0 / TY, ty1 = (r1 + TY - 1) / TY;
  const int c0 = std::max(0, ty0 * TY - R), c1 = std::min(H, ty1 * TY + R);
  h->launches = 0;
  cudaEvent_t* ev = nullptr;
  if (h->prof_ev && h->prof_n < h->prof_cap) ev = h->prof_ev + kEv * h->prof_n++;
  if (ev) cudaEventRecord(ev[0], s);
  cudaError_t e;
  {
    PrepArgs p;
    p.W = W; p.H = H; p.Wp = h->Wp; p.Wg = h->Wg; p.Wb = h->Wb; p.R = R; p.y0 = c0; p.y1 = c1;
    p.img[0] = L; p.img[1] = Rimg;
    for (int im = 0; im < 2; ++im) { p.P[im] = h->P[im]; p.SR[im] = h->SR[im]; p.G[im] = h->G[im]; p.bits[im] = h->bits[im]; }
    p.gfs = h->gfs;
    e = launch_pdl(k_prep, dim3((W + 127) / 128, c1 - c0, 2 * nf), dim3(128), 0, s, p);
    if (e != cudaSuccess) return cuda_check(e, "k_prep launch");
    h->launches += 1;
  }
  if (ev) cudaEventRecord(ev[1], s);
  {
    WalkArgs& a = h->wa;
    a.r0 = r0; a.r1 = r1;
    a.ty0 = ty0; a.nty = ty1 - ty0; a.nframes = nf;
    a.total = (long long)nf * 2 * a.nstrips * a.nty;
    a.expC[0] = expC ? expC[0] : nullptr; a.expC[1] = expC ? expC[1] : nullptr;
    a.expA[0] = expA ? expA[0] : nullptr; a.expA[1] = expA ? expA[1] : nullptr;
    a.tile_stats = ev ? h->tile_stats : nullptr;
    a.trace = h->trace;
    e = launch_walk(h, a, expC || expA, s);
    if (e != cudaSuccess) return cuda_check(e, "k_fbs launch");
    h->launches += 1;
  }
  if (ev) cudaEventRecord(ev[2], s);
  e = launch_pdl(h->scat.n ? k_final<true> : k_final<false>, dim3((W + 127) / 128, r1 - r0, nf), dim3(128), 0, s,
                 (const int32_t*)h->dmap[0],
                 (const int32_t*)h->dmap[1], (const float4*)h->agg3, W, H, r0, r1, h->d_min, h->d_max, out,
                 h->scat);
  if (e != cudaSuccess) return cuda_check(e, "k_final launch");
  h->launches += 1;
  if (ev) cudaEventRecord(ev[3], s);
  return cuda_check(cudaGetLastError(), "fbs launch");
}

static bool full_frame(const fbs_ctx* h) { return h->rb0 == 0 && h->rb1 == h->H; }

extern "C" int fbs_compute(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* disp_out,
                           fbs_stream_t stream) {
  if (!h || !left || !right || !disp_out) return fail(FBS_E_ARG, "fbs_compute: NULL argument");
  if (!full_frame(h)) return fail(FBS_E_ARG, "fbs_compute: band handle (use fbs_compute_rows)");
  return run(h, left, right, 1, 0, h->H, disp_out, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int fbs_compute_rows(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int row_begin,
                                int row_end, float* disp_band, fbs_stream_t stream) {
  if (!h || !left || !right || !disp_band) return fail(FBS_E_ARG, "fbs_compute_rows: NULL argument");
  if (row_begin < h->rb0 || row_end > h->rb1 || row_begin >= row_end)
    return fail(FBS_E_ARG, "fbs_compute_rows: need rb0 <= row_begin < row_end <= rb1 (the handle's rows; [0, H) "
                           "unless created by fbs_create_band)");
  return run(h, left, right, 1, row_begin, row_end, disp_band, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int fbs_compute_rows_scatter(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int row_begin,
                                        int row_end, float* const* outs, int nouts, fbs_stream_t stream) {
  if (!h || !left || !right || !outs) return fail(FBS_E_ARG, "fbs_compute_rows_scatter: NULL argument");
  if (nouts < 1 || nouts > kMaxScatter) return fail(FBS_E_ARG, "fbs_compute_rows_scatter: need 1 <= nouts <= 8");
  if (row_begin < h->rb0 || row_end > h->rb1 || row_begin >= row_end)
    return fail(FBS_E_ARG, "fbs_compute_rows_scatter: rows outside the handle's band");
  OutSet os{};
  for (int k = 0; k < nouts; ++k) {
    if (!outs[k]) return fail(FBS_E_ARG, "fbs_compute_rows_scatter: NULL destination");
    os.p[k] = outs[k];
  }
  os.n = nouts;
  h->scat = os;
  const int rc = run(h, left, right, 1, row_begin, row_end, outs[0], nullptr, nullptr, (cudaStream_t)stream);
  h->scat = OutSet{};
  return rc;
}

extern "C" int fbs_compute_batch(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int n,
                                 float* disp_out, fbs_stream_t stream) {
  if (!h || !left || !right || !disp_out) return fail(FBS_E_ARG, "fbs_compute_batch: NULL argument");
  if (!full_frame(h)) return fail(FBS_E_ARG, "fbs_compute_batch: band handle");
  if (n < 1) return fail(FBS_E_ARG, "fbs_compute_batch: n must be >= 1");
  const size_t npix = (size_t)h->W * h->H;
  int launches = 0;
  for (int i = 0; i < n; i += h->fcap) {
    const int m = std::min(h->fcap, n - i);
    int rc = run(h, left + i * npix, right + i * npix, m, 0, h->H, disp_out + i * npix, nullptr, nullptr,
                 (cudaStream_t)stream);
    if (rc != FBS_OK) return rc;
    launches += h->launches;
  }
  h->launches = launches;
  return FBS_OK;
}

// Host path: frame i's copies in (stream cs_in), compute (caller's stream) and
// copy out (cs_out) are ordered by events; two staging slots let frame i+1's
// upload and frame i-1's download run on the copy engines while frame i computes.
static int host_setup(fbs_ctx* h) {
  if (h->staging_ready) return FBS_OK;
  const size_t npix = (size_t)h->W * h->H;
  bool ok = cudaMalloc(&h->hL, 2 * npix) == cudaSuccess && cudaMalloc(&h->hR, 2 * npix) == cudaSuccess &&
            cudaMalloc(&h->hOut, 2 * npix * 4) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&h->cs_in, cudaStreamNonBlocking) == cudaSuccess &&
       cudaStreamCreateWithFlags(&h->cs_out, cudaStreamNonBlocking) == cudaSuccess &&
       cudaEventCreateWithFlags(&h->ev_entry, cudaEventDisableTiming) == cudaSuccess;
  for (int k = 0; ok && k < 2; ++k)
    ok = cudaEventCreateWithFlags(&h->ev_in[k], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&h->ev_done[k], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&h->ev_out[k], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    free_host_path(h);  // leaves no half-built state behind
    return fail(FBS_E_OOM, "fbs_compute_host_batch: staging allocation failed");
  }
  h->staging_ready = true;
  return FBS_OK;
}

extern "C" int fbs_compute_host_batch(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int n,
                                      float* disp_out, fbs_stream_t stream) {
  if (!h || !left || !right || !disp_out) return fail(FBS_E_ARG, "fbs_compute_host_batch: NULL argument");
  if (!full_frame(h)) return fail(FBS_E_ARG, "fbs_compute_host_batch: band handle");
  if (n < 1) return fail(FBS_E_ARG, "fbs_compute_host_batch: n must be >= 1");
  int rc = host_setup(h);
  if (rc) return rc;
  const size_t npix = (size_t)h->W * h->H;
  cudaStream_t s = (cudaStream_t)stream;
  // the copy streams start after everything already enqueued on the caller's stream
  cudaEventRecord(h->ev_entry, s);
  cudaStreamWaitEvent(h->cs_in, h->ev_entry, 0);
  cudaStreamWaitEvent(h->cs_out, h->ev_entry, 0);
  for (int i = 0; i < n; ++i) {
    const int k = i & 1;
    uint8_t *dl = h->hL + k * npix, *dr = h->hR + k * npix;
    float* dout = h->hOut + k * npix;
    if (i >= 2) cudaStreamWaitEvent(h->cs_in, h->ev_done[k], 0);  // slot k's inputs consumed (frame i-2)
    if ((rc = cuda_check(cudaMemcpyAsync(dl, left + i * npix, npix, cudaMemcpyHostToDevice, h->cs_in), "H2D left")))
      return rc;
    if ((rc = cuda_check(cudaMemcpyAsync(dr, right + i * npix, npix, cudaMemcpyHostToDevice, h->cs_in), "H2D right")))
      return rc;
    cudaEventRecord(h->ev_in[k], h->cs_in);
    cudaStreamWaitEvent(s, h->ev_in[k], 0);
    if (i >= 2) cudaStreamWaitEvent(s, h->ev_out[k], 0);  // slot k's map downloaded (frame i-2)
    if ((rc = fbs_compute(h, dl, dr, dout, stream))) return rc;
    cudaEventRecord(h->ev_done[k], s);
    cudaStreamWaitEvent(h->cs_out, h->ev_done[k], 0);
    if ((rc = cuda_check(cudaMemcpyAsync(disp_out + i * npix, dout, npix * 4, cudaMemcpyDeviceToHost, h->cs_out),
                         "D2H")))
      return rc;
    cudaEventRecord(h->ev_out[k], h->cs_out);
  }
  // the caller's stream resumes after the last download
  cudaStreamWaitEvent(s, h->ev_out[(n - 1) & 1], 0);
  if ((rc = cuda_check(cudaStreamSynchronize(h->cs_out), "fbs_compute_host_batch sync"))) return rc;
  return cuda_check(cudaStreamSynchronize(s), "fbs_compute_host_batch sync");
}

extern "C" int fbs_compute_host(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* disp_out,
                                fbs_stream_t stream) {
  if (!h || !left || !right || !disp_out) return fail(FBS_E_ARG, "fbs_compute_host: NULL argument");
  return fbs_compute_host_batch(h, left, right, 1, disp_out, stream);
}

extern "C" int fbs_debug_volumes(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* cost_l,
                                 float* cost_r, float* agg_l, float* agg_r, float* disp_out, int32_t* disp_l,
                                 int32_t* disp_r, fbs_stream_t stream) {
  if (!h || !left || !right) return fail(FBS_E_ARG, "fbs_debug_volumes: NULL argument");
  if (!full_frame(h)) return fail(FBS_E_ARG, "fbs_debug_volumes: band handle");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t npix = (size_t)h->W * h->H;
  float* tmp = nullptr;
  if (!disp_out && cudaMalloc(&tmp, npix * 4) != cudaSuccess) return fail(FBS_E_OOM, "fbs_debug_volumes: scratch");
  float* expC[2] = {cost_l, cost_r};
  float* expA[2] = {agg_l, agg_r};
  const bool any = cost_l || cost_r || agg_l || agg_r;
  int rc = run(h, left, right, 1, 0, h->H, disp_out ? disp_out : tmp, any ? expC : nullptr, any ? expA : nullptr, s);
  if (rc == FBS_OK && disp_l) rc = cuda_check(cudaMemcpyAsync(disp_l, h->dmap[0], npix * 4, cudaMemcpyDeviceToDevice, s), "copy d_L");
  if (rc == FBS_OK && disp_r) rc = cuda_check(cudaMemcpyAsync(disp_r, h->dmap[1], npix * 4, cudaMemcpyDeviceToDevice, s), "copy d_R");
  if (tmp) {
    cudaStreamSynchronize(s);
    cudaFree(tmp);
  }
  return rc;
}

extern "C" int fbs_debug_select(fbs_ctx* h, const float* agg_l, const float* agg_r, int32_t* disp_l,
                                int32_t* disp_r, float* disp_out, fbs_stream_t stream) {
  if (!h || !agg_l || !agg_r) return fail(FBS_E_ARG, "fbs_debug_select: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t npix = (size_t)h->W * h->H;
  const int nb = (int)((npix + 255) / 256);
  k_select_wta<<<nb, 256, 0, s>>>(agg_r, h->W, h->H, h->D, h->d_min, h->dmap[1], nullptr);
  k_select_wta<<<nb, 256, 0, s>>>(agg_l, h->W, h->H, h->D, h->d_min, h->dmap[0], h->agg3);
  if (disp_out)
    k_final<false><<<dim3((h->W + 127) / 128, h->H, 1), 128, 0, s>>>(h->dmap[0], h->dmap[1], h->agg3, h->W, h->H, 0, h->H,
                                                              h->d_min, h->d_max, disp_out, OutSet{});
  if (disp_l) cudaMemcpyAsync(disp_l, h->dmap[0], npix * 4, cudaMemcpyDeviceToDevice, s);
  if (disp_r) cudaMemcpyAsync(disp_r, h->dmap[1], npix * 4, cudaMemcpyDeviceToDevice, s);
  return cuda_check(cudaGetLastError(), "fbs_debug_select");
}

extern "C" int fbs_debug_maps(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* disp_out,
                              int32_t* disp_l, int32_t* disp_r, fbs_stream_t stream) {
  if (!h || !left || !right || !disp_out) return fail(FBS_E_ARG, "fbs_debug_maps: NULL argument");
  if (!full_frame(h)) return fail(FBS_E_ARG, "fbs_debug_maps: band handle");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t npix = (size_t)h->W * h->H;
  int rc = run(h, left, right, 1, 0, h->H, disp_out, nullptr, nullptr, s);
  if (rc != FBS_OK) return rc;
  if (disp_l) cudaMemcpyAsync(disp_l, h->dmap[0], npix * 4, cudaMemcpyDeviceToDevice, s);
  if (disp_r) cudaMemcpyAsync(disp_r, h->dmap[1], npix * 4, cudaMemcpyDeviceToDevice, s);
  return cuda_check(cudaGetLastError(), "fbs_debug_maps");
}

extern "C" int fbs_stats(const fbs_ctx* h, int* launches) {
  if (!h) return fail(FBS_E_ARG, "fbs_stats: NULL handle");
  if (launches) *launches = h->launches;
  return FBS_OK;
}

extern "C" int fbs_profile_enable(fbs_ctx* h, int n) {
  if (!h || n < 0 || n > 65536) return fail(FBS_E_ARG, "fbs_profile_enable: bad handle or n");
  prof_free(h);
  if (n == 0) return FBS_OK;
  h->prof_ev = new (std::nothrow) cudaEvent_t[kEv * n];
  if (!h->prof_ev) return fail(FBS_E_OOM, "fbs_profile_enable: host allocation");
  for (int i = 0; i < kEv * n; ++i)
    if (cudaEventCreate(&h->prof_ev[i]) != cudaSuccess) {
      for (int j = 0; j < i; ++j) cudaEventDestroy(h->prof_ev[j]);
      delete[] h->prof_ev;
      h->prof_ev = nullptr;
      return fail(FBS_E_CUDA, "fbs_profile_enable: cudaEventCreate");
    }
  h->prof_cap = n;
  h->prof_n = 0;
  return FBS_OK;
}

extern "C" int fbs_profile_read(fbs_ctx* h, double* stage_ms, int* ncalls) {
  if (!h || !stage_ms) return fail(FBS_E_ARG, "fbs_profile_read: NULL argument");
  for (int k = 0; k < FBS_NSTAGES; ++k) stage_ms[k] = 0.0;
  for (int i = 0; i < h->prof_n; ++i) {
    cudaEvent_t* ev = h->prof_ev + kEv * i;
    if (cudaEventSynchronize(ev[FBS_NSTAGES]) != cudaSuccess) return cuda_check(cudaGetLastError(), "fbs_profile_read");
    for (int k = 0; k < FBS_NSTAGES; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
      stage_ms[k] += ms;
    }
  }
  if (ncalls) *ncalls = h->prof_n;
  h->prof_n = 0;
  return FBS_OK;
}

extern "C" int fbs_tile_stats(fbs_ctx* h, long long* fast, long long* edge, long long* general,
                              long long* empty) {
  if (!h) return fail(FBS_E_ARG, "fbs_tile_stats: NULL handle");
  unsigned long long v[4] = {0, 0, 0, 0};
  int rc = cuda_check(cudaMemcpy(v, h->tile_stats, sizeof(v), cudaMemcpyDeviceToHost), "fbs_tile_stats");
  if (rc != FBS_OK) return rc;
  cudaMemset(h->tile_stats, 0, sizeof(v));
  if (fast) *fast = (long long)v[0];
  if (edge) *edge = (long long)v[1];
  if (general) *general = (long long)v[2];
  if (empty) *empty = (long long)v[3];
  return FBS_OK;
}

#ifdef FBS_TRACE
// Trace builds only (not in include/fbs.h): copy the last launch's timeline of CTA 0.
extern "C" int fbs_debug_trace(fbs_ctx* h, unsigned long long* host, int n) {
  if (!h || !h->trace || !host || n > 8192) return fail(FBS_E_ARG, "fbs_debug_trace");
  return cuda_check(cudaMemcpy(host, h->trace, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "trace");
}
#endif

// ---------------------------------------------------------------------------
// Disparity-range split (NEXT-3, SURVEY §8(e) "Alternative").
extern "C" int fbs_compute_keys(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int c_lo, int c_hi,
                                uint64_t* keys_l, uint64_t* keys_r, float* rec_l, fbs_stream_t stream) {
  if (!h || !left || !right || !keys_l || !keys_r || !rec_l) return fail(FBS_E_ARG, "fbs_compute_keys: NULL argument");
  if (h->path != FBS_PATH_VOLUME) return fail(FBS_E_UNSUPPORTED, "fbs_compute_keys: volume path only");
  if (!full_frame(h)) return fail(FBS_E_ARG, "fbs_compute_keys: band handle");
  if (c_lo < h->d_min || c_hi > h->d_max || c_lo > c_hi)
    return fail(FBS_E_ARG, "fbs_compute_keys: need d_min <= c_lo <= c_hi <= d_max (the handle's range)");
  KeysReq kq{c_lo - h->d_min, c_hi - h->d_min, (unsigned long long*)keys_l, (unsigned long long*)keys_r,
             (float4*)rec_l};
  return run_volume(h, left, right, 0, h->H, nullptr, nullptr, nullptr, (cudaStream_t)stream, &kq);
}

extern "C" int fbs_finalize_keys(int W, int H, int d_min, int d_max, const uint64_t* keys_l, const uint64_t* keys_r,
                                 const float* rec_l, float* disp_out, fbs_stream_t stream) {
  if (!keys_l || !keys_r || !rec_l || !disp_out) return fail(FBS_E_ARG, "fbs_finalize_keys: NULL argument");
  if (W < 3 || H < 3 || d_min < 0 || d_max <= d_min) return fail(FBS_E_PARAM, "fbs_finalize_keys: bad geometry");
  const dim3 grd((W + 127) / 128, H);
  vol::k_finalize_keys<<<grd, 128, 0, (cudaStream_t)stream>>>((const unsigned long long*)keys_l,
                                                              (const unsigned long long*)keys_r,
                                                              (const float4*)rec_l, W, H, d_min, d_max, disp_out);
  return cuda_check(cudaGetLastError(), "fbs_finalize_keys");
}

// ---------------------------------------------------------------------------
// Sparse search range (NEXT-4, the paper's future work P:L358; R#31-R#33).
extern "C" int fbs_suggest_ranges(fbs_ctx* h, const float* seed_disp, int margin, int16_t* ranges_l,
                                  int16_t* ranges_r, fbs_stream_t stream) {
  if (!h || !seed_disp || !ranges_l || !ranges_r) return fail(FBS_E_ARG, "fbs_suggest_ranges: NULL argument");
  if (margin < 0) return fail(FBS_E_PARAM, "fbs_suggest_ranges: margin must be >= 0");
  if (h->path != FBS_PATH_VOLUME) return fail(FBS_E_UNSUPPORTED, "fbs_suggest_ranges: volume path only");
  cudaStream_t s = (cudaStream_t)stream;
  const int W = h->W, H = h->H, T = vol::kRangeTile;
  const int tx = (W + T - 1) / T, ty = (H + T - 1) / T, n = 2 * tx * ty;
  int* tiles = h->rtiles;  // (min, max) per tile, left then right (allocated in fbs_create)
  vol::k_range_init<<<(2 * n + 255) / 256, 256, 0, s>>>(tiles, 2 * n);
  vol::k_range_seeds<<<dim3((W + 127) / 128, H), 128, 0, s>>>(seed_disp, W, H, tx, tiles, tiles + n);
  vol::k_range_expand<<<dim3((W + 127) / 128, H), 128, 0, s>>>(tiles, tiles + n, W, H, tx, h->d_min, h->d_max, margin,
                                                              (short2*)ranges_l, (short2*)ranges_r);
  return cuda_check(cudaGetLastError(), "fbs_suggest_ranges");
}

extern "C" int fbs_compute_ranged(fbs_ctx* h, const uint8_t* left, const uint8_t* right, const int16_t* ranges_l,
                                  const int16_t* ranges_r, float* disp_out, fbs_stream_t stream) {
  if (!h || !left || !right || !ranges_l || !ranges_r || !disp_out)
    return fail(FBS_E_ARG, "fbs_compute_ranged: NULL argument");
  if (h->path != FBS_PATH_VOLUME) return fail(FBS_E_UNSUPPORTED, "fbs_compute_ranged: volume path only");
  if (!full_frame(h)) return fail(FBS_E_ARG, "fbs_compute_ranged: band handle");
  const short2* rg[2] = {(const short2*)ranges_l, (const short2*)ranges_r};
  return run_volume(h, left, right, 0, h->H, disp_out, nullptr, nullptr, (cudaStream_t)stream, nullptr, rg);
}
