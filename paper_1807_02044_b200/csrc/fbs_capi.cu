// fbs_capi.cu — C ABI of libfbs.so (declared in include/fbs.h).
//
// Host side: parameter validation, ω_d / ω_r tables (Eq.(7)(8), built in
// double and rounded once to fp32, "pre-calculated"), scratch
// allocation, and the launch sequence per frame (3 launches):
//   k_cost      block statistics + twin cost volumes, both sides   Eq.(1)-(3)
//   k_agg       aggregation + WTA, both sides                      Eq.(6)-(8)
//   k_finalize  LRC + subpixel -> disp_out                         Eq.(9)(10)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <utility>

#include "../../include/fbs.h"
#include "fbs_kernels.cuh"

using namespace fbs;

struct fbs_ctx {
  int W, H, d_min, d_max, D, nblk, R, Wv, Hv;
  float sigma_s, sigma_r;
  int device;
  // Eq.(7)(8) in the exponent form k_agg evaluates: w' = 2^(cd(dx,dy) + nkr Δ²)
  float cd[(2 * kMaxRadius + 1) * (2 * kMaxRadius + 1)];
  float nkr;
  // scratch
  uint32_t *bitsL, *bitsR;
  float *gpadL, *gpadR;    // padded guide images for k_agg (k_cost), [guide_rows][Wg]
  int Wg;
  bool empty_form;         // k_agg<R, true>: GENERAL units test for EMPTY (FBS_EMPTY_FORM=1 at create)
  int Wb;
  float *volL, *volR;
  int32_t *dL, *dR;
  float* aggL;       // left aggregated costs [H][nblk][W][64] (k_agg -> k_finalize)
  float4* agg3;      // one d-block: (c(d*-1), c(d*), c(d*+1)) per left pixel [H][W] (k_agg -> k_finalize)
  uint8_t *hL, *hR;  // device staging for fbs_compute_host[_batch]: two frame slots each
  float* hOut;
  cudaStream_t cs_in, cs_out;          // copy streams of the host path (created on first use)
  cudaEvent_t ev_in[2], ev_done[2], ev_out[2];
  unsigned long long* tile_stats;  // device [4] FAST/EDGE/GENERAL/EMPTY, counting when prof_ev is set
  int launches;
  // live profiling (fbs_profile_enable): kEv events per frame
  cudaEvent_t* prof_ev;
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

static void free_host_path(fbs_ctx* h) {
  if (h->cs_in) {
    cudaStreamDestroy(h->cs_in);
    cudaStreamDestroy(h->cs_out);
    for (int k = 0; k < 2; ++k) {
      cudaEventDestroy(h->ev_in[k]);
      cudaEventDestroy(h->ev_done[k]);
      cudaEventDestroy(h->ev_out[k]);
    }
    h->cs_in = h->cs_out = nullptr;
  }
}

static void free_all(fbs_ctx* h) {
  free_host_path(h);
  void* ptrs[] = {h->gpadL, h->gpadR, h->bitsL, h->bitsR, h->volL, h->volR, h->dL, h->dR, h->aggL, h->agg3, h->hL, h->hR, h->hOut,
                  h->tile_stats};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}

extern "C" fbs_ctx* fbs_create(int W, int H, int d_min, int d_max, int radius, float sigma_s,
                               float sigma_r) {
  g_err.clear();
  if (W < 3 || H < 3) {
    fail(FBS_E_DIM, "fbs_create: W and H must be >= 3 (one 3x3 NCC block)");
    return nullptr;
  }
  if (d_min < 0 || d_max <= d_min || radius < 0 || !std::isfinite(sigma_s) || !(sigma_s > 0) ||
      !std::isfinite(sigma_r) || !(sigma_r > 0)) {
    fail(FBS_E_PARAM, "fbs_create: need 0 <= d_min < d_max, radius >= 0, finite sigma_s, sigma_r > 0");
    return nullptr;
  }
  if (sigma_r > FBS_MAX_SIGMA_R) {
    fail(FBS_E_UNSUPPORTED, "fbs_create: sigma_r > FBS_MAX_SIGMA_R");
    return nullptr;
  }
  if (radius > kMaxRadius) {
    fail(FBS_E_UNSUPPORTED, "fbs_create: radius > FBS_MAX_RADIUS");
    return nullptr;
  }
  if ((long long)(d_max - d_min + 1) > 4096) {
    fail(FBS_E_UNSUPPORTED, "fbs_create: more than 4096 disparities");
    return nullptr;
  }
  fbs_ctx* h = new (std::nothrow) fbs_ctx();
  if (!h) {
    fail(FBS_E_OOM, "fbs_create: host allocation failed");
    return nullptr;
  }
  std::memset(h, 0, sizeof(*h));
  h->W = W; h->H = H; h->d_min = d_min; h->d_max = d_max; h->D = d_max - d_min + 1;
  h->nblk = (h->D + kDB - 1) / kDB;
  h->R = radius;
  h->Wv = (W + kTX - 1) / kTX * kTX + 2 * radius;
  h->Hv = (H + kTYMax - 1) / kTYMax * kTYMax + kTYMax + 2 * radius;
  h->sigma_s = sigma_s; h->sigma_r = sigma_r;
  {  // tuning knob for scenes with large textureless regions
    const char* e = std::getenv("FBS_EMPTY_FORM");
    h->empty_form = e && e[0] == '1';
  }
  cudaGetDevice(&h->device);
  // Eq.(7): ω_d(dx,dy) = exp(-(dx²+dy²)/γ_d²); Eq.(8): ω_r(Δ) = exp(-Δ²/γ_r²)  (R#10).
  // k_agg evaluates the product as one power of two: ω_d ω_r = 2^(cd(dx,dy) + nkr Δ²),
  // cd = -log2(e)(dx²+dy²)/γ_d², nkr = -log2(e)/γ_r² (built in double, rounded once;
  // P:L199 "pre-calculated").
  const int K1 = 2 * radius + 1;
  const double gd = sigma_s, gr = sigma_r, l2e = 1.4426950408889634;
  for (int dy = -radius; dy <= radius; ++dy)
    for (int dx = -radius; dx <= radius; ++dx)
      h->cd[(dy + radius) * K1 + (dx + radius)] = (float)(-l2e * (double)(dx * dx + dy * dy) / (gd * gd));
  h->nkr = (float)(-l2e / (gr * gr));

  const size_t npix = (size_t)W * H;
  const size_t nvol = (size_t)h->Hv * h->Wv * h->nblk * kDB;
  bool ok = true;
  h->Wb = (W + kCX - 1) / kCX * (kCX / 32);
  h->Wg = guide_pitch(W, radius);
  const size_t ngp = (size_t)guide_rows(H, radius) * h->Wg;
  ok &= cudaMalloc(&h->gpadL, ngp * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->gpadR, ngp * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->bitsL, (size_t)H * h->Wb * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->bitsR, (size_t)H * h->Wb * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->volL, nvol * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->volR, nvol * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->dL, npix * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->dR, npix * 4) == cudaSuccess;
  ok &= cudaMalloc(&h->aggL, npix * h->nblk * kDB * sizeof(float)) == cudaSuccess;
  ok &= cudaMalloc(&h->agg3, npix * sizeof(float4)) == cudaSuccess;
  ok &= cudaMalloc(&h->tile_stats, 4 * sizeof(unsigned long long)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    free_all(h);
    delete h;
    fail(FBS_E_OOM, "fbs_create: device allocation failed");
    return nullptr;
  }
  // margins (and never-written rows) of the volumes hold the undefined cost
  k_fill<<<1184, 256>>>(h->volL, nvol, kUndef);
  k_fill<<<1184, 256>>>(h->volR, nvol, kUndef);
  k_fill<<<256, 256>>>(h->gpadL, ngp, kGuideUndef);  // margins: taps outside the frame
  k_fill<<<256, 256>>>(h->gpadR, ngp, kGuideUndef);
  cudaMemset(h->tile_stats, 0, 4 * sizeof(unsigned long long));
  cudaMemset(h->dL, 0xff, npix * 4);
  cudaMemset(h->dR, 0xff, npix * 4);
  cudaMemset(h->bitsL, 0, (size_t)H * h->Wb * 4);
  cudaMemset(h->bitsR, 0, (size_t)H * h->Wb * 4);
  if (cuda_check(cudaDeviceSynchronize(), "fbs_create init") != FBS_OK) {
    free_all(h);
    delete h;
    return nullptr;
  }
  // opt-in shared memory for every aggregation variant
#define FBS_SMEM_ATTR(RR) \
  cudaFuncSetAttribute(k_agg<RR, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(AggSmem<RR>)); \
  cudaFuncSetAttribute(k_agg<RR, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(AggSmem<RR>)); \
  cudaFuncSetAttribute(k_agg<RR, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(AggSmem<RR>));
  FBS_SMEM_ATTR(0) FBS_SMEM_ATTR(1) FBS_SMEM_ATTR(2) FBS_SMEM_ATTR(3) FBS_SMEM_ATTR(4)
  FBS_SMEM_ATTR(5) FBS_SMEM_ATTR(6)
#undef FBS_SMEM_ATTR
  cudaFuncSetAttribute(k_cost, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cost_smem_bytes(h->nblk));
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
static void fill_agg_args(const fbs_ctx* h, AggArgs& a) {
  a.W = h->W; a.H = h->H; a.D = h->D; a.d_min = h->d_min; a.d_max = h->d_max;
  a.nblk = h->nblk; a.Wv = h->Wv;
  std::memcpy(a.cd, h->cd, sizeof(a.cd));
  a.nkr = h->nkr;
  a.gpadL = h->gpadL; a.gpadR = h->gpadR; a.Wg = h->Wg;
}

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

static void launch_agg(const fbs_ctx* h, const AggArgs& a, int ty1, cudaStream_t s) {
  dim3 grid((h->W + kTX - 1) / kTX, ty1 - a.ty0, 2);
  switch (h->R) {
#define FBS_CASE(RR) \
  case RR:                                                                                        \
    if (a.exportR) /* debug export (results identical to both production variants) */                 \
      launch_pdl(k_agg<RR, false, true>, grid, dim3(AggGeom<RR>::THREADS), sizeof(AggSmem<RR>), s, a);   \
    else if (h->empty_form)                                                                             \
      launch_pdl(k_agg<RR, true, false>, grid, dim3(AggGeom<RR>::THREADS), sizeof(AggSmem<RR>), s, a);   \
    else                                                                                                \
      launch_pdl(k_agg<RR, false, false>, grid, dim3(AggGeom<RR>::THREADS), sizeof(AggSmem<RR>), s, a);  \
    break;
    FBS_CASE(0) FBS_CASE(1) FBS_CASE(2) FBS_CASE(3) FBS_CASE(4) FBS_CASE(5) FBS_CASE(6)
#undef FBS_CASE
  }
}

// Rows [r0, r1) of the output; every stage restricted to the rows it needs.
static int run_rows(fbs_ctx* h, const uint8_t* L, const uint8_t* Rimg, int r0, int r1, float* out,
                    float* aggL_exp, float* aggR_exp, cudaStream_t s) {
  const int W = h->W, H = h->H, R = h->R;
  // aggregation tiles are anchored at multiples of the tile height in frame rows, so a
  // pixel's denominator form never depends on the band; cost rows cover the
  // tiles' windows (the classification reads validity masks over them too)
  const int TY = agg_tile_h(R);
  const int ty0 = r0 / TY, ty1 = (r1 + TY - 1) / TY;
  const int c0 = std::max(0, ty0 * TY - R), c1 = std::min(H, ty1 * TY + R);  // cost rows
  h->launches = 0;
  cudaEvent_t* ev = nullptr;
  if (h->prof_ev && h->prof_n < h->prof_cap) ev = h->prof_ev + kEv * h->prof_n++;
  if (ev) cudaEventRecord(ev[0], s);
  {
    CostArgs ca;
    ca.W = W; ca.H = H; ca.D = h->D; ca.d_min = h->d_min; ca.nblk = h->nblk; ca.Wv = h->Wv; ca.R = R;
    ca.r0 = c0; ca.r1 = c1;
    ca.L = L; ca.Rimg = Rimg; ca.volL = h->volL; ca.volR = h->volR;
    ca.bitsL = h->bitsL; ca.bitsR = h->bitsR; ca.Wb = h->Wb;
    ca.gpadL = h->gpadL; ca.gpadR = h->gpadR; ca.Wg = h->Wg;
    const size_t smem = cost_smem_bytes(h->nblk);
    dim3 grd((W + kCX - 1) / kCX, c1 - c0, 2);
    k_cost<<<grd, 256, smem, s>>>(ca);
    h->launches += 1;
  }
  if (ev) cudaEventRecord(ev[1], s);
  AggArgs a;
  fill_agg_args(h, a);
  a.r0 = r0; a.r1 = r1; a.ty0 = ty0;
  a.volL = h->volL; a.volR = h->volR;

  a.bitsL = h->bitsL; a.bitsR = h->bitsR; a.Wb = h->Wb;
  a.dL = h->dL; a.dR = h->dR; a.aggL = h->aggL; a.exportR = aggR_exp;
  // one d-block: the left costs stay on chip and only Eq.(10)'s three are stored
  // (unless the debug export wants the whole left volume)
  a.agg3 = (h->nblk == 1 && !aggL_exp) ? h->agg3 : nullptr;
  a.tile_stats = ev ? h->tile_stats : nullptr;
  launch_agg(h, a, ty1, s);
  h->launches += 1;
  if (ev) cudaEventRecord(ev[2], s);
  {
    dim3 grd((W + 127) / 128, r1 - r0);
    launch_pdl(k_finalize, grd, dim3(128), 0, s, (const int32_t*)h->dL, (const int32_t*)h->dR,
               (const float*)h->aggL, (const float4*)a.agg3, h->nblk, W, r0, r1, h->d_min, h->d_max, out);
    h->launches += 1;
  }
  if (ev) cudaEventRecord(ev[3], s);
  if (aggL_exp) k_export_agg<<<1184, 256, 0, s>>>(h->aggL, W, H, h->D, h->nblk, aggL_exp);
  return cuda_check(cudaGetLastError(), "fbs launch");
}

extern "C" int fbs_compute(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* disp_out,
                           fbs_stream_t stream) {
  if (!h || !left || !right || !disp_out) return fail(FBS_E_ARG, "fbs_compute: NULL argument");
  return run_rows(h, left, right, 0, h->H, disp_out, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int fbs_compute_rows(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int row_begin,
                                int row_end, float* disp_band, fbs_stream_t stream) {
  if (!h || !left || !right || !disp_band) return fail(FBS_E_ARG, "fbs_compute_rows: NULL argument");
  if (row_begin < 0 || row_end > h->H || row_begin >= row_end)
    return fail(FBS_E_ARG, "fbs_compute_rows: need 0 <= row_begin < row_end <= H");
  return run_rows(h, left, right, row_begin, row_end, disp_band, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int fbs_compute_batch(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int n,
                                 float* disp_out, fbs_stream_t stream) {
  if (!h || !left || !right || !disp_out) return fail(FBS_E_ARG, "fbs_compute_batch: NULL argument");
  if (n < 1) return fail(FBS_E_ARG, "fbs_compute_batch: n must be >= 1");
  const size_t npix = (size_t)h->W * h->H;
  int launches = 0;
  for (int i = 0; i < n; ++i) {
    int rc = run_rows(h, left + i * npix, right + i * npix, 0, h->H, disp_out + i * npix, nullptr,
                      nullptr, (cudaStream_t)stream);
    if (rc != FBS_OK) return rc;
    launches += h->launches;
  }
  h->launches = launches;
  return FBS_OK;
}

// Host path: frame i's copies in (stream cs_in), compute (caller's stream) and
// copy out (cs_out) are ordered by events; two staging slots let frame i+1's
// upload and frame i-1's download run on the copy engines while frame i computes.
extern "C" int fbs_compute_host_batch(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int n,
                                      float* disp_out, fbs_stream_t stream) {
  if (!h || !left || !right || !disp_out) return fail(FBS_E_ARG, "fbs_compute_host_batch: NULL argument");
  if (n < 1) return fail(FBS_E_ARG, "fbs_compute_host_batch: n must be >= 1");
  const size_t npix = (size_t)h->W * h->H;
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->hL) {
    bool ok = cudaMalloc(&h->hL, 2 * npix) == cudaSuccess && cudaMalloc(&h->hR, 2 * npix) == cudaSuccess &&
              cudaMalloc(&h->hOut, 2 * npix * 4) == cudaSuccess;
    ok = ok && cudaStreamCreateWithFlags(&h->cs_in, cudaStreamNonBlocking) == cudaSuccess &&
         cudaStreamCreateWithFlags(&h->cs_out, cudaStreamNonBlocking) == cudaSuccess;
    for (int k = 0; ok && k < 2; ++k)
      ok = cudaEventCreateWithFlags(&h->ev_in[k], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&h->ev_done[k], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&h->ev_out[k], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      return fail(FBS_E_OOM, "fbs_compute_host_batch: staging allocation failed");
    }
  }
  int rc;
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
  if ((rc = cuda_check(cudaStreamSynchronize(h->cs_out), "fbs_compute_host_batch sync"))) return rc;
  return cuda_check(cudaStreamSynchronize(s), "fbs_compute_host_batch sync");
}

extern "C" int fbs_compute_host(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* disp_out,
                                fbs_stream_t stream) {
  if (!h || !left || !right || !disp_out) return fail(FBS_E_ARG, "fbs_compute_host: NULL argument");
  return fbs_compute_host_batch(h, left, right, 1, disp_out, stream);
}

extern "C" int fbs_debug_volumes(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* cost_l,
                                 float* cost_r, float* agg_l, float* agg_r, fbs_stream_t stream) {
  if (!h || !left || !right) return fail(FBS_E_ARG, "fbs_debug_volumes: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t npix = (size_t)h->W * h->H;
  float* tmp = nullptr;
  if (cudaMalloc(&tmp, npix * 4) != cudaSuccess) return fail(FBS_E_OOM, "fbs_debug_volumes: scratch");
  int rc = run_rows(h, left, right, 0, h->H, tmp, agg_l, agg_r, s);
  if (rc == FBS_OK) {
    if (cost_l) k_export_vol<<<1184, 256, 0, s>>>(h->volL, h->W, h->H, h->D, h->nblk, h->Wv, h->R, cost_l);
    if (cost_r) k_export_vol<<<1184, 256, 0, s>>>(h->volR, h->W, h->H, h->D, h->nblk, h->Wv, h->R, cost_r);
    rc = cuda_check(cudaGetLastError(), "fbs_debug_volumes export");
  }
  cudaStreamSynchronize(s);
  cudaFree(tmp);
  return rc;
}

extern "C" int fbs_debug_select(fbs_ctx* h, const float* agg_l, const float* agg_r, int32_t* disp_l,
                                int32_t* disp_r, float* disp_out, fbs_stream_t stream) {
  if (!h || !agg_l || !agg_r) return fail(FBS_E_ARG, "fbs_debug_select: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t npix = (size_t)h->W * h->H;
  const int nb = (int)((npix + 255) / 256);
  k_select_wta<<<nb, 256, 0, s>>>(agg_r, h->W, h->H, h->D, h->d_min, h->nblk, h->dR, nullptr);
  k_select_wta<<<nb, 256, 0, s>>>(agg_l, h->W, h->H, h->D, h->d_min, h->nblk, h->dL, h->aggL);
  if (disp_out) {
    dim3 grd((h->W + 127) / 128, h->H);
    k_finalize<<<grd, 128, 0, s>>>(h->dL, h->dR, h->aggL, nullptr, h->nblk, h->W, 0, h->H, h->d_min, h->d_max,
                                   disp_out);
  }
  if (disp_l) cudaMemcpyAsync(disp_l, h->dL, npix * 4, cudaMemcpyDeviceToDevice, s);
  if (disp_r) cudaMemcpyAsync(disp_r, h->dR, npix * 4, cudaMemcpyDeviceToDevice, s);
  return cuda_check(cudaGetLastError(), "fbs_debug_select");
}

extern "C" int fbs_debug_maps(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* disp_out,
                              int32_t* disp_l, int32_t* disp_r, fbs_stream_t stream) {
  if (!h || !left || !right || !disp_out) return fail(FBS_E_ARG, "fbs_debug_maps: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t npix = (size_t)h->W * h->H;
  int rc = run_rows(h, left, right, 0, h->H, disp_out, nullptr, nullptr, s);
  if (rc != FBS_OK) return rc;
  if (disp_l) cudaMemcpyAsync(disp_l, h->dL, npix * 4, cudaMemcpyDeviceToDevice, s);
  if (disp_r) cudaMemcpyAsync(disp_r, h->dR, npix * 4, cudaMemcpyDeviceToDevice, s);
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
