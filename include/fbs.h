/*
 * fbs.h — C ABI of the B200 (sm_100a) fast bilateral stereo (FBS) hot path.
 *
 * The library (paper_1807_02044_b200/libfbs.so) runs the method of
 * arXiv 1807.02044 ("Real-Time Subpixel Fast Bilateral Stereo", PAPER.md):
 *
 *   NCC matching cost      Eq.(1)-(3)   P:L66-84   (block statistics pre-computed)
 *   twin cost volumes      P:L86, P:L185           (left (u,v,d) == right (u-d,v,d))
 *   bilateral aggregation  Eq.(6)-(8)   P:L118-132 (ω_d ω_r pre-computed as exponent constants)
 *   winner-take-all        P:L140, P:L201          (highest aggregated NCC over [d_min, d_max])
 *   left-right consistency Eq.(9)       P:L148-153 (left image is the reference)
 *   parabola subpixel      Eq.(10)
 *
 * "P:Lnn" is a line of PAPER.md; DESIGN.md §3 lists every reading taken where
 * the paper is silent (borders, sentinels, tie-breaks, tolerances).
 *
 * Conventions shared by every entry point
 *   - Images are uint8 grayscale, H rows of W pixels, row-major, pitch W
 *     (R#3).  Disparity d >= 0 matches left (u,v) with right (u-d,v)
 *     (Eq.(1): i_r(x-d, y)).
 *   - The output disparity map is float32, H x W, pitch W.  Rejected or
 *     undefined pixels hold FBS_INVALID (-1.0f).  Valid values lie in
 *     [d_min, d_max].
 *   - Unless stated otherwise, pointers are DEVICE pointers on the device that
 *     was current when the handle was created, and calls are asynchronous on
 *     the given stream (0 = legacy default stream): they enqueue work and
 *     return.  The caller owns all I/O buffers and keeps them alive until the
 *     stream work completes.  The library owns all scratch, allocated once in
 *     fbs_create; fbs_compute never allocates or synchronises, so it can be
 *     captured in a CUDA graph.
 *   - A handle is NOT safe for concurrent use from several streams or threads
 *     (its scratch is shared): use one handle per stream.
 *   - Errors: every int-returning call returns FBS_OK (0) or a negative code;
 *     fbs_last_error() gives a thread-local message.  Launch failures return
 *     FBS_E_CUDA; asynchronous device faults surface at the caller's next
 *     synchronisation (CUDA convention).  No C++ exception crosses the ABI.
 */
#ifndef FBS_H_
#define FBS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FBS_INVALID (-1.0f) /* rejected / undefined pixel in a disparity map           */
#define FBS_SENTINEL (-2.0f) /* undefined entry of a (debug) cost or aggregated volume  */

enum {
  FBS_OK = 0,
  FBS_E_ARG = -1,         /* NULL pointer, bad handle, bad row range or batch size      */
  FBS_E_PARAM = -2,       /* radius<0, sigma_s/sigma_r not finite & > 0, d_min<0,       */
                          /* d_max<=d_min                                               */
  FBS_E_DIM = -3,         /* W<3 or H<3 (image must hold one 3x3 NCC block)             */
  FBS_E_UNSUPPORTED = -4, /* radius or disparity count beyond the compiled variants     */
  FBS_E_CUDA = -5,        /* CUDA runtime error (launch, copy, device)                  */
  FBS_E_OOM = -6          /* device allocation failed in fbs_create                     */
};

/* Opaque handle: frame geometry, parameters, weight tables, device scratch. */
typedef struct fbs_ctx fbs_ctx;

/* Stream type without pulling in cuda_runtime.h (same ABI as cudaStream_t). */
typedef struct CUstream_st* fbs_stream_t;

/*
 * fbs_create — validate parameters, build the ω_d / ω_r exponent constants (Eq.(7)(8),
 * P:L199 "pre-calculated"), allocate all scratch on the current device.
 *   W, H          frame size in pixels (>= 3 each)
 *   d_min, d_max  inclusive disparity search range, 0 <= d_min < d_max
 *   radius        ρ of Eq.(6): aggregation window (2ρ+1)^2; supported 1..FBS_MAX_RADIUS
 *                 (10; 6 on FBS_PATH_FUSED)
 *                 (0 is also accepted: the aggregation is then the identity)
 *   sigma_s       γ_d of Eq.(7), used verbatim as exp(-r^2/γ_d^2)   (> 0, finite)
 *   sigma_r       γ_r of Eq.(8), used verbatim as exp(-Δ^2/γ_r^2)   (> 0, finite)
 *                 The smallest tap weight exp(-2ρ²/γ_d² - 255²/γ_r²) must be at least
 *                 2^-FBS_MAX_WEIGHT_EXP2 (a normal fp32: no defined tap may flush to
 *                 zero, R#13); else FBS_E_UNSUPPORTED.  With γ_d = 5, ρ = 4
 *                 that is γ_r >= 27.6; γ_r has no upper bound (γ_r -> ∞: box weights).
 * The NCC block half-width ϱ is fixed at 1 and the LRC tolerance at
 * 1 pixel (R#17).  Returns NULL on error (reason: fbs_last_error()).
 * Synchronises the device once (scratch initialisation); not graph-capturable.
 */
fbs_ctx* fbs_create(int W, int H, int d_min, int d_max, int radius, float sigma_s, float sigma_r);

/* Implementation paths (fbs_create_ex).  Both compute the same function, parity-
 * tested against the same oracle:
 *   FBS_PATH_VOLUME  (fbs_create's default) block statistics + twin cost volumes in
 *                    device memory (L2-resident for Middlebury-sized frames), then
 *                    aggregation + WTA reading them, then LRC + subpixel.  Fastest.
 *   FBS_PATH_FUSED   costs computed into a shared-memory ring and aggregated there
 *                    (never written to HBM); several frames per launch.  ~20x less
 *                    DRAM traffic, ~20 % slower on B200 (profiles/ and DESIGN.md). */
#define FBS_PATH_VOLUME 0
#define FBS_PATH_FUSED 1

/* fbs_create_ex — fbs_create with an explicit implementation path (above); an
 * unknown path returns NULL (FBS_E_PARAM). */
fbs_ctx* fbs_create_ex(int W, int H, int d_min, int d_max, int radius, float sigma_s, float sigma_r,
                       int path);

/* fbs_create_band — a handle that serves only output rows [row_begin, row_end)
 * through fbs_compute_rows (the row-band partitioner's per-rank handle, DESIGN.md
 * §7): its cost volumes and left aggregated store cover just those rows plus the
 * tile / halo rows they need, so per-rank memory shrinks with the number of bands.
 * fbs_compute, _batch, _host* and the debug calls return FBS_E_ARG on it.
 * 0 <= row_begin < row_end <= H, else NULL. */
fbs_ctx* fbs_create_band(int W, int H, int d_min, int d_max, int radius, float sigma_s, float sigma_r,
                         int path, int row_begin, int row_end);

/* fbs_destroy — free the handle and its scratch.  The caller must have
 * synchronised all work enqueued with it.  NULL is a no-op. */
void fbs_destroy(fbs_ctx* h);

/* fbs_last_error — message of the last failing call on this thread ("" if none). */
const char* fbs_last_error(void);

/* Maximum supported aggregation radius ρ of this build (FBS_PATH_VOLUME; the
 * fused path supports ρ <= 6 and returns FBS_E_UNSUPPORTED above). */
#define FBS_MAX_RADIUS 10
/* -log2 of the smallest accepted tap weight ω_d·ω_r (see fbs_create). */
#define FBS_MAX_WEIGHT_EXP2 124

/*
 * fbs_compute — the whole hot path for one rectified pair:
 *   left, right  device uint8 [H][W]
 *   disp_out     device float [H][W]: subpixel disparity d^s of the left image
 *                (Eq.(10)) for LRC-consistent pixels (Eq.(9)), FBS_INVALID elsewhere.
 * Asynchronous on `stream`; graph-capturable.
 */
int fbs_compute(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* disp_out,
                fbs_stream_t stream);

/*
 * fbs_compute_rows — rows [row_begin, row_end) of what fbs_compute would write,
 * bit-identical to them.  left/right are the FULL frames (device); disp_band
 * is device float [(row_end-row_begin)][W].  Reads the input rows of the
 * aggregation tiles that cover the band plus their halo:
 * [floor(row_begin/T)*T - ρ - 1, ceil(row_end/T)*T + ρ + 1) clipped to the frame,
 * T = the path's tile height (≤ 12 rows).  Used by the row-band multi-GPU
 * partitioner.  rb0 <= row_begin < row_end <= rb1 (the handle's
 * rows: [0, H), or fbs_create_band's), else FBS_E_ARG.
 */
int fbs_compute_rows(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int row_begin,
                     int row_end, float* disp_band, fbs_stream_t stream);

/*
 * fbs_compute_rows_scatter — fbs_compute_rows whose final-map kernel stores each
 * pixel of rows [row_begin, row_end) into every one of `nouts` (1..8) full-frame
 * buffers (device float [H][W], frame coordinates) instead of a band buffer: the
 * WTA epilogue's band scatter of the row-band partitioner (NEXT-3).  With the
 * peers' symmetric-memory buffers (mapped into this GPU's address space) the
 * stores go over NVLink and replace the all-gather; `outs` is a host array of
 * device pointers.  Rows outside the band are not touched.  Asynchronous; the
 * caller synchronises the ranks (e.g. a symmetric-memory barrier) before reading.
 */
int fbs_compute_rows_scatter(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int row_begin,
                             int row_end, float* const* outs, int nouts, fbs_stream_t stream);

/*
 * fbs_compute_batch — n independent pairs, frame i at left + i*H*W,
 * right + i*H*W, output at disp_out + i*H*W (all device).  Equivalent to n
 * fbs_compute calls in order on `stream`.  n >= 1.
 */
int fbs_compute_batch(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int n,
                      float* disp_out, fbs_stream_t stream);

/*
 * fbs_compute_host — end-to-end call on HOST buffers: copies left/right
 * (host uint8 [H][W], ideally pinned) to the device, runs fbs_compute, copies
 * the map back to disp_out (host float [H][W]) and synchronises `stream`
 * before returning.  Blocking.
 */
int fbs_compute_host(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* disp_out,
                     fbs_stream_t stream);

/*
 * fbs_compute_host_batch — fbs_compute_host over n frames stored back to back
 * in HOST memory (left/right: n x [H][W] uint8, disp_out: n x [H][W] float;
 * pinned for the copies to be asynchronous).  Pipelined: frame i+1's upload and
 * frame i-1's download run on the copy engines (two internal streams, created
 * on first use and owned by the handle) while frame i computes on `stream`.
 * Results are identical to n calls of fbs_compute.  Blocking: returns after
 * the last map is in disp_out.  FBS_E_ARG for NULL pointers or n < 1.
 */
int fbs_compute_host_batch(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int n,
                           float* disp_out, fbs_stream_t stream);

/*
 * fbs_debug_volumes — test-only: one fbs_compute that also exports the
 * intermediate volumes, each device float [H][W][D] indexed
 * ((v*W+u)*D + d-d_min), FBS_SENTINEL where undefined:
 *   cost_l  c(u,v,d) of Eq.(1) (left reference)
 *   cost_r  the right-reference twin, cost_r(u-d,v,d) == cost_l(u,v,d)
 *   agg_l   Eq.(6) on cost_l guided by the left image
 *   agg_r   Eq.(6) on cost_r guided by the right image
 * and the results of that same launch:
 *   disp_out        device float [H][W] final map
 *   disp_l, disp_r  device int32 [H][W] integer WTA maps (-1 = INVALID)
 * Any output may be NULL.  The exporting kernel is a separate instantiation of
 * the production kernel (the same arithmetic plus stores); the GPU tests check
 * that its maps are bit-identical to fbs_compute's.  Asynchronous.
 */
int fbs_debug_volumes(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* cost_l,
                      float* cost_r, float* agg_l, float* agg_r, float* disp_out, int32_t* disp_l,
                      int32_t* disp_r, fbs_stream_t stream);

/*
 * fbs_debug_select — test-only: WTA on two given aggregated volumes (device
 * float [H][W][D], FBS_SENTINEL = undefined), then LRC and subpixel.
 *   disp_l, disp_r  device int32 [H][W] integer maps (-1 = INVALID), may be NULL
 *   disp_out        device float [H][W] final map, may be NULL
 * Asynchronous.
 */
int fbs_debug_select(fbs_ctx* h, const float* agg_l, const float* agg_r, int32_t* disp_l,
                     int32_t* disp_r, float* disp_out, fbs_stream_t stream);

/*
 * fbs_debug_maps — test-only: fbs_compute that also exports the integer WTA
 * maps of both sides (device int32 [H][W], -1 = INVALID; either may be NULL).
 */
int fbs_debug_maps(fbs_ctx* h, const uint8_t* left, const uint8_t* right, float* disp_out,
                   int32_t* disp_l, int32_t* disp_r, fbs_stream_t stream);

/*
 * fbs_stats — counters of the last fbs_compute* call on this handle, for the
 * bench's launch accounting (host ints, may be NULL):
 *   launches   kernels launched per frame
 * Returns FBS_OK.
 */
int fbs_stats(const fbs_ctx* h, int* launches);

/*
 * Live per-stage timing with CUDA events recorded on the launching stream.
 * fbs_profile_enable(h, n): the next n fbs_compute* frames record an event at
 * each stage boundary (n = 0 disables; n <= 65536; allocates the events, so
 * call it outside graph capture).  fbs_profile_read(h, stage_ms, ncalls)
 * waits for the recorded events, writes the summed milliseconds per stage to
 * stage_ms[FBS_NSTAGES] (host) and the number of frames to *ncalls, then
 * resets the counters.  Stages (one launch each): 0 block statistics + twin
 * cost volumes of both sides, 1 bilateral aggregation + WTA of both sides,
 * 2 LRC + subpixel.
 */
#define FBS_NSTAGES 3
int fbs_profile_enable(fbs_ctx* h, int n);
int fbs_profile_read(fbs_ctx* h, double* stage_ms, int* ncalls);

/*
 * fbs_tile_stats — how many (warp sub-tile, disparity block) units of the
 * aggregation took each exact form of the Eq.(6) denominator during the
 * frames profiled since the last call (counting is on while
 * fbs_profile_enable is active):
 *   fast     every tap defined but the guide's own border/textureless blocks
 *            (folded into the weights): Σ w', d-independent
 *   edge     the frame edge cuts taps off (left pass: x-d < 1; right pass:
 *            x+d > W-2): per-pixel prefix/suffix sums of column sums
 *   general  textureless blocks of the other image in range: explicit sum
 *   empty    no block of the other image in range is defined: every cost the
 *            unit reads is undefined, the aggregated costs are all SENTINEL
 *            (no arithmetic)
 * Synchronises the device; resets the counts.  Any pointer may be NULL.
 */
int fbs_tile_stats(fbs_ctx* h, long long* fast, long long* edge, long long* general, long long* empty);

/*
 * Disparity-range split (NEXT-3): rank k computes the WTA over its
 * own sub-range of disparities, the ranks reduce per-pixel 64-bit keys with MAX
 * (NCCL all_reduce), then one call applies LRC + subpixel.
 *
 * fbs_compute_keys — volume-path handles only (else FBS_E_UNSUPPORTED).  Only the
 * disparities [c_lo, c_hi] ⊆ [d_min, d_max] of the handle compete in the WTA; create
 * the handle with one disparity beyond each end of [c_lo, c_hi] (clipped to the
 * global range) so the subpixel neighbours exist.  Outputs (device, [H][W]):
 *   keys_l, keys_r  uint64: (order-preserving bits of c_agg(p, d*)) << 32 | (0xFFFFFFFF - d*),
 *                   d* the global disparity; MAX over keys = highest aggregated cost,
 *                   smallest d on ties; 0 = no defined cost.
 *   rec_l           float4 per pixel: (c(d*-1), c(d*), c(d*+1), 0) of the left volume,
 *                   FBS_SENTINEL where undefined or outside the handle's range.
 * fbs_finalize_keys — LRC (Eq.(9)) + subpixel (Eq.(10)) of the global range
 * [d_min, d_max] from the reduced keys and the winners' records -> disp_out
 * (device float [H][W]).  No handle needed.  Both asynchronous on `stream`.
 */
int fbs_compute_keys(fbs_ctx* h, const uint8_t* left, const uint8_t* right, int c_lo, int c_hi,
                     uint64_t* keys_l, uint64_t* keys_r, float* rec_l, fbs_stream_t stream);
int fbs_finalize_keys(int W, int H, int d_min, int d_max, const uint64_t* keys_l, const uint64_t* keys_r,
                      const float* rec_l, float* disp_out, fbs_stream_t stream);

/*
 * Sparse search range (NEXT-4; the paper's future work; readings R#31-R#33
 * in DESIGN.md).  Volume-path handles only (else FBS_E_UNSUPPORTED).
 *
 * fbs_suggest_ranges — per-pixel suggested ranges from "reliable feature points":
 *   seed_disp  device float [H][W]: a disparity map whose values >= 0 are the
 *              feature points (e.g. the previous frame's fbs_compute output)
 *   margin     disparities added on each side (>= 0)
 *   ranges_l, ranges_r  device int16 [H][W][2] out: (lo, hi) per pixel of the left
 *              / right image = [floor(min) - margin, ceil(max) + margin] of the seeds
 *              of its frame-anchored 16x16 tile (left seeds forward-warped to
 *              x - round(s) for the right image), clipped to [d_min, d_max]; tiles
 *              without a seed get [d_min, d_max].
 * fbs_compute_ranged — fbs_compute with the WTA of each pixel restricted to its
 *   range (ranges_* as above; lo > hi = no candidate); d-blocks outside the union
 *   of a tile's ranges are not aggregated at all.  Subpixel only when d*±1 lie in
 *   the pixel's range.  Both asynchronous on `stream`.
 */
int fbs_suggest_ranges(fbs_ctx* h, const float* seed_disp, int margin, int16_t* ranges_l, int16_t* ranges_r,
                       fbs_stream_t stream);
int fbs_compute_ranged(fbs_ctx* h, const uint8_t* left, const uint8_t* right, const int16_t* ranges_l,
                       const int16_t* ranges_r, float* disp_out, fbs_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* FBS_H_ */
