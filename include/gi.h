/* gi.h -- C ABI of libgi, the B200 (sm_100a) GaussianImage hot path.
 *
 * GaussianImage (arXiv 2403.08551) represents an image by N 2-D Gaussians of
 * 8 parameters each (Sec. 3.2) and renders pixel i as the
 * order-free accumulated sum  C_i = sum_n c'_n exp(-sigma_n)   (Eq. 7,
 * PAPER.md:226-232), sigma_n = 1/2 d^T Sigma_n^-1 d (Eq. 5),
 * Sigma = L L^T (Eq. 1).  Fitting minimises the L2 loss
 * with the analytic gradients of Appendix A.
 * Codec decode: fp16 positions, Eq. 8 dequantisation, Eq. 9 RVQ
 * (PAPER.md:254-270).  Readings of silent/garbled passages (R1..R25) are in
 * DESIGN.md; the numbers below refer to them.
 *
 * Conventions (all entry points):
 *  - Every array argument is a caller-owned DEVICE pointer unless stated.
 *    libgi never allocates on the hot path; workspaces are caller-provided and
 *    sized by the *_workspace_bytes queries (the one exception is the setup
 *    call gi_peer_alloc, which creates an IPC-shareable exchange buffer).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call taking a stream is stream-ordered, never synchronises the host
 *    and is CUDA-graph capturable (gi_check, which syncs, and the gi_peer_*
 *    setup calls are the exceptions).
 *  - Layouts are fixed: parameters/gradients AoS [B][N][8] fp32 =
 *    {mu_x, mu_y, l1, l2, l3, c'_r, c'_g, c'_b}, 16-byte aligned; images
 *    planar fp32 [B][3][H][W], y down, pixel (x, y) has centre (x+1/2, y+1/2)
 *    (R1, R2).  B = gi_frame.batch images of the same size and the same N
 *    are processed per launch; tile and Gaussian ids are global:
 *    tile = img*T + ty*ceil(W/16) + tx, gid = img*N + n.
 *  - Errors: GI_EINVAL for bad host-visible arguments (nothing is launched);
 *    GI_ECUDA for a launch failure (detail in gi_last_error(), thread-local);
 *    device-side conditions (key-capacity overflow, non-finite parameters)
 *    are written to device words the caller checks after a sync.
 *  - No global mutable state: calls are re-entrant.
 */
#ifndef GI_H
#define GI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GI_ABI_VERSION 1

typedef enum {
    GI_OK = 0,
    GI_EINVAL = 1,      /* bad argument (shape, alignment, size, NULL)        */
    GI_ECUDA = 2,       /* CUDA launch / runtime error, see gi_last_error()   */
    GI_ECAPACITY = 3,   /* more (tile, gaussian) keys than key_capacity       */
    GI_EFORMAT = 4,     /* codec metadata inconsistent with the payload size  */
    GI_ENONFINITE = 5   /* a parameter became NaN/Inf                         */
} gi_status;

/* One frame geometry shared by the B images of a launch. */
typedef struct {
    int32_t width, height;  /* pixels, 1..32767                                */
    int32_t tile;           /* tile edge in pixels; must be 16 (R23)           */
    int32_t batch;          /* images per launch B >= 1                        */
    float k;                /* box half-extent in standard deviations (R6), >0 */
} gi_frame;

/* Parameterisation flags (bit field).  Position, params[0:2]: */
#define GI_POS_LOGIT 0u       /* raw logits, u = tanh(mu_raw) (App. C)  */
#define GI_POS_NORMALIZED 1u  /* already u in [-1,1] (decode path, R19) */
/* Covariance, params[2:5]: Cholesky (l1, l2, l3), Sigma = L L^T (Eq. 1), the
 * default; or, OR-ed in, the rotation-scaling factorisation (theta, s1, s2),
 * Sigma = (R S)(R S)^T with S = diag(s1 + 1/2, s2 + 1/2) (Eq. 2-3, App. C;
 * NEXT-3); its gradients follow App. A.2. */
#define GI_COV_RS 2u

/* Size in bytes of one projected-Gaussian record (opaque, 16-B aligned). */
#define GI_PROJ_BYTES 48

const char* gi_status_string(gi_status s);
const char* gi_last_error(void);
int32_t gi_abi_version(void);

/* T = ceil(W/16) * ceil(H/16) tiles per image. */
int32_t gi_num_tiles(const gi_frame* f);
size_t gi_proj_bytes(int32_t n, const gi_frame* f);   /* B * n * GI_PROJ_BYTES */

/* --- a1. Projection ("formation"; Eq. 1; App. C) ---------------------
 * For every Gaussian: u = tanh(mu_raw) (or u given), mu = (u + 1) * (W, H)/2
 * in fp64, split into an integer pixel plus an fp32 fraction; effective
 * L = [[l1 + 1/2, 0], [l2, l3 + 1/2]]; the conic of Sigma^-1 = L^-T L^-1; the
 * integer pixel box of the k-sigma ellipse by the fp32 recipe of R7 (box
 * empty and Gaussian culled iff l1+1/2 == 0 or l3+1/2 == 0, R8); its tile
 * rectangle and tile count.
 *   params         [B][n][8] fp32 in
 *   proj           [B][n] records of GI_PROJ_BYTES out
 *   tiles_touched  [B][n] u32 out: number of 16x16 tiles the box overlaps
 * n may be 0. */
gi_status gi_project(const float* params, int32_t n, const gi_frame* f, uint32_t flags,
                     void* proj, uint32_t* tiles_touched, void* stream);

/* --- a2. Tile binning, no depth key (north_star) --------------------
 * One key (tile, gid) per tile of each Gaussian's rectangle, grouped by tile
 * id only (no depth key) and ascending gid inside a tile, i.e. the unique
 * lexicographic (tile, gid) order (R9).  Done as one counting pass on the
 * tile digit (per-tile counts -> scan -> slot scatter) followed by a per-tile
 * sort on gid; hand-written, CUB-free.
 *   key_tile, key_gid  [key_capacity] u32 out (first K valid)
 *   tile_range [B*T + 1] u32 out: tile_range[t] = first key index with
 *              key_tile >= t (entries clamped to key_capacity)
 *   n_keys     [1] u32 device out: K, the TRUE key count.  If
 *              K > key_capacity the keys are truncated (consistently with
 *              the clamped ranges) and the caller must retry with a larger
 *              capacity (gi_check reports GI_ECAPACITY).
 *   ws         workspace of gi_bin_workspace_bytes() bytes (device). */
size_t gi_bin_workspace_bytes(int32_t n, int64_t key_capacity, const gi_frame* f);
gi_status gi_bin(const void* proj, const uint32_t* tiles_touched, int32_t n, const gi_frame* f,
                 int64_t key_capacity, void* ws, size_t ws_bytes, uint32_t* key_tile,
                 uint32_t* key_gid, uint32_t* tile_range, uint32_t* n_keys, void* stream);

/* --- a3. Forward accumulated summation (Eq. 7) -----------------------------
 * C_k(x, y) = sum over keys of tile(x, y) of
 *             [x0 <= x <= x1 and y0 <= y <= y1] c'_k exp(-sigma(x + 1/2, y + 1/2))
 * Unclamped (R10).  image [B][3][H][W] fp32 out.  The sum is order-free
 * (P:214): per batch of a tile's keys each term is rounded to a 2^-s fixed
 * point (s from the batch's largest |c'|, terms <= 2^22) and added exactly
 * with integer atomics, then converted once (launches of < 3,072 tiles with
 * >= 8 Gaussians per tile; else fp32 sums in ascending gid) -- deterministic
 * either way.  A non-finite c' makes its tiles' pixels NaN. */
gi_status gi_render(const void* proj, const uint32_t* key_gid, const uint32_t* tile_range,
                    int32_t n, const gi_frame* f, float* image, void* stream);

/* --- a4. Loss + backward (Appendix A) ---------------------
 * Upstream g = dL/dC: either given (dL_dimage != NULL), or the L2 loss
 * L = mean over 3HW of (C - target)^2 with g = 2 (C - target) / (3HW), where
 * C is recomputed in-kernel (fused forward; image_out may receive it).
 * grads [B][n][8] fp32 OVERWRITTEN with dL/dparams (same layout as params;
 * dl1 = 2 g1 l1 + 2 g2 l2, dl2 = 2 g2 l1 + 2 g3 l2 (R14 corrects P:627),
 * dl3 = 2 g3 l3 in G = dL/dSigma; dmu_raw chained through tanh when flags ==
 * GI_POS_LOGIT).  Deterministic: per-(tile, Gaussian) partial sums are
 * written to the workspace at the key's index and reduced per Gaussian in
 * row-major tile order (no atomics).
 *   loss       [B] fp32 out, or NULL (MSE mode only)
 *   image_out  [B][3][H][W] fp32 out, or NULL (MSE mode only)
 *   ws         gi_backward_workspace_bytes() bytes (device). */
size_t gi_backward_workspace_bytes(int32_t n, int64_t key_capacity, const gi_frame* f);
gi_status gi_render_backward(const float* params, const void* proj, const uint32_t* key_gid,
                             const uint32_t* tile_range, int32_t n, const gi_frame* f,
                             uint32_t flags,
                             const float* dL_dimage, const float* target,
                             int64_t key_capacity, void* ws, size_t ws_bytes,
                             float* grads, float* loss, float* image_out, void* stream);

/* --- a5. Adam (north_star; R16) ---------------------------------------------
 * Elementwise over `count` fp32 scalars, step t >= 1 (1-based):
 *   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;
 *   p -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
 * nonfinite_flag (device u32, may be NULL) gets bit 0 set if any updated p is
 * NaN/Inf (GI_ENONFINITE via gi_check).  params/grads/m/v 16-B aligned. */
gi_status gi_adam_step(float* params, const float* grads, float* m, float* v, int64_t count,
                       int32_t step, float lr, float beta1, float beta2, float eps,
                       uint32_t* nonfinite_flag, void* stream);

/* --- NEXT-1: Adan, the paper's optimiser (rule of the cited Adan
 * reference, R28) -----------------------------------------------
 *   d = g - g_prev (0 at t = 1); m = b1 m + (1-b1) g; v = b2 v + (1-b2) d;
 *   n = b3 n + (1-b3) (g + b2 d)^2;
 *   p = p (1 - lr wd) - lr (m/(1-b1^t) + b2 v/(1-b2^t)) / (sqrt(n/(1-b3^t)) + eps);
 *   g_prev = g.   Defaults b = (0.98, 0.92, 0.99), eps = 1e-8, wd = 0.
 * count multiple of 8, all buffers 16-B aligned. */
gi_status gi_adan_step(float* params, const float* grads, float* m, float* v, float* n,
                       float* grad_prev, int64_t count, int32_t step, float lr, float beta1,
                       float beta2, float beta3, float eps, float weight_decay,
                       uint32_t* nonfinite_flag, void* stream);

/* lr_t = lr0 * 0.5^floor((t - 1) / half_every)  ("halved every 20000
 * steps", R17).  Host helper. */
double gi_lr_at(int32_t step, double lr0, int32_t half_every);

/* --- fused fit iteration (graph-capturable) ---------------------------------
 * One step of the fitting loop on B images: project (+ per-tile counts) ->
 * bin -> fused forward/L2/backward -> per-Gaussian finalize fused with Adam
 * (grads are still written out), with the 1-based step
 * counter t kept on the device (*step_counter is incremented once per call by
 * the projection kernel, then used for the bias correction and
 * lr_t = lr0 * 0.5^floor((t-1)/half_every)).
 *   fit_ws        gi_fit_workspace_bytes() bytes: holds proj, tiles_touched,
 *                 keys, ranges, n_keys and both stage workspaces.  MUST be
 *                 zero-filled once before its first use (it carries per-tile
 *                 counters that every non-chained fused call leaves zeroed
 *                 for the next).  gi_fit_step, gi_fit_grads and gi_fit_prime
 *                 clear the binning state themselves (one memset), so they
 *                 may follow chained steps on the same workspace
 *   loss          [B] fp32 out (L2 loss of the step's forward), may be NULL
 *   status_flags  device u32, bit 0 set on a non-finite parameter, may be NULL
 *   stage_events  NULL, or 6 cudaEvent_t (as void*) recorded (external) at
 *                 the stage boundaries: [0] start, [1] after project,
 *                 [2] after bin, [3] after the fused tile kernel,
 *                 [4] after finalize + Adam + loss, [5] end.  Lets a caller
 *                 time each stage inside a captured CUDA graph. */
size_t gi_fit_workspace_bytes(int32_t n, int64_t key_capacity, const gi_frame* f);
gi_status gi_fit_step(float* params, float* grads, float* m, float* v, const float* target,
                      int32_t n, const gi_frame* f, uint32_t flags, int64_t key_capacity,
                      void* fit_ws, size_t ws_bytes, uint32_t* step_counter, float lr0,
                      int32_t half_every, float beta1, float beta2, float eps, float* loss,
                      uint32_t* status_flags, void* const* stage_events, void* stream);
/* Fused fit step with Adan (NEXT-1, the paper's optimiser; update rule
 * of gi_adan_step) instead of Adam: the same stages as gi_fit_step, the Adan
 * update fused into the finalize kernel (3 kernels); device step counter.
 * n, grad_prev: [B][N][8] fp32 Adan state (zero before step 1), 16-B aligned. */
gi_status gi_fit_step_adan(float* params, float* grads, float* m, float* v, float* n,
                           float* grad_prev, const float* target, int32_t n_gauss, const gi_frame* f,
                           uint32_t flags, int64_t key_capacity, void* fit_ws, size_t ws_bytes,
                           uint32_t* step_counter, float lr0, int32_t half_every, float beta1,
                           float beta2, float beta3, float eps, float weight_decay, float* loss,
                           uint32_t* status_flags, void* stream);

/* Chained fit steps: identical arithmetic to gi_fit_step, but the projection
 * of step t+1 is fused into the finalize + Adam kernel of step t (the thread
 * that updated a Gaussian projects it at once), so a step is 2 kernels.
 * gi_fit_prime projects the current params into fit_ws; every
 * gi_fit_step_chained call then REQUIRES that fit_ws holds the projection of
 * the current params -- i.e. it follows gi_fit_prime or another chained call
 * on the same params/fit_ws with no other writer of params in between -- and
 * leaves it so for the next call.  Same arguments as gi_fit_step.
 * A chained call leaves the NEXT step's keys (per-tile counts, slab entries)
 * in fit_ws.  gi_fit_prime clears that state before it projects, so it is
 * also the recovery path after params were modified between chained steps.
 * gi_fit_reset clears it without projecting: required before gi_render_frame
 * or gi_decode_render_frame reuse a workspace a chained step left (they
 * assume zeroed counters and do not clear them, to stay one memset-free
 * graph).  Errors: GI_EINVAL (frame, n, capacity, workspace size/alignment),
 * GI_ECUDA. */
gi_status gi_fit_reset(int32_t n, const gi_frame* f, int64_t key_capacity, void* fit_ws,
                       size_t ws_bytes, void* stream);
gi_status gi_fit_prime(const float* params, int32_t n, const gi_frame* f, uint32_t flags,
                       int64_t key_capacity, void* fit_ws, size_t ws_bytes, void* stream);
gi_status gi_fit_step_chained(float* params, float* grads, float* m, float* v, const float* target,
                              int32_t n, const gi_frame* f, uint32_t flags, int64_t key_capacity,
                              void* fit_ws, size_t ws_bytes, uint32_t* step_counter, float lr0,
                              int32_t half_every, float beta1, float beta2, float eps, float* loss,
                              uint32_t* status_flags, void* const* stage_events, void* stream);
/* Chained Adan fit step: gi_fit_step_adan's arithmetic with gi_fit_step_chained's
 * structure (2 kernels; requires gi_fit_prime as gi_fit_step_chained does). */
gi_status gi_fit_step_adan_chained(float* params, float* grads, float* m, float* v, float* n,
                                   float* grad_prev, const float* target, int32_t n_gauss,
                                   const gi_frame* f, uint32_t flags, int64_t key_capacity,
                                   void* fit_ws, size_t ws_bytes, uint32_t* step_counter, float lr0,
                                   int32_t half_every, float beta1, float beta2, float beta3,
                                   float eps, float weight_decay, float* loss,
                                   uint32_t* status_flags, void* stream);

/* --- NEXT-4: single-image spatial sharding -----------
 * The gradient half of a fused fit step restricted to the tile rows
 * [tile_row0, tile_row0 + tile_rows) of every image (tile_rows < 0: all;
 * tile_rows = 0: an empty window -- zero grads and loss, as for a rank that
 * owns no rows):
 * project (+ direct binning of the keys in the window) -> fused Eq. 7 + L2 +
 * App. A backward over the window's tiles -> finalize WITHOUT an optimiser.
 * grads [B][n][8] out = the window's share of dL/dparams and loss [B] out =
 * its share of the L2 loss (normalised by the whole image): both are
 * sums over tiles, so over a partition of the rows they add up to the whole
 * image's (up to fp32 summation order).  Ranks of a sharded fit all-reduce
 * grads and loss (NCCL) and apply the same gi_adam_step, or exchange them
 * over peer memory with gi_peer_adam_step (below).  Workspace as
 * gi_fit_step (gi_fit_workspace_bytes), zero-filled once. */
gi_status gi_fit_grads(const float* params, float* grads, const float* target, int32_t n,
                       const gi_frame* f, uint32_t flags, int32_t tile_row0, int32_t tile_rows,
                       int64_t key_capacity, void* fit_ws, size_t ws_bytes, float* loss,
                       void* stream);

/* --- NEXT-4 gradient exchange over peer memory -----------------------------
 * The exchange of spatial sharding fused with the optimiser: each of G ranks
 * (one process per GPU of a node, NVLink/NVSwitch peers) writes its window's
 * gradients ([B][n][8] fp32, `count` floats) followed by its n_loss loss
 * floats into an exchange buffer from gi_peer_alloc; the ranks swap the
 * 64-byte IPC handles (any host channel, e.g. torch.distributed) and map each
 * other's buffers with gi_peer_open.  gi_peer_adam_step then reads the G
 * buffers (grads[r], rank order r = 0 .. G-1, the same array on every rank),
 * sums them elementwise in that order -- so every rank computes identical
 * sums and the replicas stay bit-identical -- and applies Adam with
 * gi_adam_step's arithmetic (bit-identical to gi_adam_step on the summed
 * gradient); loss_out[j] = sum_r grads[r][count + j].  The caller orders the
 * ranks around the step (every rank's gradients complete before any rank
 * reads them; every read complete before the next step overwrites them):
 * a barrier of its host channel after a stream sync, on both sides.
 * G <= 8, n_loss <= 32; buffers 16-B aligned (gi_peer_alloc's are).
 * gi_peer_alloc: cudaMalloc of `bytes` (zero-filled) + its IPC handle
 * (handle: 64 bytes out); gi_peer_open: map a peer's handle (not one of this
 * process's own allocations); gi_peer_close / gi_peer_free undo them. */
gi_status gi_peer_alloc(size_t bytes, void** ptr, void* handle);
gi_status gi_peer_free(void* ptr);
gi_status gi_peer_open(const void* handle, void** ptr);
gi_status gi_peer_close(void* ptr);
gi_status gi_peer_adam_step(float* params, float* m, float* v, const float* const* grads,
                            int32_t G, int64_t count, int32_t step, float lr, float beta1,
                            float beta2, float eps, int32_t n_loss, float* loss_out,
                            uint32_t* nonfinite_flag, void* stream);

/* --- fused render of a frame (graph-capturable) ---------------------------
 * project (+ per-tile counts) -> bin -> Eq. 7 render in one call; the per-tile
 * gid ordering of binning happens inside the render kernel.  Same workspace
 * layout, size and zero-fill rule as gi_fit_step (gi_fit_workspace_bytes);
 * consecutive kernels overlap via programmatic dependent launch; n_keys for
 * gi_check via gi_fit_n_keys(frame_ws, ...).  image [B][3][H][W] out. */
gi_status gi_render_frame(const float* params, int32_t n, const gi_frame* f, uint32_t flags,
                          int64_t key_capacity, void* frame_ws, size_t ws_bytes, float* image,
                          void* stream);

/* Direct-binning state inside fit_ws (inspection, e.g. parity tests): after
 * gi_fit_prime or a chained step, image b's tile t (global tile g = b*T + t)
 * holds tile_count[g * count_stride] keys (the fit paths' layout; the frame
 * entry points space the counters 4x wider below 3,072 tiles per launch); the first min(count, slab_capacity)
 * gids are slab[g * slab_capacity + 0 ..) in atomic (unordered) order; a
 * tile with more keys streams them from all Gaussians of its image.  Device
 * pointers into fit_ws; nothing is launched.  GI_EINVAL on bad arguments. */
gi_status gi_fit_bin_view(const void* fit_ws, int32_t n, int64_t key_capacity, const gi_frame* f,
                          const uint32_t** tile_count, uint32_t* count_stride,
                          const uint32_t** slab, uint32_t* slab_capacity);

/* Segment statistics inside fit_ws (device u32[2], accumulated by every
 * consumer tile kernel since the last gi_fit_prime / gi_fit_reset /
 * non-chained step, which zero them): [0] tiles whose key count exceeded the
 * direct-binning slab (streamed from all N Gaussians of the image: the slow
 * path), [1] tiles whose segment exceeded the kernel's shared sort buffer
 * (rebuilt in gid order in global memory).  The per-tile slab holds
 * max(key_capacity / tiles, 1024) keys (GI_SLAB_MIN overrides the 1024).
 * NULL on bad arguments; nothing is launched. */
uint32_t* gi_fit_seg_stats(void* fit_ws, int32_t n, int64_t key_capacity, const gi_frame* f);

/* Device status words inside fit_ws (for gi_check): */
const uint32_t* gi_fit_n_keys(const void* fit_ws, int32_t n, int64_t key_capacity,
                              const gi_frame* f);

/* --- a6. Attribute decode (record layout SPEC.md:404) ------------
 * payload: n records of R = 32 + 3*bits + stages*ceil(log2 codebook) bits,
 * MSB-first, concatenated (device bytes, >= ceil(n*R/8)).  Per record:
 *   u_x, u_y  = IEEE binary16 -> fp32 (exact)
 *   l_i       = fmaf(code_i, gamma_i, beta_i)  (one fp32 rounding)    Eq. 8
 *   c'        = C^1[i^1] + ... + C^M[i^M] (fp32, stage order)         Eq. 9
 * params [n][8] fp32 out, positions normalised: project with
 * GI_POS_NORMALIZED.  GI_EFORMAT if R > 64, bits > 16, codebook < 2 or
 * stages > 8 or payload_bytes too small.  An index field >= codebook (only
 * possible when codebook is not a power of two: a corrupt record) is clamped
 * to codebook - 1, so no read leaves the codebooks. */
typedef struct {
    int32_t n, bits, stages, codebook;
    float gamma[3], beta[3];
    const float* codebooks;   /* device [stages][codebook][3] fp32 */
} gi_codec_meta;
gi_status gi_vq_decode(const uint8_t* payload, size_t payload_bytes, const gi_codec_meta* meta,
                       float* params, void* stream);

/* Decode + render of one codec frame (configs[4]) in two kernels: the decode
 * of record g (exactly gi_vq_decode's) is fused into the projection of
 * Gaussian g (GI_POS_NORMALIZED; a6 + a1 in one pass, no parameter round
 * trip), then the Eq. 7 render as in gi_render_frame.  f->batch must be 1 and
 * n = meta->n.  frame_ws: as gi_render_frame (gi_fit_workspace_bytes(n, ...),
 * zero-filled once).  params [n][8] out (may be NULL): the decoded records,
 * bit-identical to gi_vq_decode.  image [1][3][H][W] out: bit-identical to
 * gi_vq_decode followed by gi_render_frame(GI_POS_NORMALIZED).  Errors as
 * gi_vq_decode and gi_render_frame. */
gi_status gi_decode_render_frame(const uint8_t* payload, size_t payload_bytes,
                                 const gi_codec_meta* meta, const gi_frame* f,
                                 int64_t key_capacity, void* frame_ws, size_t ws_bytes,
                                 float* params, float* image, void* stream);

/* --- NEXT-2 encoder: attribute quantisation (SPEC quant/codec) ---
 * The inverse of gi_vq_decode: per Gaussian of params [n][8] fp32 (raw
 * positions through tanh unless flags & GI_POS_NORMALIZED; Cholesky l as
 * stored; colours c'):
 *   u     = binary16(round_fp32(tanh(mu_raw))), round to nearest even
 *   code  = rint(clamp((l_i - beta_i) / gamma_i, 0, 2^bits - 1)) in fp32 Eq. 8
 *   i^m   = argmin_k ||C^m[k] - (c' - c^^{m-1})||^2, fp32, ties -> lowest
 *           index, c^^{m-1} = C^1[i^1] + ... in stage order              Eq. 9
 * (reading R30: the paper fixes no precision or tie rule).  Outputs (either
 * may be NULL): payload -- the records packed exactly as gi_vq_decode reads
 * them (the call zero-fills the first ceil(n*R/8) bytes; payload_bytes must
 * cover them); eff [n][8] fp32 -- the dequantised parameters, bit-identical
 * to gi_vq_decode(payload).  Same GI_EFORMAT rules as gi_vq_decode.
 * payload must be 4-byte aligned (records are OR-ed into 32-bit words):
 * GI_EINVAL otherwise. */
gi_status gi_vq_encode(const float* params, uint32_t flags, const gi_codec_meta* meta,
                       uint8_t* payload, size_t payload_bytes, float* eff, void* stream);

/* NEXT-2 RVQ codebook initialisation: one K-means (Lloyd) iteration (P:307
 * "initialized using the K-means algorithm"; 5 iterations).  points
 * [n][3] fp32 (colours c', or stage-m residuals); centroids [B][3] fp32
 * in/out (2 <= B <= 256); assign [n] u32 out (may be NULL): the nearest
 * centroid by the fp32 distance and tie rule of gi_vq_encode.  A centroid
 * with points becomes their mean (sums in 2^-40 fixed point, order-
 * independent, divided in fp64, rounded once to fp32); an empty cluster keeps
 * its centroid (reading R31).  ws: gi_kmeans_workspace_bytes(B) device
 * bytes, zero-filled before the first call (left zeroed by each call). */
size_t gi_kmeans_workspace_bytes(int32_t B);
gi_status gi_kmeans_step(const float* points, int32_t n, int32_t B, float* centroids,
                         uint32_t* assign, void* ws, size_t ws_bytes, void* stream);

/* NEXT-2 attribute quantisation-aware fine-tuning step (QAT; Fig. 3, P:249-
 * 276), one image (f->batch == 1), graph-capturable:
 *   p^ = Q(p) (gi_vq_encode's quantisers, gamma|beta = qparams[0..5] and
 *   books read on the device) -> project + direct binning -> fused Eq. 7 +
 *   L2 + App. A backward on p^ (positions normalised) -> straight-through
 *   gradients (reading R32: d/draw_mu = d/du / cosh^2, l passes inside the
 *   clamp range, LSQ+ gamma/beta gradients without scaling, c' gets d/dc^)
 *   -> Adam (constant cfg->lr, bias-corrected by the device step counter) on
 *   params and on qparams -> EMA codebooks (reading R33: N <- d N + (1-d) n,
 *   S <- d S + (1-d) sum r, C <- S / N where n > 0).
 * params, m, v [n][8] in/out; eff [n][8] out (p^); grads [n][8] out
 * (d/draw); qparams, qm, qv [6] in/out; books [M][B][3], ema_n [M][B],
 * ema_s [M][B][3] in/out; losses [9] out = {L_rec + lambda L_c, L_rec, L_c
 * (Eq. 10 with the pre-update books), d/dgamma_0..2, d/dbeta_0..2}.  All sums across Gaussians are
 * fixed-point integer sums: deterministic.  ws: gi_qat_workspace_bytes()
 * device bytes, zero-filled once. */
typedef struct {
    int32_t bits, stages, codebook;
    float lr, lambda, decay, beta1, beta2, eps;
} gi_qat_config;
size_t gi_qat_workspace_bytes(int32_t n, int64_t key_capacity, const gi_frame* f,
                              const gi_qat_config* cfg);
gi_status gi_qat_step(float* params, float* m, float* v, float* eff, float* grads, float* qparams,
                      float* qm, float* qv, float* books, float* ema_n, float* ema_s,
                      const float* target, int32_t n, const gi_frame* f, const gi_qat_config* cfg,
                      int64_t key_capacity, void* ws, size_t ws_bytes, uint32_t* step_counter,
                      float* losses, uint32_t* status_flags, void* stream);

/* --- fit targets from 8-bit images ------------------------------------------
 * The paper's datasets (Kodak, DIV2K) are 24-bit RGB images.  A fit
 * whose targets stream in (one image per step) moves each across the host
 * link as 8-bit RGB (1.18 MB for a Kodak image, a quarter of its fp32 form):
 * gi_target_upload_rgb8 on a copy stream, gi_target_from_rgb8 on the compute
 * stream before the step.  Events are cudaEvent_t handles the caller created
 * (NULL: no wait / no record).  Errors: GI_EINVAL for a bad frame or a NULL
 * buffer with a non-empty frame (nothing enqueued); a failed event, copy or
 * launch call is GI_ECUDA.  B, H, W from f (k unused).  Caller owns every
 * buffer; no alignment needed.
 *
 * gi_target_from_rgb8: on `stream`, wait for wait_event, then expand
 * rgb (device u8 [B][H][W][3], interleaved as a decoder returns it) into
 * target (device fp32 [B][3][H][W], planar: the layout every fit / loss entry
 * point reads), target = u / 255 (IEEE fp32 division, round to nearest), then
 * record done_event (rgb may be overwritten after it).  One kernel. */
gi_status gi_target_from_rgb8(const uint8_t* rgb, const gi_frame* f, float* target,
                              void* wait_event, void* done_event, void* stream);

/* gi_target_upload_rgb8: on `stream`, wait for wait_event (e.g. the previous
 * expansion's done_event: dev_rgb is free), copy host_rgb (host u8
 * [B][H][W][3]; pinned for an asynchronous copy) to dev_rgb (device, same
 * size), record ready_event.  One copy, no kernel. */
gi_status gi_target_upload_rgb8(const uint8_t* host_rgb, uint8_t* dev_rgb, const gi_frame* f,
                                void* wait_event, void* ready_event, void* stream);

/* --- harness helpers (not on the hot path) ---------------------------------
 * PSNR of each image on [0,1]-clamped values, capped at 100 dB:
 * psnr[B] fp32 out; ws of gi_psnr_workspace_bytes() bytes (device). */
size_t gi_psnr_workspace_bytes(const gi_frame* f);
gi_status gi_psnr(const float* image, const float* target, const gi_frame* f, float* psnr,
                  void* ws, void* stream);

/* Number of kernels this thread has launched (or captured into a graph)
 * through libgi since load.  Diagnostic; the bench reports it. */
int64_t gi_launch_count(void);

/* Synchronise `stream` and translate the device status words:
 * n_keys (device u32, may be NULL) > key_capacity -> GI_ECAPACITY;
 * status_flags (device u32, may be NULL) bit 0 -> GI_ENONFINITE. */
gi_status gi_check(const uint32_t* n_keys, int64_t key_capacity, const uint32_t* status_flags,
                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GI_H */
