// C ABI of libgi (include/gi.h): argument validation, workspace carving and
// dispatch to the sm_100a kernels.  Host-side only; no allocation, no sync
// except in gi_check.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "codec_core.cuh"
#include "gi_internal.cuh"
#include <nvtx3/nvToolsExt.h>

// NVTX range around every compute entry point (SURVEY §5 tracing): a no-op
// unless a tool (nsys, ncu --nvtx) is attached.
namespace {
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace
#define GI_NVTX(name) const NvtxRange gi_nvtx_range_(name)

namespace gi {
namespace {
thread_local int64_t g_launches = 0;
}
void note_launches(int k) { g_launches += k; }
bool use_pdl() {
    static const bool on = [] {
        const char* e = std::getenv("GI_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}
int64_t g_launches_get() { return g_launches; }
}  // namespace gi

namespace {

thread_local char g_err[512] = "";

gi_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return GI_OK;
    std::snprintf(g_err, sizeof(g_err), "%s: %s (%s)", where, cudaGetErrorName(e),
                  cudaGetErrorString(e));
    return GI_ECUDA;
}

gi_status invalid(const char* msg) {
    std::snprintf(g_err, sizeof(g_err), "invalid argument: %s", msg);
    return GI_EINVAL;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

gi_status check_frame(const gi_frame* f) {
    if (!f) return invalid("frame is NULL");
    if (f->width < 1 || f->height < 1 || f->width > 32767 || f->height > 32767)
        return invalid("width/height must be in [1, 32767]");
    if (f->tile != gi::kTile) return invalid("tile must be 16");
    if (f->batch < 1) return invalid("batch must be >= 1");
    if (!(f->k > 0.0f) || !std::isfinite(f->k)) return invalid("k must be finite and > 0");
    const int64_t tt = (int64_t)gi::tiles_x(f->width) * gi::tiles_y(f->height) * f->batch;
    if (tt >= (1LL << 30)) return invalid("too many tiles");
    return GI_OK;
}

gi_status check_n(int32_t n, const gi_frame* f) {
    if (n < 0) return invalid("n must be >= 0");
    if ((int64_t)n * f->batch >= (1LL << 30)) return invalid("batch * n too large");
    return GI_OK;
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

struct FitWs {
    gi::Proj* proj;
    uint32_t* touched;
    uint32_t* key_tile;
    uint32_t* key_gid;
    uint32_t* tile_range;
    uint32_t* n_keys;
    void* bin_ws;
    void* bwd_ws;
    size_t bytes;
};

FitWs carve_fit(void* base, int32_t n, int64_t cap, const gi_frame& f) {
    using gi::align_up;
    const size_t total = (size_t)n * f.batch;
    const size_t T = (size_t)gi::tiles_x(f.width) * gi::tiles_y(f.height) * f.batch;
    char* p = static_cast<char*>(base);
    FitWs w;
    size_t off = 0;
    w.proj = reinterpret_cast<gi::Proj*>(p + off); off += align_up(sizeof(gi::Proj) * total);
    w.touched = reinterpret_cast<uint32_t*>(p + off); off += align_up(4 * total);
    w.key_tile = reinterpret_cast<uint32_t*>(p + off); off += align_up(4 * (size_t)cap);
    // key_gid doubles as the direct-binning slab array (>= cap words)
    const size_t kg = std::max((size_t)cap, gi::slab_words(cap, f));
    w.key_gid = reinterpret_cast<uint32_t*>(p + off); off += align_up(4 * kg);
    w.tile_range = reinterpret_cast<uint32_t*>(p + off); off += align_up(4 * (T + 1));
    w.n_keys = reinterpret_cast<uint32_t*>(p + off); off += align_up(4);
    w.bin_ws = p + off; off += align_up(gi::bin_ws_bytes(n, cap, f));
    w.bwd_ws = p + off; off += align_up(gi::backward_ws_bytes(n, cap, f));
    w.bytes = off;
    return w;
}

}  // namespace

extern "C" {

const char* gi_status_string(gi_status s) {
    switch (s) {
        case GI_OK: return "GI_OK";
        case GI_EINVAL: return "GI_EINVAL";
        case GI_ECUDA: return "GI_ECUDA";
        case GI_ECAPACITY: return "GI_ECAPACITY";
        case GI_EFORMAT: return "GI_EFORMAT";
        case GI_ENONFINITE: return "GI_ENONFINITE";
    }
    return "GI_UNKNOWN";
}

const char* gi_last_error(void) { return g_err; }

int32_t gi_abi_version(void) { return GI_ABI_VERSION; }

int32_t gi_num_tiles(const gi_frame* f) {
    if (check_frame(f) != GI_OK) return -1;
    return gi::tiles_x(f->width) * gi::tiles_y(f->height);
}

size_t gi_proj_bytes(int32_t n, const gi_frame* f) {
    if (check_frame(f) != GI_OK || n < 0) return 0;
    return (size_t)n * f->batch * GI_PROJ_BYTES;
}

gi_status gi_project(const float* params, int32_t n, const gi_frame* f, uint32_t flags, void* proj,
                     uint32_t* tiles_touched, void* stream) {
    GI_NVTX("gi_project");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK || (st = check_n(n, f)) != GI_OK) return st;
    if (!gi::flags_valid(flags)) return invalid("flags");
    if (n > 0 && (!params || !proj || !tiles_touched)) return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(proj)) return invalid("params/proj must be 16-B aligned");
    if (n == 0) return GI_OK;
    return cuda_status(gi::launch_project(params, n, *f, flags, static_cast<gi::Proj*>(proj),
                                          tiles_touched, gi::ProjectFuse{nullptr, gi::BinCounts{}},
                                          S(stream)),
                       "gi_project");
}

size_t gi_bin_workspace_bytes(int32_t n, int64_t key_capacity, const gi_frame* f) {
    if (check_frame(f) != GI_OK || n < 0 || key_capacity < 0) return 0;
    return gi::bin_ws_bytes(n, key_capacity, *f);
}

gi_status gi_bin(const void* proj, const uint32_t* tiles_touched, int32_t n, const gi_frame* f,
                 int64_t key_capacity, void* ws, size_t ws_bytes, uint32_t* key_tile,
                 uint32_t* key_gid, uint32_t* tile_range, uint32_t* n_keys, void* stream) {
    GI_NVTX("gi_bin");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK || (st = check_n(n, f)) != GI_OK) return st;
    if (key_capacity < 0 || key_capacity >= (1LL << 31)) return invalid("key_capacity");
    if (ws_bytes < gi::bin_ws_bytes(n, key_capacity, *f)) return invalid("bin workspace too small");
    if (!tile_range || !n_keys || (key_capacity > 0 && (!key_tile || !key_gid)) ||
        (n > 0 && (!proj || !tiles_touched)) || !ws)
        return invalid("NULL buffer");
    return cuda_status(gi::launch_bin(static_cast<const gi::Proj*>(proj), tiles_touched, n, *f,
                                      key_capacity, ws, key_tile, key_gid, tile_range, n_keys,
                                      S(stream)),
                       "gi_bin");
}

gi_status gi_render(const void* proj, const uint32_t* key_gid, const uint32_t* tile_range,
                    int32_t n, const gi_frame* f, float* image, void* stream) {
    GI_NVTX("gi_render");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK || (st = check_n(n, f)) != GI_OK) return st;
    if (!tile_range || !image || (n > 0 && (!proj || !key_gid))) return invalid("NULL buffer");
    // gi_bin output is already in gid order: presorted, key_gid only read
    return cuda_status(gi::launch_render(static_cast<const gi::Proj*>(proj),
                                         const_cast<uint32_t*>(key_gid), tile_range, n, *f, true,
                                         image, gi::ChainState{}, S(stream)),
                       "gi_render");
}

size_t gi_backward_workspace_bytes(int32_t n, int64_t key_capacity, const gi_frame* f) {
    if (check_frame(f) != GI_OK || n < 0 || key_capacity < 0) return 0;
    return gi::backward_ws_bytes(n, key_capacity, *f);
}

gi_status gi_render_backward(const float* params, const void* proj, const uint32_t* key_gid,
                             const uint32_t* tile_range, int32_t n, const gi_frame* f,
                             uint32_t flags, const float* dL_dimage, const float* target,
                             int64_t key_capacity, void* ws, size_t ws_bytes, float* grads,
                             float* loss, float* image_out, void* stream) {
    GI_NVTX("gi_render_backward");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK || (st = check_n(n, f)) != GI_OK) return st;
    if (!gi::flags_valid(flags)) return invalid("flags");
    if (key_capacity < 0 || key_capacity >= (1LL << 31)) return invalid("key_capacity");
    if (ws_bytes < gi::backward_ws_bytes(n, key_capacity, *f)) return invalid("backward workspace too small");
    if (!dL_dimage && !target) return invalid("need dL_dimage or target");
    if (!tile_range || !ws || (n > 0 && (!params || !proj || !key_gid || !grads)))
        return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(grads) || !aligned16(ws)) return invalid("alignment");
    return cuda_status(gi::launch_backward(params, static_cast<const gi::Proj*>(proj), key_gid,
                                           tile_range, n, *f, flags, dL_dimage, target,
                                           key_capacity, ws, grads, loss, image_out, S(stream)),
                       "gi_render_backward");
}

gi_status gi_adam_step(float* params, const float* grads, float* m, float* v, int64_t count,
                       int32_t step, float lr, float beta1, float beta2, float eps,
                       uint32_t* nonfinite_flag, void* stream) {
    GI_NVTX("gi_adam_step");
    if (count < 0) return invalid("count");
    if (step < 1) return invalid("step is 1-based");
    if (!(beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f)) return invalid("betas");
    if (count > 0 && (!params || !grads || !m || !v)) return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(grads) || !aligned16(m) || !aligned16(v))
        return invalid("alignment");
    if (count == 0) return GI_OK;
    return cuda_status(gi::launch_adam(params, grads, m, v, count, step, nullptr, lr, 1, beta1,
                                       beta2, eps, nonfinite_flag, S(stream)),
                       "gi_adam_step");
}

// --- NEXT-4 peer exchange ------------------------------------------------
gi_status gi_peer_alloc(size_t bytes, void** ptr, void* handle) {
    if (!ptr || !handle || bytes == 0) return invalid("NULL argument or zero size");
    *ptr = nullptr;
    cudaError_t e = cudaMalloc(ptr, bytes);
    if (e != cudaSuccess) return cuda_status(e, "gi_peer_alloc");
    if ((e = cudaMemset(*ptr, 0, bytes)) != cudaSuccess) return cuda_status(e, "gi_peer_alloc");
    cudaIpcMemHandle_t h;
    if ((e = cudaIpcGetMemHandle(&h, *ptr)) != cudaSuccess) return cuda_status(e, "gi_peer_alloc");
    std::memcpy(handle, &h, sizeof(h));
    return GI_OK;
}

gi_status gi_peer_free(void* ptr) { return cuda_status(cudaFree(ptr), "gi_peer_free"); }

gi_status gi_peer_open(const void* handle, void** ptr) {
    if (!ptr || !handle) return invalid("NULL argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    return cuda_status(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "gi_peer_open");
}

gi_status gi_peer_close(void* ptr) { return cuda_status(cudaIpcCloseMemHandle(ptr), "gi_peer_close"); }

gi_status gi_peer_adam_step(float* params, float* m, float* v, const float* const* grads,
                            int32_t G, int64_t count, int32_t step, float lr, float beta1,
                            float beta2, float eps, int32_t n_loss, float* loss_out,
                            uint32_t* nonfinite_flag, void* stream) {
    GI_NVTX("gi_peer_adam_step");
    if (count < 0) return invalid("count");
    if (G < 1 || G > gi::kMaxPeers) return invalid("G must be 1..8");
    if (n_loss < 0 || n_loss > 32) return invalid("n_loss must be 0..32");
    if (step < 1) return invalid("step is 1-based");
    if (!(beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f)) return invalid("betas");
    if (!grads) return invalid("NULL buffer");
    for (int r = 0; r < G; ++r)
        if (!grads[r] || !aligned16(grads[r])) return invalid("grads[r] NULL or unaligned");
    if (count > 0 && (!params || !m || !v)) return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(m) || !aligned16(v)) return invalid("alignment");
    return cuda_status(gi::launch_peer_adam(params, m, v, grads, G, count, step, lr, beta1, beta2,
                                            eps, n_loss, loss_out, nonfinite_flag, S(stream)),
                       "gi_peer_adam_step");
}

gi_status gi_adan_step(float* params, const float* grads, float* m, float* v, float* n,
                       float* grad_prev, int64_t count, int32_t step, float lr, float beta1,
                       float beta2, float beta3, float eps, float weight_decay,
                       uint32_t* nonfinite_flag, void* stream) {
    GI_NVTX("gi_adan_step");
    if (count < 0 || count % 8 != 0) return invalid("count must be a multiple of 8");
    if (step < 1) return invalid("step is 1-based");
    if (!(beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f && beta3 >= 0.f && beta3 < 1.f))
        return invalid("betas");
    if (count > 0 && (!params || !grads || !m || !v || !n || !grad_prev)) return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(grads) || !aligned16(m) || !aligned16(v) || !aligned16(n) ||
        !aligned16(grad_prev))
        return invalid("alignment");
    return cuda_status(gi::launch_adan(params, grads, m, v, n, grad_prev, count, step, nullptr, lr, 1,
                                       beta1, beta2, beta3, eps, weight_decay, nonfinite_flag,
                                       S(stream)),
                       "gi_adan_step");
}

double gi_lr_at(int32_t step, double lr0, int32_t half_every) {
    if (step < 1 || half_every < 1) return 0.0;
    return std::ldexp(lr0, -((step - 1) / half_every));
}

size_t gi_fit_workspace_bytes(int32_t n, int64_t key_capacity, const gi_frame* f) {
    if (check_frame(f) != GI_OK || n < 0 || key_capacity < 0) return 0;
    return carve_fit(nullptr, n, key_capacity, *f).bytes;
}

const uint32_t* gi_fit_n_keys(const void* fit_ws, int32_t n, int64_t key_capacity, const gi_frame* f) {
    if (check_frame(f) != GI_OK || !fit_ws) return nullptr;
    return carve_fit(const_cast<void*>(fit_ws), n, key_capacity, *f).n_keys;
}

gi_status gi_fit_bin_view(const void* fit_ws, int32_t n, int64_t key_capacity, const gi_frame* f,
                          const uint32_t** tile_count, uint32_t* count_stride,
                          const uint32_t** slab, uint32_t* slab_capacity) {
    gi_status st;
    if ((st = check_frame(f)) != GI_OK || (st = check_n(n, f)) != GI_OK) return st;
    if (!fit_ws || key_capacity < 0 || !tile_count || !count_stride || !slab || !slab_capacity)
        return invalid("NULL argument");
    FitWs w = carve_fit(const_cast<void*>(fit_ws), n, key_capacity, *f);
    const gi::BinCounts bc =
        gi::bin_counts_direct(w.bin_ws, n, key_capacity, *f, w.key_gid, nullptr);
    *tile_count = bc.tile_count;
    *count_stride = gi::count_stride_for((int64_t)gi::tiles_x(f->width) * gi::tiles_y(f->height) *
                                         f->batch);   // the fit paths' layout
    *slab = w.key_gid;
    *slab_capacity = gi::slab_capacity(key_capacity, *f);
    return GI_OK;
}

uint32_t* gi_fit_seg_stats(void* fit_ws, int32_t n, int64_t key_capacity, const gi_frame* f) {
    if (check_frame(f) != GI_OK || !fit_ws || n < 0 || key_capacity < 0) return nullptr;
    FitWs w = carve_fit(fit_ws, n, key_capacity, *f);
    return gi::bin_seg_stats(w.bin_ws, n, key_capacity, *f);
}

static cudaError_t record_stage(void* const* ev, int i, cudaStream_t s) {
    if (ev == nullptr || ev[i] == nullptr) return cudaSuccess;
    // external: becomes an event-record node when the stream is being captured
    return cudaEventRecordWithFlags(static_cast<cudaEvent_t>(ev[i]), s, cudaEventRecordExternal);
}

// Adan state of a fused Adan fit step (NEXT-1); null for Adam.
struct AdanOpt {
    float* n;
    float* grad_prev;
    float beta3, weight_decay;
};

static gi_status fit_step_impl(float* params, float* grads, float* m, float* v, const float* target,
                               int32_t n, const gi_frame* f, uint32_t flags, int64_t key_capacity,
                               void* fit_ws, size_t ws_bytes, uint32_t* step_counter, float lr0,
                               int32_t half_every, float beta1, float beta2, float eps, float* loss,
                               uint32_t* status_flags, void* const* stage_events, void* stream,
                               bool chained, const AdanOpt* adan = nullptr) {
    gi_status st;
    if ((st = check_frame(f)) != GI_OK || (st = check_n(n, f)) != GI_OK) return st;
    if (!gi::flags_valid(flags)) return invalid("flags");
    if (key_capacity < 0 || key_capacity >= (1LL << 31)) return invalid("key_capacity");
    if (half_every < 1) return invalid("half_every");
    if (!(beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f)) return invalid("betas");
    if (!fit_ws || ws_bytes < carve_fit(nullptr, n, key_capacity, *f).bytes)
        return invalid("fit workspace too small");
    if (!step_counter || !target || (n > 0 && (!params || !grads || !m || !v)))
        return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(grads) || !aligned16(m) || !aligned16(v) || !aligned16(fit_ws))
        return invalid("alignment");
    if (adan != nullptr) {
        if (!(adan->beta3 >= 0.f && adan->beta3 < 1.f)) return invalid("betas");
        if (n > 0 && (!adan->n || !adan->grad_prev)) return invalid("NULL buffer");
        if (!aligned16(adan->n) || !aligned16(adan->grad_prev)) return invalid("alignment");
    }
    FitWs w = carve_fit(fit_ws, n, key_capacity, *f);
    cudaStream_t s = S(stream);
    cudaError_t e;
#define GI_TRY(expr, where) \
    if ((e = (expr)) != cudaSuccess) return cuda_status(e, where)
    // Direct binning: the producer (project, or the previous step's finalize
    // when chained) counts every key with a rank-returning atomic and writes it
    // to its tile's slab of the key array; the per-tile counters are zero on
    // entry (zero-filled workspace, then left zeroed by the consumer tile
    // kernel of each call).
    uint32_t* gauss_off = gi::backward_gauss_off(w.bwd_ws, n, key_capacity, *f);
    const gi::BinCounts bc = gi::bin_counts_direct(w.bin_ws, n, key_capacity, *f, w.key_gid, gauss_off);
    gi::ChainState cs = gi::bin_chain_direct(w.bin_ws, n, key_capacity, *f, w.key_gid, gauss_off,
                                             w.n_keys, chained ? step_counter : nullptr);
    float* consts = gi::backward_adam_consts(w.bwd_ws, n, key_capacity, *f);
    cs.adam_consts = consts;          // {lr_t, 1/(1 - b1^t), 1/(1 - b2^t)} from the tile kernel
    cs.step_read = step_counter;
    cs.lr0 = lr0;
    cs.half_every = half_every;
    cs.b1 = beta1;
    cs.b2 = beta2;
    if (adan != nullptr) {
        cs.adan = 1;
        cs.b3 = adan->beta3;
        cs.wd = adan->weight_decay;
    }
    GI_TRY(record_stage(stage_events, 0, s), "gi_fit_step/event");
    if (!chained)   // the workspace may hold a chained step's pending keys: start from zero
        GI_TRY(gi::bin_clear(w.bin_ws, n, key_capacity, *f, s), "gi_fit_step/clear");
    if (!chained)
        GI_TRY(gi::launch_project(params, n, *f, flags, w.proj, w.touched,
                                  gi::ProjectFuse{step_counter, bc}, s),
               "gi_fit_step/project");
    GI_TRY(record_stage(stage_events, 1, s), "gi_fit_step/event");
    GI_TRY(record_stage(stage_events, 2, s), "gi_fit_step/event");
    GI_TRY(gi::launch_backward_tiles(w.proj, w.key_gid, nullptr, n, *f, false, nullptr, target,
                                     key_capacity, w.bwd_ws, nullptr, cs, s),
           "gi_fit_step/backward");
    GI_TRY(record_stage(stage_events, 3, s), "gi_fit_step/event");
    gi::FusedAdam fa{};
    fa.params = params;
    fa.m = m;
    fa.v = v;
    fa.consts = consts;
    fa.b1 = beta1;
    fa.b2 = beta2;
    fa.eps = eps;
    fa.flag = status_flags;
    if (adan != nullptr) {
        fa.n = adan->n;
        fa.gprev = adan->grad_prev;
        fa.b3 = adan->beta3;
    }
    fa.proj_out = chained ? w.proj : nullptr;
    fa.touched_out = w.touched;
    fa.counts = bc;
    fa.k = f->k;
    fa.pos_flags = flags;
    GI_TRY(gi::launch_backward_finalize(params, w.proj, n, *f, flags, true, key_capacity, w.bwd_ws,
                                        grads, loss, &fa, s),
           "gi_fit_step/finalize+adam");
    GI_TRY(record_stage(stage_events, 4, s), "gi_fit_step/event");
    GI_TRY(record_stage(stage_events, 5, s), "gi_fit_step/event");
#undef GI_TRY
    return GI_OK;
}

gi_status gi_fit_grads(const float* params, float* grads, const float* target, int32_t n,
                       const gi_frame* f, uint32_t flags, int32_t tile_row0, int32_t tile_rows,
                       int64_t key_capacity, void* fit_ws, size_t ws_bytes, float* loss,
                       void* stream) {
    GI_NVTX("gi_fit_grads");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK || (st = check_n(n, f)) != GI_OK) return st;
    if (!gi::flags_valid(flags)) return invalid("flags");
    if (key_capacity < 0 || key_capacity >= (1LL << 31)) return invalid("key_capacity");
    const int TY = gi::tiles_y(f->height);
    if (tile_rows < 0) {
        tile_row0 = 0;
        tile_rows = TY;
    }
    if (tile_row0 < 0 || tile_row0 + tile_rows > TY) return invalid("tile window");
    if (!fit_ws || ws_bytes < carve_fit(nullptr, n, key_capacity, *f).bytes)
        return invalid("fit workspace too small");
    if (!target || (n > 0 && (!params || !grads))) return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(grads) || !aligned16(fit_ws)) return invalid("alignment");
    FitWs w = carve_fit(fit_ws, n, key_capacity, *f);
    cudaStream_t s = S(stream);
    cudaError_t e;
#define GI_TRY(expr, where) \
    if ((e = (expr)) != cudaSuccess) return cuda_status(e, where)
    if (tile_rows == 0) {             // empty window: this rank contributes nothing
        if (n > 0)
            GI_TRY(cudaMemsetAsync(grads, 0, sizeof(float) * 8 * (size_t)n * f->batch, s),
                   "gi_fit_grads/zero");
        if (loss) GI_TRY(cudaMemsetAsync(loss, 0, sizeof(float) * f->batch, s), "gi_fit_grads/zero");
        return GI_OK;
    }
    const int r0 = tile_row0, r1 = tile_row0 + tile_rows;
    GI_TRY(gi::bin_clear(w.bin_ws, n, key_capacity, *f, s), "gi_fit_grads/clear");
    uint32_t* gauss_off = gi::backward_gauss_off(w.bwd_ws, n, key_capacity, *f);
    gi::BinCounts bc = gi::bin_counts_direct(w.bin_ws, n, key_capacity, *f, w.key_gid, gauss_off);
    bc.row0 = r0;
    bc.row1 = r1;
    gi::ChainState cs = gi::bin_chain_direct(w.bin_ws, n, key_capacity, *f, w.key_gid, gauss_off,
                                             w.n_keys, nullptr);
    cs.row0 = r0;
    cs.row1 = r1;
    GI_TRY(gi::launch_project(params, n, *f, flags, w.proj, w.touched, gi::ProjectFuse{nullptr, bc},
                              s),
           "gi_fit_grads/project");
    if (tile_rows > 0)
        GI_TRY(gi::launch_backward_tiles(w.proj, w.key_gid, nullptr, n, *f, false, nullptr, target,
                                         key_capacity, w.bwd_ws, nullptr, cs, s),
               "gi_fit_grads/backward");
    GI_TRY(gi::launch_backward_finalize(params, w.proj, n, *f, flags, true, key_capacity, w.bwd_ws,
                                        grads, loss, nullptr, s, r0, r1),
           "gi_fit_grads/finalize");
#undef GI_TRY
    return GI_OK;
}

gi_status gi_fit_step(float* params, float* grads, float* m, float* v, const float* target,
                      int32_t n, const gi_frame* f, uint32_t flags, int64_t key_capacity,
                      void* fit_ws, size_t ws_bytes, uint32_t* step_counter, float lr0,
                      int32_t half_every, float beta1, float beta2, float eps, float* loss,
                      uint32_t* status_flags, void* const* stage_events, void* stream) {
    GI_NVTX("gi_fit_step");
    return fit_step_impl(params, grads, m, v, target, n, f, flags, key_capacity, fit_ws, ws_bytes,
                         step_counter, lr0, half_every, beta1, beta2, eps, loss, status_flags,
                         stage_events, stream, false);
}

gi_status gi_fit_step_adan(float* params, float* grads, float* m, float* v, float* n,
                           float* grad_prev, const float* target, int32_t n_gauss, const gi_frame* f,
                           uint32_t flags, int64_t key_capacity, void* fit_ws, size_t ws_bytes,
                           uint32_t* step_counter, float lr0, int32_t half_every, float beta1,
                           float beta2, float beta3, float eps, float weight_decay, float* loss,
                           uint32_t* status_flags, void* stream) {
    GI_NVTX("gi_fit_step_adan");
    const AdanOpt opt{n, grad_prev, beta3, weight_decay};
    return fit_step_impl(params, grads, m, v, target, n_gauss, f, flags, key_capacity, fit_ws,
                         ws_bytes, step_counter, lr0, half_every, beta1, beta2, eps, loss,
                         status_flags, nullptr, stream, false, &opt);
}

gi_status gi_fit_step_adan_chained(float* params, float* grads, float* m, float* v, float* n,
                                   float* grad_prev, const float* target, int32_t n_gauss,
                                   const gi_frame* f, uint32_t flags, int64_t key_capacity,
                                   void* fit_ws, size_t ws_bytes, uint32_t* step_counter, float lr0,
                                   int32_t half_every, float beta1, float beta2, float beta3,
                                   float eps, float weight_decay, float* loss,
                                   uint32_t* status_flags, void* stream) {
    GI_NVTX("gi_fit_step_adan_chained");
    const AdanOpt opt{n, grad_prev, beta3, weight_decay};
    return fit_step_impl(params, grads, m, v, target, n_gauss, f, flags, key_capacity, fit_ws,
                         ws_bytes, step_counter, lr0, half_every, beta1, beta2, eps, loss,
                         status_flags, nullptr, stream, true, &opt);
}

gi_status gi_fit_prime(const float* params, int32_t n, const gi_frame* f, uint32_t flags,
                       int64_t key_capacity, void* fit_ws, size_t ws_bytes, void* stream) {
    GI_NVTX("gi_fit_prime");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK || (st = check_n(n, f)) != GI_OK) return st;
    if (!gi::flags_valid(flags)) return invalid("flags");
    if (key_capacity < 0 || key_capacity >= (1LL << 31)) return invalid("key_capacity");
    if (!fit_ws || ws_bytes < carve_fit(nullptr, n, key_capacity, *f).bytes)
        return invalid("fit workspace too small");
    if (n > 0 && !params) return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(fit_ws)) return invalid("alignment");
    FitWs w = carve_fit(fit_ws, n, key_capacity, *f);
    uint32_t* gauss_off = gi::backward_gauss_off(w.bwd_ws, n, key_capacity, *f);
    // a workspace left by a chained step already holds the next step's keys
    // (per-tile counts, slab entries, allocation counter): start from zero
    cudaError_t e = gi::bin_clear(w.bin_ws, n, key_capacity, *f, S(stream));
    if (e != cudaSuccess) return cuda_status(e, "gi_fit_prime/clear");
    return cuda_status(
        gi::launch_project(params, n, *f, flags, w.proj, w.touched,
                           gi::ProjectFuse{nullptr, gi::bin_counts_direct(w.bin_ws, n, key_capacity,
                                                                          *f, w.key_gid, gauss_off)},
                           S(stream)),
        "gi_fit_prime");
}

gi_status gi_fit_reset(int32_t n, const gi_frame* f, int64_t key_capacity, void* fit_ws,
                       size_t ws_bytes, void* stream) {
    GI_NVTX("gi_fit_reset");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK || (st = check_n(n, f)) != GI_OK) return st;
    if (key_capacity < 0 || key_capacity >= (1LL << 31)) return invalid("key_capacity");
    if (!fit_ws || ws_bytes < carve_fit(nullptr, n, key_capacity, *f).bytes)
        return invalid("fit workspace too small");
    if (!aligned16(fit_ws)) return invalid("alignment");
    FitWs w = carve_fit(fit_ws, n, key_capacity, *f);
    return cuda_status(gi::bin_clear(w.bin_ws, n, key_capacity, *f, S(stream)), "gi_fit_reset");
}

gi_status gi_fit_step_chained(float* params, float* grads, float* m, float* v, const float* target,
                              int32_t n, const gi_frame* f, uint32_t flags, int64_t key_capacity,
                              void* fit_ws, size_t ws_bytes, uint32_t* step_counter, float lr0,
                              int32_t half_every, float beta1, float beta2, float eps, float* loss,
                              uint32_t* status_flags, void* const* stage_events, void* stream) {
    GI_NVTX("gi_fit_step_chained");
    return fit_step_impl(params, grads, m, v, target, n, f, flags, key_capacity, fit_ws, ws_bytes,
                         step_counter, lr0, half_every, beta1, beta2, eps, loss, status_flags,
                         stage_events, stream, true);
}

int64_t gi_launch_count(void) { return gi::g_launches_get(); }

gi_status gi_render_frame(const float* params, int32_t n, const gi_frame* f, uint32_t flags,
                          int64_t key_capacity, void* frame_ws, size_t ws_bytes, float* image,
                          void* stream) {
    GI_NVTX("gi_render_frame");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK || (st = check_n(n, f)) != GI_OK) return st;
    if (!gi::flags_valid(flags)) return invalid("flags");
    if (key_capacity < 0 || key_capacity >= (1LL << 31)) return invalid("key_capacity");
    if (!frame_ws || ws_bytes < carve_fit(nullptr, n, key_capacity, *f).bytes)
        return invalid("frame workspace too small");
    if (!image || (n > 0 && !params)) return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(frame_ws)) return invalid("alignment");
    FitWs w = carve_fit(frame_ws, n, key_capacity, *f);
    cudaStream_t s = S(stream);
    cudaError_t e;
#define GI_TRY(expr, where) \
    if ((e = (expr)) != cudaSuccess) return cuda_status(e, where)
    const gi::ChainState cs = gi::bin_chain_direct(w.bin_ws, n, key_capacity, *f, w.key_gid, nullptr,
                                                   w.n_keys, nullptr, true);
    GI_TRY(gi::launch_project(params, n, *f, flags, w.proj, w.touched,
                              gi::ProjectFuse{nullptr, gi::bin_counts_direct(w.bin_ws, n, key_capacity,
                                                                             *f, w.key_gid, nullptr,
                                                                             true)},
                              s),
           "gi_render_frame/project");
    GI_TRY(gi::launch_render(w.proj, w.key_gid, nullptr, n, *f, false, image, cs, s),
           "gi_render_frame/render");
#undef GI_TRY
    return GI_OK;
}

gi_status gi_vq_decode(const uint8_t* payload, size_t payload_bytes, const gi_codec_meta* meta,
                       float* params, void* stream) {
    GI_NVTX("gi_vq_decode");
    if (!meta) return invalid("meta is NULL");
    if (meta->n < 0) return invalid("n");
    if (meta->bits < 1 || meta->bits > 16 || meta->stages < 1 || meta->stages > 8 ||
        meta->codebook < 2 || meta->codebook > 256) {
        std::snprintf(g_err, sizeof(g_err), "codec metadata out of range");
        return GI_EFORMAT;
    }
    int ib = 1;
    while ((1 << ib) < meta->codebook) ++ib;
    const int64_t rec = 32 + 3LL * meta->bits + (int64_t)meta->stages * ib;
    if (rec > 64) {
        std::snprintf(g_err, sizeof(g_err), "record wider than 64 bits");
        return GI_EFORMAT;
    }
    if ((size_t)((rec * meta->n + 7) / 8) > payload_bytes) {
        std::snprintf(g_err, sizeof(g_err), "payload shorter than n records");
        return GI_EFORMAT;
    }
    if (meta->n > 0 && (!payload || !params || !meta->codebooks)) return invalid("NULL buffer");
    if (!aligned16(params)) return invalid("alignment");
    return cuda_status(gi::launch_vq_decode(payload, *meta, params, S(stream)), "gi_vq_decode");
}

// Shared gi_codec_meta checks of the decode entry points; rec_out = bits per record.
static gi_status check_codec(const gi_codec_meta* meta, size_t payload_bytes, int64_t* rec_out) {
    if (!meta) return invalid("meta is NULL");
    if (meta->n < 0) return invalid("n");
    if (meta->bits < 1 || meta->bits > 16 || meta->stages < 1 || meta->stages > 8 ||
        meta->codebook < 2 || meta->codebook > 256) {
        std::snprintf(g_err, sizeof(g_err), "codec metadata out of range");
        return GI_EFORMAT;
    }
    int ib = 1;
    while ((1 << ib) < meta->codebook) ++ib;
    const int64_t rec = 32 + 3LL * meta->bits + (int64_t)meta->stages * ib;
    if (rec > 64) {
        std::snprintf(g_err, sizeof(g_err), "record wider than 64 bits");
        return GI_EFORMAT;
    }
    if ((size_t)((rec * meta->n + 7) / 8) > payload_bytes) {
        std::snprintf(g_err, sizeof(g_err), "payload shorter than n records");
        return GI_EFORMAT;
    }
    *rec_out = rec;
    return GI_OK;
}

gi_status gi_decode_render_frame(const uint8_t* payload, size_t payload_bytes,
                                 const gi_codec_meta* meta, const gi_frame* f,
                                 int64_t key_capacity, void* frame_ws, size_t ws_bytes,
                                 float* params, float* image, void* stream) {
    GI_NVTX("gi_decode_render_frame");
    gi_status st;
    int64_t rec = 0;
    if ((st = check_codec(meta, payload_bytes, &rec)) != GI_OK) return st;
    if ((st = check_frame(f)) != GI_OK) return st;
    if (f->batch != 1) return invalid("batch (one image per payload)");
    const int32_t n = meta->n;
    if ((st = check_n(n, f)) != GI_OK) return st;
    if (key_capacity < 0 || key_capacity >= (1LL << 31)) return invalid("key_capacity");
    if (!frame_ws || ws_bytes < carve_fit(nullptr, n, key_capacity, *f).bytes)
        return invalid("frame workspace too small");
    if (!image || (n > 0 && (!payload || !meta->codebooks))) return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(frame_ws)) return invalid("alignment");
    FitWs w = carve_fit(frame_ws, n, key_capacity, *f);
    cudaStream_t s = S(stream);
    cudaError_t e;
#define GI_TRY(expr, where) \
    if ((e = (expr)) != cudaSuccess) return cuda_status(e, where)
    const gi::ChainState cs = gi::bin_chain_direct(w.bin_ws, n, key_capacity, *f, w.key_gid, nullptr,
                                                   w.n_keys, nullptr, true);
    GI_TRY(gi::launch_decode_project(payload, *meta, params, *f, w.proj, w.touched,
                                     gi::ProjectFuse{nullptr, gi::bin_counts_direct(
                                                                  w.bin_ws, n, key_capacity, *f,
                                                                  w.key_gid, nullptr, true)},
                                     s),
           "gi_decode_render_frame/decode+project");
    GI_TRY(gi::launch_render(w.proj, w.key_gid, nullptr, n, *f, false, image, cs, s, true),
           "gi_decode_render_frame/render");
#undef GI_TRY
    return GI_OK;
}

gi_status gi_vq_encode(const float* params, uint32_t flags, const gi_codec_meta* meta,
                       uint8_t* payload, size_t payload_bytes, float* eff, void* stream) {
    GI_NVTX("gi_vq_encode");
    if (!meta) return invalid("meta is NULL");
    if (meta->n < 0) return invalid("n");
    if (!gi::flags_valid(flags) || (flags & GI_COV_RS)) return invalid("flags");
    if (meta->bits < 1 || meta->bits > 16 || meta->stages < 1 || meta->stages > 8 ||
        meta->codebook < 2 || meta->codebook > 256) {
        std::snprintf(g_err, sizeof(g_err), "codec metadata out of range");
        return GI_EFORMAT;
    }
    int ib = 1;
    while ((1 << ib) < meta->codebook) ++ib;
    const int64_t rec = 32 + 3LL * meta->bits + (int64_t)meta->stages * ib;
    if (rec > 64) {
        std::snprintf(g_err, sizeof(g_err), "record wider than 64 bits");
        return GI_EFORMAT;
    }
    size_t need = (size_t)((rec * meta->n + 7) / 8);
    if (rec % 8 != 0) need = (need + 3) & ~(size_t)3;   // whole words (see launch_vq_encode)
    if (payload && need > payload_bytes) {
        std::snprintf(g_err, sizeof(g_err), "payload buffer shorter than the packed records");
        return GI_EFORMAT;
    }
    if (meta->n > 0 && (!params || !meta->codebooks)) return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(eff)) return invalid("alignment");
    // records narrower than a byte multiple are OR-ed into 32-bit words from the base
    if (reinterpret_cast<uintptr_t>(payload) % 4 != 0) return invalid("payload alignment (4 B)");
    return cuda_status(gi::launch_vq_encode(params, !(flags & GI_POS_NORMALIZED), *meta, payload,
                                            eff, S(stream)),
                       "gi_vq_encode");
}

size_t gi_kmeans_workspace_bytes(int32_t B) {
    return (B < 2 || B > 256) ? 0 : (size_t)B * 4 * sizeof(unsigned long long);
}

gi_status gi_kmeans_step(const float* points, int32_t n, int32_t B, float* centroids,
                         uint32_t* assign, void* ws, size_t ws_bytes, void* stream) {
    GI_NVTX("gi_kmeans_step");
    if (n < 0) return invalid("n");
    if (B < 2 || B > 256) return invalid("B");
    if (!ws || ws_bytes < gi_kmeans_workspace_bytes(B)) return invalid("workspace too small");
    if (!centroids || (n > 0 && !points)) return invalid("NULL buffer");
    return cuda_status(gi::launch_kmeans_step(points, n, B, centroids, assign, ws, S(stream)),
                       "gi_kmeans_step");
}

static gi_status check_qat_cfg(const gi_qat_config* cfg) {
    if (!cfg) return invalid("cfg is NULL");
    if (cfg->bits < 1 || cfg->bits > 16 || cfg->stages < 1 || cfg->stages > 8 ||
        cfg->codebook < 2 || cfg->codebook > 256) {
        std::snprintf(g_err, sizeof(g_err), "codec metadata out of range");
        return GI_EFORMAT;
    }
    int ib = 1;
    while ((1 << ib) < cfg->codebook) ++ib;
    if (32 + 3 * cfg->bits + cfg->stages * ib > 64) {
        std::snprintf(g_err, sizeof(g_err), "record wider than 64 bits");
        return GI_EFORMAT;
    }
    if (!(cfg->decay >= 0.f && cfg->decay < 1.f) || !(cfg->beta1 >= 0.f && cfg->beta1 < 1.f) ||
        !(cfg->beta2 >= 0.f && cfg->beta2 < 1.f) || !(cfg->lr >= 0.f))
        return invalid("qat config");
    return GI_OK;
}

size_t gi_qat_workspace_bytes(int32_t n, int64_t key_capacity, const gi_frame* f,
                              const gi_qat_config* cfg) {
    if (check_frame(f) != GI_OK || n < 0 || key_capacity < 0 || check_qat_cfg(cfg) != GI_OK)
        return 0;
    return carve_fit(nullptr, n, key_capacity, *f).bytes +
           gi::align_up(8 * gi::qat_acc_words(cfg->stages, cfg->codebook)) + gi::align_up(16);
}

gi_status gi_qat_step(float* params, float* m, float* v, float* eff, float* grads, float* qparams,
                      float* qm, float* qv, float* books, float* ema_n, float* ema_s,
                      const float* target, int32_t n, const gi_frame* f, const gi_qat_config* cfg,
                      int64_t key_capacity, void* ws, size_t ws_bytes, uint32_t* step_counter,
                      float* losses, uint32_t* status_flags, void* stream) {
    GI_NVTX("gi_qat_step");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK || (st = check_n(n, f)) != GI_OK) return st;
    if (f->batch != 1) return invalid("gi_qat_step takes one image (batch 1)");
    if ((st = check_qat_cfg(cfg)) != GI_OK) return st;
    if (key_capacity < 0 || key_capacity >= (1LL << 31)) return invalid("key_capacity");
    if (!ws || ws_bytes < gi_qat_workspace_bytes(n, key_capacity, f, cfg))
        return invalid("qat workspace too small");
    if (!step_counter || !target || !losses || !qparams || !qm || !qv || !books || !ema_n ||
        !ema_s || (n > 0 && (!params || !m || !v || !eff || !grads)))
        return invalid("NULL buffer");
    if (!aligned16(params) || !aligned16(m) || !aligned16(v) || !aligned16(eff) ||
        !aligned16(grads) || !aligned16(ws))
        return invalid("alignment");
    FitWs w = carve_fit(ws, n, key_capacity, *f);
    char* extra = static_cast<char*>(ws) + w.bytes;
    void* acc = extra;
    float* consts = reinterpret_cast<float*>(extra + gi::align_up(8 * gi::qat_acc_words(cfg->stages,
                                                                                        cfg->codebook)));
    cudaStream_t s = S(stream);
    cudaError_t e;
#define GI_TRY(expr, where) \
    if ((e = (expr)) != cudaSuccess) return cuda_status(e, where)
    int ib = 1;
    while ((1 << ib) < cfg->codebook) ++ib;
    const gi::QuantParams qp{cfg->bits, cfg->stages, cfg->codebook, ib, {1.f, 1.f, 1.f},
                             {0.f, 0.f, 0.f}};
    GI_TRY(gi::launch_qat_quantize(params, n, qp, qparams, books, eff, acc, step_counter, consts,
                                   cfg->lr, cfg->beta1, cfg->beta2, s),
           "gi_qat_step/quantize");
    uint32_t* gauss_off = gi::backward_gauss_off(w.bwd_ws, n, key_capacity, *f);
    const gi::BinCounts bc = gi::bin_counts_direct(w.bin_ws, n, key_capacity, *f, w.key_gid, gauss_off);
    const gi::ChainState cs = gi::bin_chain_direct(w.bin_ws, n, key_capacity, *f, w.key_gid,
                                                   gauss_off, w.n_keys, nullptr);
    GI_TRY(gi::launch_project(eff, n, *f, GI_POS_NORMALIZED, w.proj, w.touched,
                              gi::ProjectFuse{nullptr, bc}, s),
           "gi_qat_step/project");
    GI_TRY(gi::launch_backward_tiles(w.proj, w.key_gid, nullptr, n, *f, false, nullptr, target,
                                     key_capacity, w.bwd_ws, nullptr, cs, s),
           "gi_qat_step/backward");
    GI_TRY(gi::launch_backward_finalize(eff, w.proj, n, *f, GI_POS_NORMALIZED, true, key_capacity,
                                        w.bwd_ws, grads, losses + 1, nullptr, s),
           "gi_qat_step/finalize");
    GI_TRY(gi::launch_qat_update(params, m, v, grads, n, cfg->bits, qparams, consts, cfg->beta1,
                                 cfg->beta2, cfg->eps, acc, cfg->stages, cfg->codebook,
                                 status_flags, s),
           "gi_qat_step/update");
    GI_TRY(gi::launch_qat_finish(qparams, qm, qv, books, ema_n, ema_s, acc, cfg->stages,
                                 cfg->codebook, n, consts, cfg->beta1, cfg->beta2, cfg->eps,
                                 cfg->decay, cfg->lambda, losses, s),
           "gi_qat_step/finish");
#undef GI_TRY
    return GI_OK;
}

static cudaError_t wait_on(void* ev, cudaStream_t s) {
    return ev == nullptr ? cudaSuccess : cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev), 0);
}
static cudaError_t record_on(void* ev, cudaStream_t s) {
    return ev == nullptr ? cudaSuccess : cudaEventRecord(static_cast<cudaEvent_t>(ev), s);
}

gi_status gi_target_from_rgb8(const uint8_t* rgb, const gi_frame* f, float* target,
                              void* wait_event, void* done_event, void* stream) {
    GI_NVTX("gi_target_from_rgb8");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK) return st;
    if ((int64_t)f->width * f->height * f->batch > 0 && (!rgb || !target)) return invalid("NULL buffer");
    cudaStream_t s = S(stream);
    cudaError_t e;
    if ((e = wait_on(wait_event, s)) != cudaSuccess) return cuda_status(e, "gi_target_from_rgb8/wait");
    if ((e = gi::launch_target_from_rgb8(rgb, *f, target, s)) != cudaSuccess)
        return cuda_status(e, "gi_target_from_rgb8");
    if ((e = record_on(done_event, s)) != cudaSuccess) return cuda_status(e, "gi_target_from_rgb8/record");
    return GI_OK;
}

gi_status gi_target_upload_rgb8(const uint8_t* host_rgb, uint8_t* dev_rgb, const gi_frame* f,
                                void* wait_event, void* ready_event, void* stream) {
    GI_NVTX("gi_target_upload_rgb8");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK) return st;
    const size_t bytes = (size_t)3 * f->width * f->height * f->batch;
    if (bytes > 0 && (!host_rgb || !dev_rgb)) return invalid("NULL buffer");
    cudaStream_t s = S(stream);
    cudaError_t e;
    if ((e = wait_on(wait_event, s)) != cudaSuccess) return cuda_status(e, "gi_target_upload_rgb8/wait");
    if (bytes > 0 &&
        (e = cudaMemcpyAsync(dev_rgb, host_rgb, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return cuda_status(e, "gi_target_upload_rgb8/copy");
    if ((e = record_on(ready_event, s)) != cudaSuccess) return cuda_status(e, "gi_target_upload_rgb8/record");
    return GI_OK;
}

gi_status gi_psnr(const float* image, const float* target, const gi_frame* f, float* psnr, void* ws,
                  void* stream) {
    GI_NVTX("gi_psnr");
    gi_status st;
    if ((st = check_frame(f)) != GI_OK) return st;
    if (!image || !target || !psnr || !ws) return invalid("NULL buffer");
    return cuda_status(gi::launch_psnr(image, target, *f, psnr, ws, S(stream)), "gi_psnr");
}

size_t gi_psnr_workspace_bytes(const gi_frame* f) {
    if (check_frame(f) != GI_OK) return 0;
    return (size_t)8 * 296 * f->batch;
}

gi_status gi_check(const uint32_t* n_keys, int64_t key_capacity, const uint32_t* status_flags,
                   void* stream) {
    GI_NVTX("gi_check");
    cudaError_t e = cudaStreamSynchronize(S(stream));
    if (e != cudaSuccess) return cuda_status(e, "gi_check/sync");
    if (status_flags) {
        uint32_t fl = 0;
        if ((e = cudaMemcpy(&fl, status_flags, 4, cudaMemcpyDeviceToHost)) != cudaSuccess)
            return cuda_status(e, "gi_check/flags");
        if (fl & 1u) return GI_ENONFINITE;
    }
    if (n_keys) {
        uint32_t k = 0;
        if ((e = cudaMemcpy(&k, n_keys, 4, cudaMemcpyDeviceToHost)) != cudaSuccess)
            return cuda_status(e, "gi_check/n_keys");
        if ((int64_t)k > key_capacity) return GI_ECAPACITY;
    }
    return GI_OK;
}

}  // extern "C"
