// a3 + a4 with Gaussian-parallel passes (chunks.cuh): the tile kernels the
// fused entry points (gi_render_frame, gi_fit_step*, gi_render_backward,
// gi_render) launch by default.  GI_TILE3=0 selects the round-1 kernels
// (pixel-parallel forward with per-warp candidate lists: render.cu,
// backward.cu) for A/B.
//
// One CTA of NT threads per 16x16 tile.  Per batch of <= NT staged records: plan work-balanced chunks of the records' in-tile boxes (one per
// lane), then
//   forward  (Eq. 7): each lane walks its chunk and adds
//            round(c' w 2^s) to its pixels' 32-bit fixed-point sums in shared
//            memory -- integer atomics, exact and order-independent;
//   residual g = 2 (C - T) / (3HW) (L2 loss) per pixel;
//   backward (App. A): the same chunks accumulate the 8 per-pair
//            sums of backward.cu's pass 2; a record's chunk sums are added in
//            a fixed order and written once to its partial slot.
// Every evaluated pair is in its Gaussian's box, and the forward no longer
// depends on the order of the tile's keys: a segment that fits one batch is
// staged straight from the direct-binning slab without the per-tile gid sort
// (longer segments are still sorted so that their batches are deterministic).
// Results are deterministic run to run and chained == plain bitwise.
#include <cstdlib>

#include "chunks.cuh"

namespace gi {
namespace {

constexpr double kSseScale3 = 1099511627776.0;   // 2^40, backward.cu's loss fixed point
constexpr int kSortMax3 = 1024;                  // sort buffer of multi-batch segments
// records per batch (256-thread CTAs): the fit kernel stages 128 (its shared
// memory then leaves room for the finalize CTAs that start in its tail, PDL:
// fit 23.9k -> 26.6k it/s vs 256; 112: -2 %), the render kernel 192 (one
// batch for the decoded C5 cloud's ~120-key tiles -- 128: decode -11 % --;
// C2 frame 57.8k -> 58.5k FPS vs 256)
#ifndef GI_TILE3_BATCH
#define GI_TILE3_BATCH 128
#endif
#ifndef GI_RENDER3_BATCH
#define GI_RENDER3_BATCH 192
#endif
constexpr int kBwdBatch = GI_TILE3_BATCH, kRenderBatch = GI_RENDER3_BATCH;

// a batch is NB <= NT records (one staged and planned record per thread)
template <int NT, int NB, bool kBwd>
struct FusedShared {
    StagedRecordsN<NB> sr;
    union {
        int acc[3][kTilePix];            // forward: fixed-point channel sums of the batch
        float4 red[kBwd ? NT : 1][2];    // backward: the 8 sums of each chunk
    } u;
    alignas(16) uint32_t sl[kSortMax3];
    float4 g[kBwd ? kTilePix : 1];       // per-pixel upstream dL/dC
    ChunkShared<NT> ch;
    uint32_t scratch[NT / 32];
    float sse[NT / 32];
    uint32_t cursor;
};

// The tile's key segment for the Gaussian-parallel kernels: a direct-binning
// segment of <= NT keys (one batch) is used in slab (atomic) order -- nothing in
// these kernels depends on the order within one batch; longer segments are
// brought into gid order (sorted_segment) or streamed past the slab.
template <int NT, int NB, bool kGidAhead, bool kFit>
__device__ __forceinline__ Seg open_segment3(const Proj* __restrict__ proj,
                                             uint32_t* __restrict__ key_gid,
                                             const uint32_t* __restrict__ tile_range,
                                             bool presorted, const ChainState& cs, int n, int T,
                                             const TileCtx& t, uint32_t* sl, uint32_t* scratch,
                                             uint32_t* cursor, uint32_t& gid0) {
    const int tt = t.img * T + t.tile;
    if (cs.slab != nullptr) {
        // written by the producer kernel (visible after griddepcontrol.wait);
        // re-zeroed by thread 0 only after the CTA's last barrier.  The slab's
        // first NB entries are read with the count, before it is known (the
        // slab holds >= 1,024 entries; entries past the count are ignored):
        // one memory round trip for both instead of two
        const uint32_t s = (uint32_t)tt * cs.slab_cap;
        // (the 256-thread fit kernel reads them after the count: at its 40-
        // register budget the early value costs a spill -- tile kernel 27.5
        // -> 29.3 us; render 55.3k -> 56.3k FPS, C3 fit 12.5k -> 12.8k it/s)
        if (kGidAhead && (int)threadIdx.x < NB && threadIdx.x < cs.slab_cap)   // inside the tile's slab
            gid0 = __ldcg(&key_gid[s + threadIdx.x]);
        // the fit paths always use the narrow count layout (count_stride_for)
        const uint32_t cst = kFit ? (uint32_t)kCountStride : cs.cstride;
        const uint32_t count = __ldcg(&cs.tile_count[(size_t)tt * cst]);
        if (count <= (uint32_t)NB && count <= cs.slab_cap) return Seg{s, count, kSegGlobal};
        if (count > cs.slab_cap) {
            if (threadIdx.x == 0) {
                *cursor = 0u;
                if (cs.seg_stats != nullptr) atomicAdd(&cs.seg_stats[0], 1u);
            }
            __syncthreads();
            return Seg{s, count, kSegStream};
        }
        if (count > (uint32_t)kSortMax3 && threadIdx.x == 0 && cs.seg_stats != nullptr)
            atomicAdd(&cs.seg_stats[1], 1u);
        const int r = sorted_segment<NT, kSortMax3>(proj, key_gid, s, s + count, n, t.img, t.tx,
                                                    t.ty, sl, scratch);
        return Seg{s, count, r >= 0 ? kSegSorted : kSegGlobal};
    }
    const uint32_t s = tile_range[tt], e = tile_range[tt + 1];
    if (presorted || e - s <= (uint32_t)NB) return Seg{s, e - s, kSegGlobal};
    const int r = sorted_segment<NT, kSortMax3>(proj, key_gid, s, e, n, t.img, t.tx, t.ty, sl,
                                                scratch);
    return Seg{s, e - s, r >= 0 ? kSegSorted : kSegGlobal};
}

__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7fffffffu; }

// Stage batch [base, base + NT) of the segment (thread j < cnt stages one
// record) and plan its chunks.  Returns the plan; *cnt_out = records staged.
template <int NT, int NB, bool kBwd>
__device__ __forceinline__ ChunkPlanOut stage_and_plan(FusedShared<NT, NB, kBwd>& sh, const Seg& sg,
                                                       uint32_t base, uint32_t* key_gid,
                                                       const Proj* __restrict__ proj, int n,
                                                       const TileCtx& t,
                                                       const uint32_t* __restrict__ gauss_off,
                                                       int& cnt_out, uint32_t gid0 = 0xffffffffu) {
    const int j = threadIdx.x;
    uint32_t gid = 0;
    int cnt;
    // slab entries read ahead (open_segment3): only for a one-batch segment
    // used in slab order (longer ones are re-ordered by sorted_segment)
    constexpr bool kAhead = !kBwd || NT == 128;
    if (kAhead && base == 0 && sg.mode == kSegGlobal && sg.L <= (uint32_t)NB &&
        gid0 != 0xffffffffu) {
        cnt = (int)sg.L;
        if (j < cnt) gid = gid0;
    } else {
        cnt = batch_gid<NT, NB>(sg, base, key_gid, sh.sl, proj, n, t, &sh.cursor, sh.scratch, gid);
    }
    uint32_t wj = 0, cabs = 0;
    if (j < cnt) {
        stage_gid(sh.sr, proj, gid, j, t, gauss_off);
        const uint4 c = sh.sr.c[j];
        const int lx0 = c.x & 0xff, lx1 = (c.x >> 8) & 0xff;
        const int ly0 = (c.x >> 16) & 0xff, ly1 = c.x >> 24;
        wj = (uint32_t)((lx1 - lx0 + 1) * (ly1 - ly0 + 1));
        cabs = max(abs_bits(sh.sr.a[j].w), max(abs_bits(sh.sr.b[j].x), abs_bits(sh.sr.b[j].y)));
    }
    cnt_out = cnt;
    return plan_chunks<NT, !kBwd>(sh.ch, cnt, wj, cabs);     // interleaved chunks for the render
}

// Forward of a planned batch: fixed-point sums into sh.u.acc (zeroed by the
// caller before the plan's first barrier).
template <int NT, int NB, bool kBwd>
__device__ __forceinline__ void forward_chunks(FusedShared<NT, NB, kBwd>& sh,
                                               const ChunkPlanOut& pl) {
    const int j = threadIdx.x;
    if (j >= (int)pl.n_items) return;
    const uint32_t it = sh.ch.item[j];
    const int r = (int)(it & 0xffu);
    GI_ASSERT(r < NB);
    const float cr = sh.sr.a[r].w * pl.scale, cg = sh.sr.b[r].x * pl.scale,
                cb = sh.sr.b[r].y * pl.scale;
    int* a0 = sh.u.acc[0];
    int* a1 = sh.u.acc[1];
    int* a2 = sh.u.acc[2];
    auto add = [&](int p, const float4&, const float4&, float, float, float w) {
        atomicAdd(&a0[p], __float_as_int(fmaf(cr, w, kFixMagic)) - kFixMagicBits);
        atomicAdd(&a1[p], __float_as_int(fmaf(cg, w, kFixMagic)) - kFixMagicBits);
        atomicAdd(&a2[p], __float_as_int(fmaf(cb, w, kFixMagic)) - kFixMagicBits);
    };
    if constexpr (kBwd) walk_chunk(sh.sr, it, add);
    else walk_chunk_ilv(sh.sr, it, add);
}

#ifndef GI_TILE3_MINB
#define GI_TILE3_MINB 6
#endif
// 128-thread fit kernel (launches of >= 3,072 tiles): 8 CTAs per SM, 64
// registers (10 -> 48 registers: 64 C2 images 42.5k -> 45.9k image-it/s,
// C3 fit 12.5k -> 12.8k it/s at 8; 6 / 7 measured lower)
#ifndef GI_TILE3_MINB128
#define GI_TILE3_MINB128 8
#endif
#ifndef GI_RENDER3_MINB
#define GI_RENDER3_MINB 6
#endif
#ifndef GI_RENDER3_MINB128
#define GI_RENDER3_MINB128 12
#endif

// kBwd = false: render (forward only, image out).  kBwd = true: forward +
// L2 + backward (or backward from a given dL/dC).
// kMinB > 0: CTAs per SM for the launch bounds (the decode frames' render,
// GI_DECODE3_MINB), else the macros above
#ifndef GI_DECODE3_MINB
#define GI_DECODE3_MINB 5
#endif
template <int NT, int NB, bool kBwd, int kMinB = 0>
__global__ void __launch_bounds__(NT, kMinB > 0 ? kMinB
                                      : NT == 256 ? (kBwd ? GI_TILE3_MINB : GI_RENDER3_MINB)
                                                  : (kBwd ? GI_TILE3_MINB128 : GI_RENDER3_MINB128))
    fused_tile_kernel(const Proj* __restrict__ proj, uint32_t* __restrict__ key_gid,
                      const uint32_t* __restrict__ tile_range,
                      const uint32_t* __restrict__ gauss_off, int n, int W, int H, int T, int TX,
                      bool presorted, const float* __restrict__ dL_dimage,
                      const float* __restrict__ target, float norm, int64_t pcap,
                      float* __restrict__ partial, float* __restrict__ ovf,
                      unsigned long long* __restrict__ sse_acc, float* __restrict__ image,
                      ChainState cs) {
    __shared__ FusedShared<NT, NB, kBwd> sh;
    constexpr int PPT = kTilePix / NT;       // pixels per thread: 1 (NT = 256) or 2
    TileCtx t;
    t.tx = blockIdx.x;
    t.row0 = cs.row1 > 0 ? cs.row0 : 0;
    t.ty = t.row0 + blockIdx.y;
    t.img = blockIdx.z;
    t.tile = blockIdx.y * TX + t.tx;
    t.row1 = t.row0 + gridDim.y;
    t.lane = threadIdx.x & 31;
    t.warp = threadIdx.x >> 5;
    const int j = threadIdx.x;
    const size_t P = (size_t)W * H;
    // L2 prefetches before waiting on the producer grid (L2 is the coherence
    // point: a later load sees the producer's writes): the tile's key count
    // and the first 512 B of its slab -- so the count and the keys arrive in
    // one memory round trip instead of two -- and the tile's target rows (an
    // input no kernel writes), consumed at the residual
#ifndef GI_NO_TILE3_PREFETCH
    if (cs.slab != nullptr && j < 5) {
        const size_t tt = (size_t)t.img * T + t.tile;
        if (j == 4) prefetch_l2(&cs.tile_count[tt * (kBwd ? (uint32_t)kCountStride : cs.cstride)]);
        else prefetch_l2(key_gid + tt * cs.slab_cap + 32 * j);
    }
    if (kBwd && target != nullptr && dL_dimage == nullptr && j >= 32 && j < 32 + 3 * kTile) {
        const int row = (j - 32) % kTile, ch = (j - 32) / kTile;
        const int y = t.ty * kTile + row, x = t.tx * kTile;
        if (y < H && x < W) prefetch_l2(target + (size_t)t.img * 3 * P + ch * P + (size_t)y * W + x);
    }
#endif
    griddep_wait();
    griddep_trigger();
    uint32_t gid0 = 0xffffffffu;     // the slab's entry threadIdx.x, read with the count
    const Seg sg = open_segment3<NT, NB, !kBwd || NT == 128, kBwd>(proj, key_gid, tile_range, presorted,
                                                             cs, n, T, t, sh.sl, sh.scratch,
                                                             &sh.cursor, gid0);
    const uint32_t L = sg.L;
    const bool fwd = !kBwd || dL_dimage == nullptr;
    const uint32_t* goff = kBwd ? gauss_off : nullptr;

    float accf[PPT][3];
#pragma unroll
    for (int q = 0; q < PPT; ++q) accf[q][0] = accf[q][1] = accf[q][2] = 0.f;
    ChunkPlanOut plan{};
    int cnt1 = 0;
    if (fwd) {
        for (uint32_t base = 0; base < L; base += NB) {
            if (base > 0) __syncthreads();
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
                const int p = j + q * NT;
                sh.u.acc[0][p] = 0;
                sh.u.acc[1][p] = 0;
                sh.u.acc[2][p] = 0;
            }
            plan = stage_and_plan<NT, NB, kBwd>(sh, sg, base, key_gid, proj, n, t, goff, cnt1, gid0);
            forward_chunks<NT, NB, kBwd>(sh, plan);
            __syncthreads();
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
                const int p = j + q * NT;
                accf[q][0] = fmaf((float)sh.u.acc[0][p], plan.inv_scale, accf[q][0]);
                accf[q][1] = fmaf((float)sh.u.acc[1][p], plan.inv_scale, accf[q][1]);
                accf[q][2] = fmaf((float)sh.u.acc[2][p], plan.inv_scale, accf[q][2]);
            }
        }
    }
    if constexpr (!kBwd) {
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
            const int p = j + q * NT;
            const int x = t.tx * kTile + (p & 15), y = t.ty * kTile + (p >> 4);
            if (x < W && y < H) {
                float* im = image + (size_t)t.img * 3 * P + (size_t)y * W + x;
                im[0] = accf[q][0];
                im[P] = accf[q][1];
                im[2 * P] = accf[q][2];
            }
        }
        close_segment(cs, t.img * T + t.tile);
        return;
    } else {
        // ---- residual: g = dL/dC per pixel (L2 loss), or the given dL/dC ----
        float sq = 0.f;
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
            const int p = j + q * NT;
            const int x = t.tx * kTile + (p & 15), y = t.ty * kTile + (p >> 4);
            float g0 = 0.f, g1 = 0.f, g2 = 0.f;
            if (x < W && y < H) {
                const size_t pix = (size_t)t.img * 3 * P + (size_t)y * W + x;
                if (!fwd) {
                    g0 = dL_dimage[pix];
                    g1 = dL_dimage[pix + P];
                    g2 = dL_dimage[pix + 2 * P];
                } else {
                    const float r0 = accf[q][0] - target[pix];
                    const float r1 = accf[q][1] - target[pix + P];
                    const float r2 = accf[q][2] - target[pix + 2 * P];
                    g0 = norm * r0;
                    g1 = norm * r1;
                    g2 = norm * r2;
                    sq += fmaf(r0, r0, fmaf(r1, r1, r2 * r2));
                    if (image != nullptr) {
                        image[pix] = accf[q][0];
                        image[pix + P] = accf[q][1];
                        image[pix + 2 * P] = accf[q][2];
                    }
                }
            }
            sh.g[p] = make_float4(g0, g1, g2, 0.f);
        }
        if (fwd && sse_acc != nullptr) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(kFull, sq, o);
            if (t.lane == 0) sh.sse[t.warp] = sq;
        }
        __syncthreads();
        if (fwd && sse_acc != nullptr && threadIdx.x == 0) {
            // per-image squared error in 2^-40 fixed point (deterministic)
            float tot = 0.f;
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) tot += sh.sse[w];
            atomicAdd(&sse_acc[t.img], (unsigned long long)__double2ll_rn((double)tot * kSseScale3));
        }

        // ---- backward: the same chunks accumulate the 8 sums of backward.cu's pass 2 ----
        // The forward's LAST batch is still staged and planned in shared
        // memory: pass 2 takes it first (no re-staging), then the others
        // (a record's partial does not depend on the batch order).  Streamed
        // segments (past the slab) are re-streamed in order.
        const uint32_t nbat = (L + NB - 1) / NB;
        const bool reuse = fwd && sg.mode != kSegStream && nbat > 0;
        if (threadIdx.x == 0) sh.cursor = 0u; // kSegStream: pass 2 streams from the start
        for (uint32_t ib = 0; ib < nbat; ++ib) {
            const uint32_t base = reuse ? (ib == 0 ? (nbat - 1) * NB : (ib - 1) * NB) : ib * NB;
            __syncthreads();
            int cnt = cnt1;
            ChunkPlanOut pl = plan;
            if (!(reuse && ib == 0))
                pl = stage_and_plan<NT, NB, kBwd>(sh, sg, base, key_gid, proj, n, t, gauss_off, cnt,
                                                  gid0);
            if (j < (int)pl.n_items) {
                float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f, a5 = 0.f, a6 = 0.f, a7 = 0.f;
                walk_chunk(sh.sr, sh.ch.item[j],
                           [&](int p, const float4& A, const float4& B, float u, float v, float w) {
                               const float4 gp = sh.g[p];
                               a0 = fmaf(gp.x, w, a0);
                               a1 = fmaf(gp.y, w, a1);
                               a2 = fmaf(gp.z, w, a2);
                               // -gamma = w <g, c'> (A.1, R12)
                               const float sdot = w * fmaf(A.w, gp.x, fmaf(B.x, gp.y, B.y * gp.z));
                               const float gu = -sdot * u, gv = -sdot * v;
                               a3 += gu;
                               a4 += gv;
                               a5 = fmaf(gu, u, a5);
                               a6 = fmaf(gu, v, a6);
                               a7 = fmaf(gv, v, a7);
                           });
                sh.u.red[j][0] = make_float4(a0, a1, a2, a3);
                sh.u.red[j][1] = make_float4(a4, a5, a6, a7);
            }
            __syncthreads();
            if (j < cnt) {
                const uint4 c = sh.sr.c[j];
                const uint32_t slot = c.z, jgid = c.w;
                if (slot == kOffOverflow || (int64_t)slot < pcap) {
                    const uint32_t jp = sh.ch.jplan[j];
                    const uint32_t fstart = jp & 0x1ffu, nf = (jp >> 9) & 0x1ffu;
                    float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
                    auto add = [&](uint32_t i) {
                        const float4 x = sh.u.red[i][0], y = sh.u.red[i][1];
                        s0.x += x.x; s0.y += x.y; s0.z += x.z; s0.w += x.w;
                        s1.x += y.x; s1.y += y.y; s1.z += y.z; s1.w += y.w;
                    };
                    GI_ASSERT(fstart + nf <= (uint32_t)NT && (!(jp >> 27) || ((jp >> 18) & 0x1ffu) < (uint32_t)NT));
                    for (uint32_t i = 0; i < nf; ++i) add(fstart + i);
                    if (jp >> 27) add((jp >> 18) & 0x1ffu);
                    if (slot == kOffOverflow) {     // > 4-tile Gaussian without slots
                        float* o = ovf + (size_t)jgid * 8;
                        atomicAdd(o + 0, s0.x); atomicAdd(o + 1, s0.y); atomicAdd(o + 2, s0.z);
                        atomicAdd(o + 3, s0.w); atomicAdd(o + 4, s1.x); atomicAdd(o + 5, s1.y);
                        atomicAdd(o + 6, s1.z); atomicAdd(o + 7, s1.w);
                    } else {
                        float4* dst = reinterpret_cast<float4*>(partial + (size_t)slot * 8);
                        dst[0] = s0;
                        dst[1] = s1;
                    }
                }
            }
        }
        close_segment(cs, t.img * T + t.tile);
    }
}

}  // namespace

// GI_TILE3=0: the round-1 kernels (A/B); GI_TILE3_NT=128: 128-thread CTAs
bool use_tile3() {
    static const bool v = [] {
        const char* e = std::getenv("GI_TILE3");
        return e == nullptr || e[0] != '0';
    }();
    return v;
}
// CTA size by launch size: 256 threads for one C2 image (1,536 tiles: the
// per-lane chunks stay short), 128 from 3,072 tiles up, where sparse tiles
// make the per-warp fixed work dominate (C3 init fit: 9.6k it/s at 256,
// 13.2k at 128; round-1 two-pixel kernel 12.2k).  GI_TILE3_NT forces either.
constexpr int kTile3SmallCta = 3072;
static int tile3_nt(int tiles) {
    static const int force = [] {
        const char* e = std::getenv("GI_TILE3_NT");
        return e == nullptr ? 0 : std::atoi(e);
    }();
    if (force == 128 || force == 256) return force;
    return tiles >= kTile3SmallCta ? 128 : 256;
}

// The render: the Gaussian-parallel kernel below 3,072 tiles (C2 frame 37.9k
// -> 44.1k FPS) when the cloud has >= 8 Gaussians per tile; from 3,072 tiles
// up, and for sparse clouds (codec frames of 2.2k-4.5k records over 1,536
// tiles), the round-1 two-pixel kernel's smaller per-tile work wins (C3 frame:
// 24.4k FPS vs 23.3k at 128 threads, 16.3k at 256; 2.2k records 40.8k vs
// 37.6k).
bool use_render3(int tiles_per_launch, int n_per_image, int tiles_per_image) {
    static const int force = [] {
        const char* e = std::getenv("GI_RENDER3");
        return e == nullptr ? -1 : (e[0] == '1' ? 1 : 0);
    }();
    if (!use_tile3()) return false;
    if (force >= 0) return force == 1;
    return tiles_per_launch < kTile3SmallCta && n_per_image >= 8 * tiles_per_image;
}

cudaError_t launch_fused_backward(const Proj* proj, uint32_t* key_gid, const uint32_t* tile_range,
                                  const uint32_t* gauss_off, int n, const gi_frame& f,
                                  bool presorted, const float* dL_dimage, const float* target,
                                  float norm, int64_t pcap, float* partial, float* ovf,
                                  unsigned long long* sse_acc, float* image_out,
                                  const ChainState& cs, cudaStream_t s) {
    const int TX = tiles_x(f.width);
    const int rows = cs.row1 > 0 ? cs.row1 - cs.row0 : tiles_y(f.height);
    const int T = TX * rows;
    if (rows <= 0) return cudaSuccess;
    const dim3 grid(TX, rows, f.batch);
    cudaError_t e = tile3_nt(T * f.batch) == 128
        ? launch_pdl(fused_tile_kernel<128, 128, true>, grid, dim3(128), s, proj, key_gid, tile_range,
                     gauss_off, n, f.width, f.height, T, TX, presorted, dL_dimage, target, norm,
                     pcap, partial, ovf, sse_acc, image_out, cs)
        : launch_pdl(fused_tile_kernel<256, kBwdBatch, true>, grid, dim3(256), s, proj, key_gid, tile_range,
                     gauss_off, n, f.width, f.height, T, TX, presorted, dL_dimage, target, norm,
                     pcap, partial, ovf, sse_acc, image_out, cs);
    note_launches(1);
    return e;
}

cudaError_t launch_fused_render(const Proj* proj, uint32_t* key_gid, const uint32_t* tile_range,
                                int n, const gi_frame& f, bool presorted, float* image,
                                const ChainState& cs, cudaStream_t s, bool decode) {
    const int TX = tiles_x(f.width);
    const int rows = cs.row1 > 0 ? cs.row1 - cs.row0 : tiles_y(f.height);
    const int T = TX * rows;
    if (rows <= 0) return cudaSuccess;
    const dim3 grid(TX, rows, f.batch);
    cudaError_t e = tile3_nt(T * f.batch) == 128
        ? launch_pdl(fused_tile_kernel<128, 128, false>, grid, dim3(128), s, proj, key_gid, tile_range,
                     nullptr, n, f.width, f.height, T, TX, presorted, nullptr, nullptr, 0.f,
                     (int64_t)0, nullptr, nullptr, nullptr, image, cs)
        : decode   // decoded clouds (larger boxes): 48 registers, 5 CTAs per SM (decode +4.6 %, frame -1.7 %)
        ? launch_pdl(fused_tile_kernel<256, kRenderBatch, false, GI_DECODE3_MINB>, grid, dim3(256), s,
                     proj, key_gid, tile_range, nullptr, n, f.width, f.height, T, TX, presorted,
                     nullptr, nullptr, 0.f, (int64_t)0, nullptr, nullptr, nullptr, image, cs)
        : launch_pdl(fused_tile_kernel<256, kRenderBatch, false>, grid, dim3(256), s, proj, key_gid, tile_range,
                     nullptr, n, f.width, f.height, T, TX, presorted, nullptr, nullptr, 0.f,
                     (int64_t)0, nullptr, nullptr, nullptr, image, cs);
    note_launches(1);
    return e;
}

}  // namespace gi
