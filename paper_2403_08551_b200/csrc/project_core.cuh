// Projection of one Gaussian (a1), shared by project_kernel and the fused
// finalize + Adam + next-step projection of the chained fit step.
// See project.cu for the precision plan (fp64 split centre, fp32 box recipe
// of reading R7; Cholesky conic by IEEE fp32 divisions, RS conic from fp64).
#pragma once
#include "gi_internal.cuh"

namespace gi {

// tanh in fp64 as sign(x) (1 - e) / (1 + e), e = exp(-2|x|): absolute error
// <= 1 ulp of 1 (checked against libm over |x| <= 20 and near 0), which is
// what mu = (u + 1) W / 2 needs (mu off by < 3e-13 px at W = 2040).  One exp
// and one division: ~4x fewer instructions than the library tanh, whose
// branchy polynomial paths are the longest part of the projection (and of the
// chained finalize, which projects the next step).
__device__ __forceinline__ double tanh_pos(double x) {
    const double e = exp(-2.0 * fabs(x));
    return copysign((1.0 - e) / (1.0 + e), x);
}

// App. C: u = tanh(mu_raw) (fp64), or the stored u (normalised positions).
__device__ __forceinline__ double activate_pos(float raw, uint32_t flags) {
    return pos_logit(flags) ? tanh_pos((double)raw) : (double)raw;
}

// The 48-byte record, pixel box and tile rectangle of one Gaussian from its
// activated position (ux, uy) and parameters; returns the tiles touched.
__device__ __forceinline__ uint32_t project_rec(double ux, double uy,
                                                const float4 p0 /* mux, muy, l1, l2 */,
                                                const float4 p1 /* l3, c'r, c'g, c'b */, int W,
                                                int H, float k, uint32_t flags, Proj& r,
                                                int4& rect /* out: tile rect when touched > 0 */) {
    // R2: mu = (u + 1) * W / 2  (fp64, no contraction)
    const double mx = __dmul_rn(__dadd_rn(ux, 1.0), (double)W * 0.5);
    const double my = __dmul_rn(__dadd_rn(uy, 1.0), (double)H * 0.5);

    // Covariance factor: Cholesky (Eq. 1) or rotation-scaling (Eq. 2-3),
    // App. C "+0.5" on l1, l3 resp. s1, s2 (fp32 as stored).
    const bool rs = cov_rs(flags);
    const float e1 = __fadd_rn(rs ? p0.w : p0.z, 0.5f);   // l1 + 1/2  |  s1 + 1/2
    const float e2 = rs ? p0.z : p0.w;                    // l2        |  theta
    const float e3 = __fadd_rn(p1.x, 0.5f);               // l3 + 1/2  |  s2 + 1/2
    double Srs[3] = {0.0, 0.0, 0.0};
    if (rs) rs_sigma((double)e2, (double)e1, (double)e3, Srs);
    uint32_t bx = kEmptyBox, by = kEmptyBox, touched = 0;
    int ix = 0, iy = 0;
    float fx = 0.f, fy = 0.f;
    const bool centre_ok = (mx >= 0.0) && (mx <= (double)W) && (my >= 0.0) && (my <= (double)H);
    if (centre_ok) {
        const double fix = floor(mx), fiy = floor(my);
        ix = (int)fix;
        iy = (int)fiy;
        fx = __double2float_rn(mx - fix);
        fy = __double2float_rn(my - fiy);
    }
    if (centre_ok && e1 != 0.0f && e3 != 0.0f) {
        // R6/R7: half extents k sqrt(Sxx), k sqrt(Syy): Cholesky k |l1e| and
        // k sqrt(l2^2 + l3e^2) in fp32; RS from the fp64 Sigma rounded once
        const float rx = rs ? __fmul_rn(k, __fsqrt_rn(__double2float_rn(Srs[0])))
                            : __fmul_rn(k, fabsf(e1));
        const float ry = rs ? __fmul_rn(k, __fsqrt_rn(__double2float_rn(Srs[2])))
                            : __fmul_rn(k, __fsqrt_rn(__fadd_rn(__fmul_rn(e2, e2),
                                                                __fmul_rn(e3, e3))));
        const float cx = __fsub_rn(fx, 0.5f), cy = __fsub_rn(fy, 0.5f);
        const float bw = (float)(W + 1), bh = (float)(H + 1);
        const float lox = fminf(fmaxf(__fsub_rn(cx, rx), -bw), bw);
        const float hix = fminf(fmaxf(__fadd_rn(cx, rx), -bw), bw);
        const float loy = fminf(fmaxf(__fsub_rn(cy, ry), -bh), bh);
        const float hiy = fminf(fmaxf(__fadd_rn(cy, ry), -bh), bh);
        const int x0 = max(0, ix + (int)ceilf(lox));
        const int x1 = min(W - 1, ix + (int)floorf(hix));
        const int y0 = max(0, iy + (int)ceilf(loy));
        const int y1 = min(H - 1, iy + (int)floorf(hiy));
        if (x0 <= x1 && y0 <= y1) {
            bx = (uint32_t)x0 | ((uint32_t)x1 << 16);
            by = (uint32_t)y0 | ((uint32_t)y1 << 16);
            touched = (uint32_t)((x1 / kTile - x0 / kTile + 1) * (y1 / kTile - y0 / kTile + 1));
            rect = make_int4(x0 / kTile, x1 / kTile, y0 / kTile, y1 / kTile);
        }
    }
    // Sigma^-1 = L^-T L^-1 with L^-1 = [[1/l1, 0], [-l2/(l1 l3), 1/l3]], scaled by
    // kappa so that sigma * log2(e) = (a dx)^2 + (b dx + c dy)^2.  Cholesky:
    // IEEE fp32 divisions (< 1e-6 relative on sigma near the box edge).  RS:
    // L = chol(Sigma) in fp64 (l3 = |s1 s2| / l1 since det Sigma = (s1 s2)^2).
    float ca, cb, cc;
    if (!rs) {
        const float kf = (float)kKappa;
        ca = __fdiv_rn(kf, e1);
        cc = __fdiv_rn(kf, e3);
        cb = -__fdiv_rn(__fmul_rn(ca, e2), e3);
    } else {
        const double l1 = sqrt(Srs[0]);
        const double l2 = Srs[1] / l1;
        const double l3 = fabs((double)e1 * (double)e3) / l1;
        ca = (float)(kKappa / l1);
        cb = (float)(-kKappa * l2 / (l1 * l3));
        cc = (float)(kKappa / l3);
    }
    r.q0 = make_float4(__int_as_float(ix), __int_as_float(iy), fx, fy);
    r.q1 = make_float4(ca, cb, cc, __uint_as_float(bx));
    r.q2 = make_float4(p1.y, p1.z, p1.w, __uint_as_float(by));
    return touched;
}

// a1 (+ binning step 1) of Gaussian g by one thread.
__device__ __forceinline__ uint32_t project_one(const float4 p0, const float4 p1, int g, int n, int W,
                                                int H, float k, uint32_t flags,
                                                Proj* __restrict__ proj, const BinCounts& bc,
                                                int4& rect) {
    Proj r;
    uint32_t touched = project_rec(activate_pos(p0.x, flags), activate_pos(p0.y, flags), p0, p1, W,
                                   H, k, flags, r, rect);
    const int TX = (W + kTile - 1) / kTile;
    int TW = TX * ((H + kTile - 1) / kTile);
    if (bc.row1 > 0) {                 // NEXT-4 window: count only the rank's tile rows
        rect = window_rect(rect, bc.row0, bc.row1);
        touched = rect_area(rect);
        TW = TX * (bc.row1 - bc.row0);
    }
    if (touched > 0u && bc.tile_count != nullptr)   // fused binning step 1: counts and ranks
        count_keys(bc, g, rect.x, rect.y, rect.z, rect.w, touched, (g / n) * TW, TX);
    proj[g] = r;
    return touched;
}

}  // namespace gi
