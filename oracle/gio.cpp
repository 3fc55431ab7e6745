// gio -- the fp64 CPU ORACLE for the GaussianImage hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.  The
// product path (paper_2403_08551_b200/, libgi.so) never links, imports or
// calls it, and this file includes nothing from it: the two share no code,
// headers, tables or constants.
//
// What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
//   * activation  -- tanh position, +0.5 on the L diagonal   App. C
//   * covariance  -- Sigma = L L^T                             Eq. 1
//   * sigma       -- 1/2 d^T Sigma^-1 d, d = pixel centre - mu Eq. 5
//   * render      -- C_i = sum_n c'_n exp(-sigma_n)           Eq. 7
//   * L2 loss     -- mean squared error                       Sec. 3.4
//   * backward    -- App. A.1 and A.2 Cholesky,
//                    with the corrections listed in DESIGN.md (R12-R14)
//   * Adam        -- textbook Kingma-Ba (north_star; reading R16), schedule
//                    "1e-3, halved every 20000 steps"
//   * decode      -- fp16 positions, Eq. 8 dequant, Eq. 9
//                    RVQ sum, record layout SPEC.md:404
//   * encode      -- (NEXT-2) the quantisers those invert: fp16 rounding of
//                    the post-tanh position, Eq. 8 codes, Eq. 9 greedy RVQ
//   * binning     -- (tile, gaussian) pairs grouped by tile, no depth key
//                    (north_star), by two independent methods
// Floating point is fp64 except the box recipe (reading R7), which is stated
// in IEEE binary32 with no FMA contraction so that the discrete box is
// reproducible bit-for-bit (compile with -ffp-contract=off).
//
// Parity pins: tests/test_oracle_*.py (worked examples from the paper/SPEC,
// closed forms, brute force, finite differences).  The fitting TRAJECTORY over
// many steps is "parity unpinned" (no worked fit values in the paper).

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// ---------------------------------------------------------------- activation
// App. C: "apply the tanh function to limit the range of position
// parameters to (-1,1)"; reading R2: mu_pix = (u + 1) * W / 2, y-down.
// pos_mode bit 0 (decode path, P:254 / R19): params already hold u in (-1, 1).
// pos_mode bit 1 (NEXT-3): params[2:5] = (theta, s1, s2) of the rotation-
// scaling factorisation Sigma = (RS)(RS)^T (Eq. 2-3) instead of the
// Cholesky vector (l1, l2, l3) (Eq. 1).
constexpr int kPosNormalized = 1;
constexpr int kCovRS = 2;

struct Gauss {
    double u[2];      // normalised position in [-1, 1]
    double mu[2];     // pixel-space centre
    double l1e, l2, l3e;   // effective Cholesky factors, App. C "+0.5" (Cholesky mode)
    double th, s1e, s2e;   // rotation angle, effective scales (RS mode, App. C "+0.5")
    int rs;
    double S[3];      // Sigma = [[S0, S1], [S1, S2]]
    double Si[3];     // Sigma^-1
    double c[3];      // weighted colour c'
    int box[4];       // x0, x1, y0, y1 (inclusive); empty if x0 > x1
    int valid;        // 0 when the box is empty / culled
};

void activate(const float* p, int pos_mode, int W, int H, Gauss& g) {
    for (int a = 0; a < 2; ++a) {
        double r = (double)p[a];
        g.u[a] = (pos_mode & kPosNormalized) ? r : std::tanh(r);
    }
    g.mu[0] = (g.u[0] + 1.0) * ((double)W * 0.5);
    g.mu[1] = (g.u[1] + 1.0) * ((double)H * 0.5);
    g.rs = (pos_mode & kCovRS) != 0;
    g.l1e = (double)p[2] + 0.5;   // App. C "add 0.5 to the diagonal elements l1, l3"
    g.l2 = (double)p[3];
    g.l3e = (double)p[4] + 0.5;
    g.th = (double)p[2];          // App. C "... or the scaling elements s1, s2"
    g.s1e = (double)p[3] + 0.5;
    g.s2e = (double)p[4] + 0.5;
    for (int k = 0; k < 3; ++k) g.c[k] = (double)p[5 + k];
}

// Eq. 1: Sigma = L L^T with L = [[l1, 0], [l2, l3]]
// Eq. 2-3: Sigma = (R S)(R S)^T, R = [[cos, -sin], [sin, cos]], S = diag(s1, s2)
void covariance(Gauss& g) {
    if (!g.rs) {
        g.S[0] = g.l1e * g.l1e;
        g.S[1] = g.l1e * g.l2;
        g.S[2] = g.l2 * g.l2 + g.l3e * g.l3e;
        return;
    }
    const double c = std::cos(g.th), s = std::sin(g.th);
    const double R[2][2] = {{c, -s}, {s, c}};
    const double M[2][2] = {{R[0][0] * g.s1e, R[0][1] * g.s2e}, {R[1][0] * g.s1e, R[1][1] * g.s2e}};
    g.S[0] = M[0][0] * M[0][0] + M[0][1] * M[0][1];
    g.S[1] = M[0][0] * M[1][0] + M[0][1] * M[1][1];
    g.S[2] = M[1][0] * M[1][0] + M[1][1] * M[1][1];
}

// closed-form inverse of a symmetric 2x2 matrix (adjugate / determinant)
void inverse2(const double S[3], double Si[3]) {
    double det = S[0] * S[2] - S[1] * S[1];
    Si[0] = S[2] / det;
    Si[1] = -S[1] / det;
    Si[2] = S[0] / det;
}

// Eq. 5: sigma = 1/2 d^T Sigma^-1 d
double eval_sigma(const double Si[3], double dx, double dy) {
    return 0.5 * (Si[0] * dx * dx + 2.0 * Si[1] * dx * dy + Si[2] * dy * dy);
}

// ------------------------------------------------------------ box (R6, R7)
// Tight axis-aligned box of the k-sigma ellipse (half extents k*sqrt(Sxx),
// k*sqrt(Syy)), sampled at pixel centres x + 1/2.  Stated in binary32 on a
// split centre mu = i + f so that both implementations take the same
// float -> int decisions.
void box_fp32(Gauss& g, const float* p, float k, int W, int H) {
    g.box[0] = 0; g.box[1] = -1; g.box[2] = 0; g.box[3] = -1;
    g.valid = 0;
    double mx = g.mu[0], my = g.mu[1];
    if (!(mx >= 0.0 && mx <= (double)W && my >= 0.0 && my <= (double)H)) return;
    double fix = std::floor(mx), fiy = std::floor(my);
    int ix = (int)fix, iy = (int)fiy;
    float fx = (float)(mx - fix);
    float fy = (float)(my - fiy);
    float rx, ry;
    if (!g.rs) {
        float l1e = p[2] + 0.5f;
        float l2 = p[3];
        float l3e = p[4] + 0.5f;
        if (l1e == 0.0f || l3e == 0.0f) return;                   // R8 cull
        rx = k * std::fabs(l1e);                                  // k sqrt(Sxx)
        float l2sq = l2 * l2;
        float l3sq = l3e * l3e;
        ry = k * std::sqrt(l2sq + l3sq);                          // k sqrt(Syy)
    } else {
        // RS: Sxx, Syy from the fp64 covariance (Eq. 2-3), rounded once
        float s1e = p[3] + 0.5f, s2e = p[4] + 0.5f;
        if (s1e == 0.0f || s2e == 0.0f) return;                   // singular Sigma
        rx = k * std::sqrt((float)g.S[0]);
        ry = k * std::sqrt((float)g.S[2]);
    }
    float cx = fx - 0.5f, cy = fy - 0.5f;
    float lox = cx - rx, hix = cx + rx;
    float loy = cy - ry, hiy = cy + ry;
    float bw = (float)(W + 1), bh = (float)(H + 1);
    lox = std::fmin(std::fmax(lox, -bw), bw);
    hix = std::fmin(std::fmax(hix, -bw), bw);
    loy = std::fmin(std::fmax(loy, -bh), bh);
    hiy = std::fmin(std::fmax(hiy, -bh), bh);
    int x0 = std::max(0, ix + (int)std::ceil(lox));
    int x1 = std::min(W - 1, ix + (int)std::floor(hix));
    int y0 = std::max(0, iy + (int)std::ceil(loy));
    int y1 = std::min(H - 1, iy + (int)std::floor(hiy));
    if (x0 > x1 || y0 > y1) return;
    g.box[0] = x0; g.box[1] = x1; g.box[2] = y0; g.box[3] = y1;
    g.valid = 1;
}

void project_one(const float* p, int pos_mode, int W, int H, float k, Gauss& g) {
    activate(p, pos_mode, W, H, g);
    covariance(g);
    inverse2(g.S, g.Si);
    box_fp32(g, p, k, W, H);
}

std::vector<Gauss> project_all(const float* params, int n, int pos_mode, int W, int H, float k) {
    std::vector<Gauss> gs((size_t)n);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) project_one(params + 8 * (size_t)i, pos_mode, W, H, k, gs[i]);
    return gs;
}

inline bool in_box(const Gauss& g, int x, int y) {
    return g.valid && x >= g.box[0] && x <= g.box[1] && y >= g.box[2] && y <= g.box[3];
}

int tiles_x(int W, int ts) { return (W + ts - 1) / ts; }
int tiles_y(int H, int ts) { return (H + ts - 1) / ts; }

void tile_rect(const Gauss& g, int ts, int r[4]) {
    if (!g.valid) { r[0] = 0; r[1] = -1; r[2] = 0; r[3] = -1; return; }
    r[0] = g.box[0] / ts; r[1] = g.box[1] / ts;
    r[2] = g.box[2] / ts; r[3] = g.box[3] / ts;
}

// method (ii): emit (tile, n) for every tile of n's rect (row-major), n
// ascending, then a stable sort by tile id only (no depth key).
int64_t bin_sort(const std::vector<Gauss>& gs, int W, int H, int ts,
                 std::vector<uint32_t>& kt, std::vector<uint32_t>& kg) {
    (void)H;
    int TX = tiles_x(W, ts);
    std::vector<std::pair<uint32_t, uint32_t>> keys;
    for (size_t n = 0; n < gs.size(); ++n) {
        int r[4];
        tile_rect(gs[n], ts, r);
        for (int ty = r[2]; ty <= r[3]; ++ty)
            for (int tx = r[0]; tx <= r[1]; ++tx)
                keys.push_back({(uint32_t)(ty * TX + tx), (uint32_t)n});
    }
    std::stable_sort(keys.begin(), keys.end(),
                     [](const std::pair<uint32_t, uint32_t>& a,
                        const std::pair<uint32_t, uint32_t>& b) { return a.first < b.first; });
    kt.resize(keys.size()); kg.resize(keys.size());
    for (size_t i = 0; i < keys.size(); ++i) { kt[i] = keys[i].first; kg[i] = keys[i].second; }
    return (int64_t)keys.size();
}

// method (i): for every tile, scan all Gaussians in index order.
int64_t bin_scan(const std::vector<Gauss>& gs, int W, int H, int ts,
                 std::vector<uint32_t>& kt, std::vector<uint32_t>& kg) {
    int TX = tiles_x(W, ts), TY = tiles_y(H, ts);
    kt.clear(); kg.clear();
    std::vector<std::array<int, 4>> rects(gs.size());
    for (size_t n = 0; n < gs.size(); ++n) tile_rect(gs[n], ts, rects[n].data());
    for (int ty = 0; ty < TY; ++ty)
        for (int tx = 0; tx < TX; ++tx)
            for (size_t n = 0; n < gs.size(); ++n) {
                const int* r = rects[n].data();
                if (tx >= r[0] && tx <= r[1] && ty >= r[2] && ty <= r[3]) {
                    kt.push_back((uint32_t)(ty * TX + tx));
                    kg.push_back((uint32_t)n);
                }
            }
    return (int64_t)kt.size();
}

void ranges_of(const std::vector<uint32_t>& kt, int T, uint32_t* range) {
    // range[t] = first index with key_tile >= t, t = 0..T
    for (int t = 0; t <= T; ++t)
        range[t] = (uint32_t)(std::lower_bound(kt.begin(), kt.end(), (uint32_t)t) - kt.begin());
}

// A.2 Cholesky: dL/dl = <G, dSigma/dl>, G = [[g1, g2], [g2, g3]]
void chol_backward(const double Gm[3], double l1, double l2, double l3, double dl[3]) {
    dl[0] = 2.0 * Gm[0] * l1 + 2.0 * Gm[1] * l2;
    dl[1] = 2.0 * Gm[1] * l1 + 2.0 * Gm[2] * l2;   // P:627 printed "2 g2 l1 + g2 l2"; corrected (R14)
    dl[2] = 2.0 * Gm[2] * l3;
}

// App. A.2 rotation-scaling: dL/dtheta = <G, dR/dtheta S S^T R^T +
// R S S^T dR^T/dtheta>; dL/ds_i = <G, R diag(2 s_i e_i) R^T> (the elided inner
// products of P:682-697 completed as in SPEC.md:188).
void rs_backward(const double Gm[3], double th, double s1, double s2, double d[3]) {
    const double c = std::cos(th), s = std::sin(th);
    const double G[2][2] = {{Gm[0], Gm[1]}, {Gm[1], Gm[2]}};
    const double R[2][2] = {{c, -s}, {s, c}};
    const double Rt[2][2] = {{c, s}, {-s, c}};
    const double dR[2][2] = {{-s, -c}, {c, -s}};
    const double dRt[2][2] = {{-s, c}, {-c, -s}};
    const double SS[2][2] = {{s1 * s1, 0.0}, {0.0, s2 * s2}};
    auto mul = [](const double A[2][2], const double B[2][2], double C[2][2]) {
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) C[i][j] = A[i][0] * B[0][j] + A[i][1] * B[1][j];
    };
    auto frob = [](const double A[2][2], const double B[2][2]) {
        return A[0][0] * B[0][0] + A[0][1] * B[0][1] + A[1][0] * B[1][0] + A[1][1] * B[1][1];
    };
    double T1[2][2], T2[2][2], T3[2][2], T4[2][2], dS[2][2];
    mul(dR, SS, T1); mul(T1, Rt, T2);               // dR S S^T R^T
    mul(R, SS, T3);  mul(T3, dRt, T4);              // R S S^T dR^T
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) dS[i][j] = T2[i][j] + T4[i][j];
    d[0] = frob(G, dS);
    const double D1[2][2] = {{2.0 * s1, 0.0}, {0.0, 0.0}};
    const double D2[2][2] = {{0.0, 0.0}, {0.0, 2.0 * s2}};
    mul(R, D1, T1); mul(T1, Rt, T2);
    d[1] = frob(G, T2);
    mul(R, D2, T1); mul(T1, Rt, T2);
    d[2] = frob(G, T2);
}

bool singular(const Gauss& g) {
    return g.rs ? (g.s1e == 0.0 || g.s2e == 0.0) : (g.l1e == 0.0 || g.l3e == 0.0);
}

}  // namespace

extern "C" {

int gio_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void gio_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

// Eq. 5, exposed for pins.
double gio_eval_sigma(const double* Si, double dx, double dy) { return eval_sigma(Si, dx, dy); }

// A.2 rotation-scaling backward, exposed for pins.
void gio_rs_backward(const double* G, double th, double s1e, double s2e, double* d) {
    rs_backward(G, th, s1e, s2e, d);
}

// A.2 Cholesky backward, exposed for pins.
void gio_chol_backward(const double* G, double l1e, double l2, double l3e, double* dl) {
    chol_backward(G, l1e, l2, l3e, dl);
}

// Closed-form 2x2 inverse, exposed for pins.
void gio_inverse2(const double* S, double* Si) { inverse2(S, Si); }

// Projection of n Gaussians of one image.  Outputs (any may be NULL):
//   mu[n][2] pixel centre; sig[n][3] Sigma (xx, xy, yy); sinv[n][3];
//   box[n][4] x0,x1,y0,y1 (empty = 0,-1,0,-1); rect[n][4] tile rect;
//   touched[n] number of tiles in the rect.
void gio_project(const float* params, int n, int W, int H, float k, int ts, int pos_mode,
                 double* mu, double* sig, double* sinv, int32_t* box, int32_t* rect,
                 uint32_t* touched) {
    std::vector<Gauss> gs = project_all(params, n, pos_mode, W, H, k);
    for (int i = 0; i < n; ++i) {
        const Gauss& g = gs[i];
        if (mu) { mu[2 * i] = g.mu[0]; mu[2 * i + 1] = g.mu[1]; }
        if (sig) for (int j = 0; j < 3; ++j) sig[3 * i + j] = g.S[j];
        if (sinv) for (int j = 0; j < 3; ++j) sinv[3 * i + j] = g.Si[j];
        if (box) for (int j = 0; j < 4; ++j) box[4 * i + j] = g.box[j];
        int r[4];
        tile_rect(g, ts, r);
        if (rect) for (int j = 0; j < 4; ++j) rect[4 * i + j] = r[j];
        if (touched) touched[i] = g.valid ? (uint32_t)((r[1] - r[0] + 1) * (r[3] - r[2] + 1)) : 0u;
    }
}

// Binning.  method 0 = per-tile scan (i), 1 = emit + stable sort (ii).
// Returns K.  Writes keys only if cap >= K (pass cap = 0 to count).
// tile_range has T + 1 entries, T = ceil(W/ts) * ceil(H/ts).
int64_t gio_bin(const float* params, int n, int W, int H, float k, int ts, int pos_mode,
                int method, uint32_t* key_tile, uint32_t* key_gid, int64_t cap,
                uint32_t* tile_range) {
    std::vector<Gauss> gs = project_all(params, n, pos_mode, W, H, k);
    std::vector<uint32_t> kt, kg;
    int64_t K = method == 0 ? bin_scan(gs, W, H, ts, kt, kg) : bin_sort(gs, W, H, ts, kt, kg);
    if (K <= cap && key_tile && key_gid) {
        std::memcpy(key_tile, kt.data(), sizeof(uint32_t) * (size_t)K);
        std::memcpy(key_gid, kg.data(), sizeof(uint32_t) * (size_t)K);
    }
    if (tile_range) ranges_of(kt, tiles_x(W, ts) * tiles_y(H, ts), tile_range);
    return K;
}

// Eq. 7 forward render, image planar [3][H][W] fp64.
//   mode 0 all-pairs: every Gaussian tested against every pixel (box predicate)
//   mode 1 tiled: Gaussians from the pixel's tile list (method ii), same predicate
//   mode 2 dense: no box, every Gaussian contributes (closed-form pins)
// Within a pixel, terms are summed in ascending Gaussian index.
void gio_render(const float* params, int n, int W, int H, float k, int ts, int pos_mode,
                int mode, double* image) {
    std::vector<Gauss> gs = project_all(params, n, pos_mode, W, H, k);
    std::vector<uint32_t> kt, kg, range;
    int TX = tiles_x(W, ts), TY = tiles_y(H, ts);
    if (mode == 1) {
        bin_sort(gs, W, H, ts, kt, kg);
        range.resize((size_t)TX * TY + 1);
        ranges_of(kt, TX * TY, range.data());
    }
    const size_t P = (size_t)W * H;
#pragma omp parallel for schedule(dynamic, 1)
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            double acc[3] = {0.0, 0.0, 0.0};
            auto add = [&](const Gauss& g) {
                double dx = (double)x + 0.5 - g.mu[0];   // R1 half-pixel centre
                double dy = (double)y + 0.5 - g.mu[1];
                double w = std::exp(-eval_sigma(g.Si, dx, dy));
                for (int c = 0; c < 3; ++c) acc[c] += g.c[c] * w;
            };
            if (mode == 0) {
                for (int i = 0; i < n; ++i) if (in_box(gs[i], x, y)) add(gs[i]);
            } else if (mode == 1) {
                int t = (y / ts) * TX + (x / ts);
                for (uint32_t j = range[t]; j < range[t + 1]; ++j) {
                    const Gauss& g = gs[kg[j]];
                    if (in_box(g, x, y)) add(g);
                }
            } else {
                for (int i = 0; i < n; ++i) {
                    const Gauss& g = gs[i];
                    if (singular(g)) continue;
                    add(g);
                }
            }
            for (int c = 0; c < 3; ++c) image[c * P + (size_t)y * W + x] = acc[c];
        }
    }
}

// Sec. 3.4 L2 loss, mean over the 3HW values (reading R11), and its
// gradient dL/dC = 2 (C - T) / (3HW).  g may be NULL.
double gio_mse(const double* image, const float* target, int W, int H, double* g) {
    const size_t cnt = (size_t)3 * W * H;
    double s = 0.0;
    for (size_t i = 0; i < cnt; ++i) {
        double r = image[i] - (double)target[i];
        s += r * r;
        if (g) g[i] = 2.0 * r / (double)cnt;
    }
    return s / (double)cnt;
}

// Appendix A backward.  g = dL/dC planar [3][H][W]; grads [n][8] in the raw
// parameter layout {mux, muy, l1, l2, l3, c'r, c'g, c'b}.
//   mode 0: pairs with the pixel inside the box (= forward modes 0 and 1)
//   mode 2: dense (no box), the derivative of the dense render
void gio_backward(const float* params, int n, int W, int H, float k, int ts, int pos_mode,
                  int mode, const double* g, double* grads) {
    (void)ts;
    std::vector<Gauss> gs = project_all(params, n, pos_mode, W, H, k);
    const size_t P = (size_t)W * H;
#pragma omp parallel for schedule(dynamic, 64)
    for (int i = 0; i < n; ++i) {
        const Gauss& G = gs[i];
        double* out = grads + 8 * (size_t)i;
        for (int j = 0; j < 8; ++j) out[j] = 0.0;
        int x0 = 0, x1 = W - 1, y0 = 0, y1 = H - 1;
        if (mode != 2) {
            if (!G.valid) continue;
            x0 = G.box[0]; x1 = G.box[1]; y0 = G.box[2]; y1 = G.box[3];
        } else if (singular(G)) {
            continue;
        }
        double dc[3] = {0, 0, 0};
        double dmu[2] = {0, 0};
        double Gm[3] = {0, 0, 0};    // dL/dSigma = [[g1, g2], [g2, g3]]
        const double* Si = G.Si;
        for (int y = y0; y <= y1; ++y) {
            for (int x = x0; x <= x1; ++x) {
                double dx = (double)x + 0.5 - G.mu[0];
                double dy = (double)y + 0.5 - G.mu[1];
                double w = std::exp(-eval_sigma(Si, dx, dy));
                size_t pix = (size_t)y * W + x;
                double gk[3] = {g[pix], g[P + pix], g[2 * P + pix]};
                // A.1 colour: dC^k/dc'^k = exp(-sigma)
                for (int c = 0; c < 3; ++c) dc[c] += gk[c] * w;
                // A.1 sigma (corrected R12): dC^k/dsigma = -c'^k exp(-sigma)
                double dL_dsigma = 0.0;
                for (int c = 0; c < 3; ++c) dL_dsigma += gk[c] * (-G.c[c] * w);
                // A.1 mean (sign R13): d = p - mu => dsigma/dmu = -Sigma^-1 d
                double sdx = Si[0] * dx + Si[1] * dy;
                double sdy = Si[1] * dx + Si[2] * dy;
                dmu[0] += dL_dsigma * (-sdx);
                dmu[1] += dL_dsigma * (-sdy);
                // A.1 covariance: dsigma/dSigma = -1/2 Sigma^-1 d d^T Sigma^-1
                Gm[0] += dL_dsigma * (-0.5 * sdx * sdx);
                Gm[1] += dL_dsigma * (-0.5 * sdx * sdy);
                Gm[2] += dL_dsigma * (-0.5 * sdy * sdy);
            }
        }
        double dl[3];
        if (G.rs) rs_backward(Gm, G.th, G.s1e, G.s2e, dl);      // NEXT-3
        else chol_backward(Gm, G.l1e, G.l2, G.l3e, dl);
        double dl1 = dl[0], dl2 = dl[1], dl3 = dl[2];
        // activation chain (App. C): mu = (tanh(r) + 1) W/2 => dmu/dr = W/2 sech^2 r
        double sx, sy;
        if ((pos_mode & kPosNormalized) == 0) {
            double chx = std::cosh((double)params[8 * (size_t)i]);
            double chy = std::cosh((double)params[8 * (size_t)i + 1]);
            sx = (double)W * 0.5 / (chx * chx);
            sy = (double)H * 0.5 / (chy * chy);
        } else {
            sx = (double)W * 0.5;
            sy = (double)H * 0.5;
        }
        out[0] = dmu[0] * sx;
        out[1] = dmu[1] * sy;
        out[2] = dl1;     // the +0.5 offset has unit derivative
        out[3] = dl2;
        out[4] = dl3;
        out[5] = dc[0]; out[6] = dc[1]; out[7] = dc[2];
    }
}

// Learning-rate schedule: lr0 halved every `half_every` steps;
// step is 1-based (reading R17).
double gio_lr_at(int step, double lr0, int half_every) {
    int halvings = (step - 1) / half_every;
    return lr0 * std::pow(0.5, (double)halvings);
}

// One Adam step (Kingma & Ba; north_star, reading R16), fp64 from fp32 state.
void gio_adam(const float* p_in, const float* g, const float* m_in, const float* v_in,
              int64_t count, int step, float lr, float beta1, float beta2, float eps,
              double* p_out, double* m_out, double* v_out) {
    const double b1 = beta1, b2 = beta2;
    const double bc1 = 1.0 - std::pow(b1, (double)step);
    const double bc2 = 1.0 - std::pow(b2, (double)step);
    for (int64_t i = 0; i < count; ++i) {
        double gi = g[i];
        double m = b1 * (double)m_in[i] + (1.0 - b1) * gi;
        double v = b2 * (double)v_in[i] + (1.0 - b2) * gi * gi;
        double mhat = m / bc1, vhat = v / bc2;
        p_out[i] = (double)p_in[i] - (double)lr * mhat / (std::sqrt(vhat) + (double)eps);
        m_out[i] = m;
        v_out[i] = v;
    }
}

// One Adan step ("optimized ... using the Adan optimizer"; the update
// rule is the cited Adan reference's, reading R28), fp64 from fp32 state:
//   d = g - g_prev (d = 0 at step 1: g_prev := g)
//   m = b1 m + (1-b1) g
//   v = b2 v + (1-b2) d
//   n = b3 n + (1-b3) (g + b2 d)^2
//   p = p (1 - lr wd) - lr (m/(1-b1^t) + b2 v/(1-b2^t)) / (sqrt(n/(1-b3^t)) + eps)
// g_prev_out = g.
void gio_adan(const float* p_in, const float* g, const float* m_in, const float* v_in,
              const float* n_in, const float* gprev_in, int64_t count, int step, float lr,
              float beta1, float beta2, float beta3, float eps, float wd, double* p_out,
              double* m_out, double* v_out, double* n_out) {
    const double b1 = beta1, b2 = beta2, b3 = beta3;
    const double bc1 = 1.0 - std::pow(b1, (double)step);
    const double bc2 = 1.0 - std::pow(b2, (double)step);
    const double bc3 = 1.0 - std::pow(b3, (double)step);
    for (int64_t i = 0; i < count; ++i) {
        const double gi = g[i];
        const double d = step == 1 ? 0.0 : gi - (double)gprev_in[i];
        const double m = b1 * (double)m_in[i] + (1.0 - b1) * gi;
        const double v = b2 * (double)v_in[i] + (1.0 - b2) * d;
        const double u = gi + b2 * d;
        const double nn = b3 * (double)n_in[i] + (1.0 - b3) * u * u;
        const double upd = (m / bc1 + b2 * v / bc2) / (std::sqrt(nn / bc3) + (double)eps);
        p_out[i] = (double)p_in[i] * (1.0 - (double)lr * (double)wd) - (double)lr * upd;
        m_out[i] = m;
        v_out[i] = v;
        n_out[i] = nn;
    }
}

// IEEE 754 binary16 -> double, written out from the format definition.
double gio_half_to_double(uint32_t h) {
    int sign = (h >> 15) & 1;
    int e = (h >> 10) & 0x1f;
    int f = h & 0x3ff;
    double v;
    if (e == 0) v = std::ldexp((double)f, -24);                  // subnormal
    else if (e == 31) v = f ? NAN : INFINITY;
    else v = std::ldexp(1.0 + (double)f / 1024.0, e - 15);
    return sign ? -v : v;
}

static uint64_t read_bits(const uint8_t* data, int64_t bitpos, int width) {
    uint64_t v = 0;
    for (int i = 0; i < width; ++i) {
        int64_t b = bitpos + i;
        uint64_t bit = (data[b >> 3] >> (7 - (b & 7))) & 1u;     // MSB-first
        v = (v << 1) | bit;
    }
    return v;
}

// Attribute decode: per record, 2 x fp16 position
// (post-tanh u), 3 x b-bit Cholesky codes, M x ceil(log2 B) RVQ indices.
//   u     = binary16 value
//   l_i   = code_i * gamma_i + beta_i, rounded once to fp32        (Eq. 8)
//   c'    = C^1[i^1] + ... + C^M[i^M] in fp32, stage order        (Eq. 9)
// Output params [n][8] fp32 for projection with pos_mode 1.
// Returns 0, or -1 if the payload is too short.
int gio_vq_decode(const uint8_t* payload, int64_t nbytes, int n, int bits, int stages,
                  int codebook, const float* gamma, const float* beta, const float* books,
                  float* params) {
    int ib = 1;
    while ((1 << ib) < codebook) ++ib;
    int64_t rec = 32 + 3 * (int64_t)bits + (int64_t)stages * ib;
    if ((rec * n + 7) / 8 > nbytes) return -1;
    for (int i = 0; i < n; ++i) {
        int64_t pos = rec * i;
        float* out = params + 8 * (size_t)i;
        out[0] = (float)gio_half_to_double((uint32_t)read_bits(payload, pos, 16));
        out[1] = (float)gio_half_to_double((uint32_t)read_bits(payload, pos + 16, 16));
        pos += 32;
        for (int j = 0; j < 3; ++j) {
            uint64_t code = read_bits(payload, pos, bits);
            pos += bits;
            out[2 + j] = std::fmaf((float)code, gamma[j], beta[j]);
        }
        float c[3] = {0.0f, 0.0f, 0.0f};
        for (int m = 0; m < stages; ++m) {
            uint64_t idx = read_bits(payload, pos, ib);
            pos += ib;
            const float* cw = books + ((size_t)m * codebook + idx) * 3;
            for (int j = 0; j < 3; ++j) c[j] = (m == 0) ? cw[j] : c[j] + cw[j];
        }
        out[5] = c[0]; out[6] = c[1]; out[7] = c[2];
    }
    return 0;
}

// PSNR: on images clamped to [0, 1], peak 1,
// identical inputs capped at 100 dB.
double gio_psnr(const double* x, const float* y, int64_t count) {
    double s = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        double a = std::min(1.0, std::max(0.0, x[i]));
        double b = std::min(1.0, std::max(0.0, (double)y[i]));
        s += (a - b) * (a - b);
    }
    double mse = s / (double)count;
    if (mse <= 1e-10) return 100.0;
    return std::min(100.0, 10.0 * std::log10(1.0 / mse));
}


// ------------------------------------------------------------ encoder (NEXT-2)
// IEEE 754 binary16 from binary32, round to nearest, ties to even (SPEC
// "fp16 = IEEE 754 binary16, round-to-nearest-even from float32"), written
// from the format definition: 1 sign, 5 exponent (bias 15), 10 fraction bits.
uint32_t gio_float_to_half(float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    const uint32_t sign = (b >> 16) & 0x8000u;
    const uint32_t e = (b >> 23) & 0xffu, m = b & 0x7fffffu;
    if (e == 0xffu) return sign | 0x7c00u | (m ? 0x200u : 0u);         // inf, nan
    const int E = (int)e - 127;
    if (E > 15) return sign | 0x7c00u;                                  // overflow
    if (E >= -14) {                                                     // normal half
        uint32_t h = ((uint32_t)(E + 15) << 10) | (m >> 13);
        const uint32_t rest = m & 0x1fffu;
        if (rest > 0x1000u || (rest == 0x1000u && (h & 1u))) h += 1u;   // may carry to inf
        return sign | h;
    }
    if (E < -25 || e == 0u) return sign;                                // below 2^-25: zero
    // subnormal half: value / 2^-24 = (m | 2^23) * 2^(E + 1)
    const uint32_t mf = m | 0x800000u;
    const int sh = -(E + 1);                                            // 14 .. 24
    uint32_t q = mf >> sh;
    const uint32_t rem = mf & ((1u << sh) - 1u), half = 1u << (sh - 1);
    if (rem > half || (rem == half && (q & 1u))) q += 1u;
    return sign | q;
}

// Attribute quantisation of one cloud (SPEC quant module):
//   position: u = tanh(mu_raw) (fp64, App. C) rounded to fp32 then to fp16
//             ("16-bit float precision for position parameters")
//   l_i:      code = round_half_even(clamp((l_i - beta_i) / gamma_i, 0,
//             2^b - 1)) in fp32 (Eq. 8; the paper fixes no precision, so the
//             decision is taken in the kernel's, reading R30)
//   c':       greedy RVQ (Eq. 9): i^m = argmin_k ||C^m[k] - (c' - c^^{m-1})||^2
//             with c^^{m-1} = sum_{k<m} C^k[i^k] in fp32 stage order and the
//             distance in fp32 ((d0^2 + d1^2) + d2^2); ties -> lowest index
// Outputs the codes and the dequantised ("effective") parameters exactly as
// gio_vq_decode produces them from the packed record.
void gio_vq_encode(const float* params, int n, int pos_mode, const float* gamma,
                   const float* beta, const float* books, int bits, int stages, int codebook,
                   uint32_t* pos16, uint32_t* codes, uint32_t* idx, float* eff) {
    const float qmax = (float)((1u << bits) - 1u);
    for (int i = 0; i < n; ++i) {
        const float* p = params + 8 * (size_t)i;
        float* out = eff + 8 * (size_t)i;
        for (int a = 0; a < 2; ++a) {
            double u = (pos_mode & kPosNormalized) ? (double)p[a] : std::tanh((double)p[a]);
            uint32_t h = gio_float_to_half((float)u);
            pos16[2 * (size_t)i + a] = h;
            out[a] = (float)gio_half_to_double(h);
        }
        for (int j = 0; j < 3; ++j) {
            float d = p[2 + j] - beta[j];
            float x = d / gamma[j];
            x = std::fmin(std::fmax(x, 0.0f), qmax);
            uint32_t code = (uint32_t)std::nearbyint(x);
            codes[3 * (size_t)i + j] = code;
            out[2 + j] = std::fmaf((float)code, gamma[j], beta[j]);
        }
        float chat[3] = {0.0f, 0.0f, 0.0f};
        for (int m = 0; m < stages; ++m) {
            float r[3];
            for (int j = 0; j < 3; ++j) r[j] = p[5 + j] - chat[j];
            int best = 0;
            float bestd = INFINITY;
            for (int k = 0; k < codebook; ++k) {
                const float* cw = books + ((size_t)m * codebook + k) * 3;
                float d0 = cw[0] - r[0], d1 = cw[1] - r[1], d2 = cw[2] - r[2];
                float dd = d0 * d0;
                dd = dd + d1 * d1;
                dd = dd + d2 * d2;
                if (dd < bestd) {
                    bestd = dd;
                    best = k;
                }
            }
            idx[(size_t)i * stages + m] = (uint32_t)best;
            const float* cw = books + ((size_t)m * codebook + best) * 3;
            for (int j = 0; j < 3; ++j) chat[j] = (m == 0) ? cw[j] : chat[j] + cw[j];
        }
        out[5] = chat[0]; out[6] = chat[1]; out[7] = chat[2];
    }
}


// K-means (Lloyd) for the RVQ codebooks ("The color codebooks are
// initialized using the K-means algorithm"; 5 iterations).  Per
// iteration: each point goes to its nearest centroid (the fp32 distance and
// tie rule of the encoder above), then every centroid with at least one
// point becomes the fp64 mean of its points rounded once to fp32; an empty
// cluster keeps its centroid (reading R31).  Returns the fp64 distortion of
// the final assignment (sum of squared distances to the centroids it used).
double gio_kmeans(const float* pts, int n, int B, float* cent, int iters, uint32_t* assign) {
    double distortion = 0.0;
    for (int it = 0; it < iters; ++it) {
        std::vector<double> sum((size_t)B * 3, 0.0), cnt((size_t)B, 0.0);
        distortion = 0.0;
        for (int i = 0; i < n; ++i) {
            const float* x = pts + 3 * (size_t)i;
            int best = 0;
            float bestd = INFINITY;
            for (int k = 0; k < B; ++k) {
                const float* c = cent + 3 * (size_t)k;
                float d0 = c[0] - x[0], d1 = c[1] - x[1], d2 = c[2] - x[2];
                float dd = d0 * d0;
                dd = dd + d1 * d1;
                dd = dd + d2 * d2;
                if (dd < bestd) {
                    bestd = dd;
                    best = k;
                }
            }
            assign[i] = (uint32_t)best;
            const float* c = cent + 3 * (size_t)best;
            for (int j = 0; j < 3; ++j) {
                sum[3 * (size_t)best + j] += (double)x[j];
                double d = (double)x[j] - (double)c[j];
                distortion += d * d;
            }
            cnt[best] += 1.0;
        }
        for (int k = 0; k < B; ++k)
            if (cnt[k] > 0.0)
                for (int j = 0; j < 3; ++j) cent[3 * (size_t)k + j] = (float)(sum[3 * (size_t)k + j] / cnt[k]);
    }
    return distortion;
}

}  // extern "C"
