/*
 * TRIPS trilinear point-splatting rasterizer -- CPU ORACLE.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` leg may load or call this library.  The product
 * path (paper_2401_06003_b200/) never imports, links or executes anything here, and
 * this file shares no code, header, table or constant generator with it.
 *
 * What it computes (arXiv 2401.06003, /root/reference/PAPER.md):
 *   project      : Sec. 3.1, Eq. (2)      s = f * s_w / z
 *   layer select : PAPER.md:189-191 (L_lower = floor(log2 s), L_upper = ceil(log2 s)),
 *                  Eq. (4), eps = 0.25 PAPER.md:208-210
 *   footprint    : Eq. (3) PAPER.md:193-198   gamma = beta * iota * alpha,
 *                  beta = (1-|x-x_i|)(1-|y-y_i|)
 *   lists        : Sec. 3.2 PAPER.md:216-217 per-pixel lists, sorted by depth,
 *                  clamped to 16
 *   blend        : Eqs. (5)-(6) PAPER.md:218-225  C = sum_m T_m alpha_m c_m,
 *                  T_m = prod_{i<m} (1 - alpha_i)
 *   backward     : chain rule of Eqs. (2)-(6); PAPER.md:294 (sorted lists reused)
 *
 * Readings of the paper where it is silent or garbled are SURVEY.md Sec. 8(c) Q1-Q24
 * and are listed in DESIGN.md ("Readings").  In short: log base 2 (Q1); s == 2^k lands
 * wholly in layer k with iota = 1 (Q2); the garbled "s_i = 0 and s < 1" means
 * "layer 0 and s < 1" (Q3); s >= 2^(n-1) clamps to layer n-1 with iota = 1 (Q5);
 * layer-l coordinates are x_l = x * 2^-l with pixel (i,j) centred at (i,j) (Q7);
 * layer sizes ceil(W/2^l) x ceil(H/2^l) (Q8); every in-bounds pixel of each 2x2
 * footprint is a fragment, zero weight included (Q9); alpha_m := gamma_m and
 * c_m := tau_i (Q10); depth is view-space z (Q11); ties broken by point index (Q12);
 * cull if !(z > near) or x, y, s non-finite or s < 0 (Q14); channel F of each layer is
 * A = sum_m T_m gamma_m (Q16); no early termination in the definition (Q17).
 *
 * Precision (Q18): the paper states none.  The "exact block" (projection, layer
 * selection, footprint, beta, gamma) is evaluated in `real`, every operation
 * rounded (this file must be compiled with -ffp-contract=off, no fast-math).  The
 * library is built twice: real = float (the parity reference; the GPU path must
 * agree bit for bit on levels, pixel indices and counts) and real = double (used
 * by the finite-difference pins).  Blending and the backward pass are always
 * evaluated in double.
 *
 * Algorithm (plain, no blocking, no fusion -- one pass per definition):
 *   1. project every point                               (Sec. 3.1)
 *   2. emit every fragment (pixel, z, i) of every point  (Eq. 3, "eight pixels")
 *   3. sort all fragments by (pixel, z, i) with qsort     (Sec. 3.2 "sorted by depth")
 *   4. per pixel keep the first min(16, |list|)           (Sec. 3.2 "clamped to 16")
 *   5. blend front to back in double                      (Eqs. 5-6)
 *   6. backward: reverse recurrences per pixel, then the projection chain per point.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef ORACLE_REAL
#error "compile with -DORACLE_REAL=float or -DORACLE_REAL=double"
#endif
typedef ORACLE_REAL real;

#define ORACLE_CAP 16          /* "clamped to a maximum size of 16 elements" */
#define ORACLE_EPS 0.25        /* "at least eps = 0.25" */

typedef struct {
    float fx, fy, cx, cy;      /* pixels; pixel (i,j) centre at (i,j) (Q7) */
    float f;                   /* focal length of Eq. (2) (Q6) */
    float R[9], t[3];          /* world -> view, row-major; OpenCV axes (Q24) */
    int32_t width, height;
    float near_plane;          /* Q14 */
} oracle_camera;

typedef struct {
    int64_t n_culled, n_visible, n_frag, n_kept, n_trunc_pixels, max_list;
} oracle_stats;

/* ---------------------------------------------------------------- geometry */

static int32_t layer_w(int32_t W, int l) { return (int32_t)((W + (1 << l) - 1) >> l); } /* Q8 */
static int32_t layer_h(int32_t H, int l) { return (int32_t)((H + (1 << l) - 1) >> l); }

int64_t oracle_num_pixels(int n_layers, int32_t W, int32_t H)
{
    int64_t p = 0;
    for (int l = 0; l < n_layers; ++l) p += (int64_t)layer_w(W, l) * layer_h(H, l);
    return p;
}

/* pyramid layout: layer-major, each layer planar [(F+1), H_l, W_l]; channel F = A. */
static int64_t layer_pixel_offset(int n_layers_unused, int32_t W, int32_t H, int l)
{
    (void)n_layers_unused;
    int64_t p = 0;
    for (int j = 0; j < l; ++j) p += (int64_t)layer_w(W, j) * layer_h(H, j);
    return p;
}

/* Sec. 3.1: p = R x + t, continuous screen coordinates and Eq. (2).
 * Pinned operation order: p_x = ((R00*X + R01*Y) + R02*Z) + t0; x = (fx*p_x)/z + cx;
 * s = (f*s_w)/z.  Returns 0 if the point is culled (Q14). */
static int project_point(const oracle_camera* c, const float* x, float sw, real out[4])
{
    real X = (real)x[0], Y = (real)x[1], Z = (real)x[2];
    real p[3];
    for (int r = 0; r < 3; ++r) {
        real a = (real)c->R[3 * r + 0] * X;
        real b = (real)c->R[3 * r + 1] * Y;
        real d = (real)c->R[3 * r + 2] * Z;
        real acc = a + b;
        acc = acc + d;
        acc = acc + (real)c->t[r];
        p[r] = acc;
    }
    real z = p[2];
    if (!(z > (real)c->near_plane)) return 0;
    real xs = ((real)c->fx * p[0]) / z + (real)c->cx;
    real ys = ((real)c->fy * p[1]) / z + (real)c->cy;
    real s = ((real)c->f * (real)sw) / z;                   /* Eq. (2) */
    if (!isfinite(xs) || !isfinite(ys) || !isfinite(s) || s < 0) return 0;
    out[0] = xs; out[1] = ys; out[2] = z; out[3] = s;
    return 1;
}

/* Layer selection, PAPER.md:189-210 with readings Q1-Q5.
 * Returns the number of selected layers (1 or 2); layer[], iota[] and diota[]
 * (d iota / d s, right derivative at kinks, Q19) are filled; *code is the level
 * code exported for parity (bits 0-3 lowest layer, 0x10 two layers, 0x20 eps
 * branch, 0x40 clamp). */
static int select_layers(real s, int n_layers, int layer[2], real iota[2], double diota[2], int* code)
{
    if (s < 1) {                                            /* second case of Eq. (4), Q3 */
        layer[0] = 0;
        iota[0] = (real)ORACLE_EPS + (real)(1.0 - ORACLE_EPS) * s;
        diota[0] = 1.0 - ORACLE_EPS;
        *code = 0x20;
        return 1;
    }
    int k = ilogb(s);                                       /* floor(log2 s), exact */
    if (k >= n_layers - 1) {                                /* Q5: clamp */
        layer[0] = n_layers - 1; iota[0] = 1; diota[0] = 0.0;
        *code = 0x40 | (n_layers - 1);
        return 1;
    }
    real m = (real)ldexp((double)s, -k);                    /* s / 2^k in [1,2), exact */
    if (m == 1) {                                           /* Q2: s == 2^k */
        layer[0] = k; iota[0] = 1; diota[0] = -ldexp(1.0, -k);
        *code = k;
        return 1;
    }
    /* first case of Eq. (4): iota = 1 - |s - s_i| / (2^Lup - 2^Llo), s_i = 2^L.
     * With m = s/2^k this is 2 - m for L = k and m - 1 for L = k + 1. */
    layer[0] = k;     iota[0] = (real)2 - m; diota[0] = -ldexp(1.0, -k);
    layer[1] = k + 1; iota[1] = m - (real)1; diota[1] = +ldexp(1.0, -k);
    *code = 0x10 | k;
    return 2;
}

/* One footprint pixel of Eq. (3) (Q7, Q9); its weights are evaluated by frag_weights(). */
typedef struct {
    int32_t px, py;             /* pixel in layer l */
    int dx, dy;                 /* which corner of the 2x2 footprint */
} corner_t;

/* Enumerates the in-bounds pixels of the 2x2 footprint in layer l.  Returns count. */
static int footprint(real xs, real ys, int l, int32_t Wl, int32_t Hl, corner_t out[4])
{
    real scale = (real)ldexp(1.0, -l);                      /* exact power of two */
    real xl = xs * scale, yl = ys * scale;
    if (!(xl >= (real)-1 && xl < (real)Wl && yl >= (real)-1 && yl < (real)Hl)) return 0;
    real x0 = floor(xl), y0 = floor(yl);
    int cnt = 0;
    for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
            int32_t px = (int32_t)x0 + dx, py = (int32_t)y0 + dy;
            if (px < 0 || px >= Wl || py < 0 || py >= Hl) continue;
            corner_t* c = &out[cnt++];
            c->px = px; c->py = py; c->dx = dx; c->dy = dy;
        }
    return cnt;
}

/* ---------------------------------------------------------------- projection export */

/* Projects all points.  proj[n*4] = (x, y, z, s) (NaN if culled), level[n] (-1 if
 * culled), iota[n*2] (second entry 0 for single-layer points). Any may be NULL. */
int oracle_project(const oracle_camera* cam, int n_layers, int64_t n, const float* pos,
                   const float* sw, real* proj, int8_t* level, real* iota)
{
    for (int64_t i = 0; i < n; ++i) {
        real pr[4];
        int vis = project_point(cam, pos + 3 * i, sw[i], pr);
        int lay[2] = {0, 0}, code = -1, ns = 0;
        real io[2] = {0, 0};
        double dio[2];
        if (vis) ns = select_layers(pr[3], n_layers, lay, io, dio, &code);
        if (proj) {
            for (int k = 0; k < 4; ++k) proj[4 * i + k] = vis ? pr[k] : (real)NAN;
        }
        if (level) level[i] = (int8_t)(vis ? code : -1);
        if (iota) { iota[2 * i] = vis ? io[0] : 0; iota[2 * i + 1] = (vis && ns == 2) ? io[1] : 0; }
    }
    return 0;
}

/* ---------------------------------------------------------------- lists */

typedef struct {
    int64_t pixel;              /* global pyramid pixel index (layer offset + y*W_l + x) */
    real z;
    uint32_t i;
    uint8_t l, dx, dy, sel;     /* layer, corner, which selected layer of the point */
} frag_t;

static int frag_cmp(const void* a, const void* b)
{
    const frag_t* x = (const frag_t*)a;
    const frag_t* y = (const frag_t*)b;
    if (x->pixel != y->pixel) return x->pixel < y->pixel ? -1 : 1;
    if (x->z != y->z) return x->z < y->z ? -1 : 1;          /* depth, ascending (Q11) */
    if (x->i != y->i) return x->i < y->i ? -1 : 1;          /* tie-break on index (Q12) */
    return 0;
}

typedef struct {
    const oracle_camera* cam;
    int n_layers, F;
    int64_t n;
    const float *pos, *sw, *alpha, *desc;
    real* pr;                   /* [n][4] projected, valid if vis[i] */
    uint8_t* vis;
    frag_t* frags;
    int64_t n_frag;
    int64_t* seg;               /* [P+1] segment starts in sorted frags */
    int64_t P;
} scene_t;

/* Builds the sorted fragment lists (steps 1-3).  mask (nullable, [P]) restricts the
 * lists to the marked pixels; unmarked pixels get empty lists. */
static int build_lists(scene_t* S, const uint8_t* mask)
{
    const oracle_camera* cam = S->cam;
    S->P = oracle_num_pixels(S->n_layers, cam->width, cam->height);
    S->pr = (real*)malloc(sizeof(real) * 4 * (size_t)(S->n ? S->n : 1));
    S->vis = (uint8_t*)malloc((size_t)(S->n ? S->n : 1));
    if (!S->pr || !S->vis) return -1;
    int64_t loff[16];
    for (int l = 0; l < S->n_layers; ++l) loff[l] = layer_pixel_offset(S->n_layers, cam->width, cam->height, l);

    size_t cap = 1024, cnt = 0;
    frag_t* fr = (frag_t*)malloc(sizeof(frag_t) * cap);
    if (!fr) return -1;
    for (int64_t i = 0; i < S->n; ++i) {
        S->vis[i] = (uint8_t)project_point(cam, S->pos + 3 * i, S->sw[i], S->pr + 4 * i);
        if (!S->vis[i]) continue;
        int lay[2], code;
        real io[2];
        double dio[2];
        int ns = select_layers(S->pr[4 * i + 3], S->n_layers, lay, io, dio, &code);
        for (int k = 0; k < ns; ++k) {
            int l = lay[k];
            int32_t Wl = layer_w(cam->width, l), Hl = layer_h(cam->height, l);
            corner_t c[4];
            int nc = footprint(S->pr[4 * i], S->pr[4 * i + 1], l, Wl, Hl, c);
            for (int q = 0; q < nc; ++q) {
                int64_t pix = loff[l] + (int64_t)c[q].py * Wl + c[q].px;
                if (mask && !mask[pix]) continue;
                if (cnt == cap) {
                    cap *= 2;
                    frag_t* nf = (frag_t*)realloc(fr, sizeof(frag_t) * cap);
                    if (!nf) { free(fr); return -1; }
                    fr = nf;
                }
                frag_t* f = &fr[cnt++];
                f->pixel = pix; f->z = S->pr[4 * i + 2]; f->i = (uint32_t)i;
                f->l = (uint8_t)l; f->dx = (uint8_t)c[q].dx; f->dy = (uint8_t)c[q].dy; f->sel = (uint8_t)k;
            }
        }
    }
    qsort(fr, cnt, sizeof(frag_t), frag_cmp);
    S->frags = fr;
    S->n_frag = (int64_t)cnt;
    S->seg = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S->P + 1));
    if (!S->seg) return -1;
    int64_t j = 0;
    for (int64_t p = 0; p <= S->P; ++p) {
        while (j < (int64_t)cnt && fr[j].pixel < p) ++j;
        S->seg[p] = j;
    }
    return 0;
}

static void free_scene(scene_t* S)
{
    free(S->pr); free(S->vis); free(S->frags); free(S->seg);
}

/* Weights of one fragment, recomputed from its point (Eq. 3-4). */
typedef struct {
    double gamma, beta, iota, diota, wx, wy;
} fw_t;

static fw_t frag_weights(const scene_t* S, const frag_t* f)
{
    const real* pr = S->pr + 4 * (int64_t)f->i;
    int lay[2], code;
    real io[2];
    double dio[2];
    select_layers(pr[3], S->n_layers, lay, io, dio, &code);
    real scale = (real)ldexp(1.0, -(int)f->l);
    real xl = pr[0] * scale, yl = pr[1] * scale;
    real x0 = floor(xl), y0 = floor(yl);                    /* exact; then one rounding in real */
    real fx = xl - x0, fy = yl - y0;
    real wx = f->dx ? fx : (real)1 - fx;
    real wy = f->dy ? fy : (real)1 - fy;
    real beta = wx * wy;
    real iota = io[f->sel];
    real gamma = (beta * iota) * (real)S->alpha[f->i];      /* Eq. (3) */
    fw_t w;
    w.gamma = (double)gamma; w.beta = (double)beta; w.iota = (double)iota;
    w.diota = dio[f->sel]; w.wx = (double)wx; w.wy = (double)wy;
    return w;
}

/* ---------------------------------------------------------------- T_min variant */

/* SURVEY.md 8(f) row 3 / reading Q17: with t_min > 0 (a variant, not the paper's definition)
 * a pixel's kept list ends with the fragment after which the transmittance drops below
 * t_min.  The cut is an integer decision taken in fp32 (T = T * (1 - gamma), each op rounded)
 * so that both implementations take it identically.  t_min = 0 (default) never cuts. */
static float g_t_min = 0.0f;

void oracle_set_t_min(float t) { g_t_min = t; }

static fw_t frag_weights(const scene_t* S, const frag_t* f);

static int64_t tmin_cut(const scene_t* S, const frag_t* const* lst, int64_t K)
{
    if (!(g_t_min > 0.0f)) return K;
    float T = 1.0f;
    for (int64_t m = 0; m < K; ++m) {
        const float g = (float)frag_weights(S, lst[m]).gamma;
        T = T * (1.0f - g);
        if (T < g_t_min) return m + 1;
    }
    return K;
}

/* ---------------------------------------------------------------- coarse-layer inclusion */

/* "we include points from coarser layers during blending (in the usual
 * way)".  Reading Q22 (a variant, off by default): with coarse = c > 0 the list
 * blended at pyramid pixel (l, x, y) is the union of the fragment lists of its ancestors
 * (l + d, x >> d, y >> d), d = 0 .. min(c, L - 1 - l), ordered by (z, i, d) -- depth, then
 * point index, then the finer layer first -- of which the first 16 are kept (Sec. 3.2).  Each
 * fragment keeps its own weight gamma (Eq. 3, evaluated in its own layer and pixel).  The
 * per-pixel counts remain the pixel's own list length.  kept_layer (nullable, [P*16]) receives
 * d for each kept entry (-1 padded). */
static int g_coarse = 0;
static int8_t* g_kept_layer = NULL;

void oracle_set_coarse(int c, int8_t* kept_layer) { g_coarse = c; g_kept_layer = kept_layer; }

static int list_cmp(const void* a, const void* b)
{
    const frag_t* x = *(const frag_t* const*)a;
    const frag_t* y = *(const frag_t* const*)b;
    if (x->z != y->z) return x->z < y->z ? -1 : 1;
    if (x->i != y->i) return x->i < y->i ? -1 : 1;
    if (x->l != y->l) return x->l < y->l ? -1 : 1;
    return 0;
}

/* The blend list of pixel (l, x, y) (global index p): up to 16 fragment pointers in blend
 * order.  Returns its length. */
static int64_t blend_list(const scene_t* S, int l, int32_t x, int32_t y, int64_t p, const frag_t** out)
{
    const int D = g_coarse <= 0 ? 0 : (g_coarse < S->n_layers - 1 - l ? g_coarse : S->n_layers - 1 - l);
    if (D == 0) {
        int64_t len = S->seg[p + 1] - S->seg[p];
        int64_t K = len < ORACLE_CAP ? len : ORACLE_CAP;    /* Sec. 3.2 */
        for (int64_t m = 0; m < K; ++m) out[m] = &S->frags[S->seg[p] + m];
        return K;
    }
    int64_t tot = 0;
    int64_t anc[16];
    for (int d = 0; d <= D; ++d) {
        const int la = l + d;
        anc[d] = layer_pixel_offset(S->n_layers, S->cam->width, S->cam->height, la)
               + (int64_t)(y >> d) * layer_w(S->cam->width, la) + (x >> d);
        tot += S->seg[anc[d] + 1] - S->seg[anc[d]];
    }
    const frag_t** all = (const frag_t**)malloc(sizeof(frag_t*) * (size_t)(tot ? tot : 1));
    int64_t k = 0;
    for (int d = 0; d <= D; ++d)
        for (int64_t j = S->seg[anc[d]]; j < S->seg[anc[d] + 1]; ++j) all[k++] = &S->frags[j];
    qsort(all, (size_t)tot, sizeof(frag_t*), list_cmp);
    const int64_t K = tot < ORACLE_CAP ? tot : ORACLE_CAP;
    for (int64_t m = 0; m < K; ++m) out[m] = all[m];
    free(all);
    return K;
}

/* With coarse inclusion a masked pixel also needs its ancestors' lists. */
static uint8_t* coarse_mask(const oracle_camera* cam, int n_layers, const uint8_t* mask)
{
    if (!mask || g_coarse <= 0) return NULL;
    const int64_t P = oracle_num_pixels(n_layers, cam->width, cam->height);
    uint8_t* m = (uint8_t*)malloc((size_t)P);
    memcpy(m, mask, (size_t)P);
    for (int l = 0; l < n_layers; ++l) {
        const int32_t Wl = layer_w(cam->width, l), Hl = layer_h(cam->height, l);
        const int64_t off = layer_pixel_offset(n_layers, cam->width, cam->height, l);
        for (int32_t y = 0; y < Hl; ++y)
            for (int32_t x = 0; x < Wl; ++x) {
                if (!mask[off + (int64_t)y * Wl + x]) continue;
                for (int d = 1; d <= g_coarse && l + d < n_layers; ++d)
                    m[layer_pixel_offset(n_layers, cam->width, cam->height, l + d)
                      + (int64_t)(y >> d) * layer_w(cam->width, l + d) + (x >> d)] = 1;
            }
    }
    return m;
}

/* ---------------------------------------------------------------- forward */

/* Forward rasterization.
 *   pyramid     [sum_l (F+1) H_l W_l] double (layout above), required
 *   pyramid_mag same layout, nullable: sum_m T_m gamma_m |tau| per channel (error scale)
 *   counts      [P] uint32 list lengths, nullable
 *   kept        [P*16] int32 kept point indices in blend order, -1 padded, nullable
 *   mask        [P] uint8, nullable: only marked pixels are computed (others zero)
 */
int oracle_forward(const oracle_camera* cam, int n_layers, int F, int64_t n, const float* pos,
                   const float* sw, const float* alpha, const float* desc, double* pyramid,
                   double* pyramid_mag, uint32_t* counts, int32_t* kept, const uint8_t* mask,
                   oracle_stats* stats)
{
    if (n_layers < 1 || n_layers > 16 || F < 1 || n < 0) return -1;
    scene_t S;
    memset(&S, 0, sizeof(S));
    S.cam = cam; S.n_layers = n_layers; S.F = F; S.n = n;
    S.pos = pos; S.sw = sw; S.alpha = alpha; S.desc = desc;
    uint8_t* cmask = coarse_mask(cam, n_layers, mask);
    const int brc = build_lists(&S, cmask ? cmask : mask);
    free(cmask);
    if (brc) { free_scene(&S); return -2; }

    oracle_stats st;
    memset(&st, 0, sizeof(st));
    for (int64_t i = 0; i < n; ++i) { if (S.vis[i]) st.n_visible++; else st.n_culled++; }
    st.n_frag = S.n_frag;

    for (int l = 0; l < n_layers; ++l) {
        int32_t Wl = layer_w(cam->width, l), Hl = layer_h(cam->height, l);
        int64_t poff = layer_pixel_offset(n_layers, cam->width, cam->height, l);
        int64_t foff = poff * (F + 1);                      /* float offset of the layer */
        int64_t plane = (int64_t)Wl * Hl;
        for (int64_t q = 0; q < plane; ++q) {
            int64_t p = poff + q;
            const int in = !(mask && !mask[p]);             /* unmarked: empty (even if an ancestor) */
            const int64_t len = in ? S.seg[p + 1] - S.seg[p] : 0;
            if (counts) counts[p] = (uint32_t)len;
            if (len > ORACLE_CAP) st.n_trunc_pixels++;
            if (len > st.max_list) st.max_list = len;
            st.n_kept += len < ORACLE_CAP ? len : ORACLE_CAP; /* Sec. 3.2 */
            const frag_t* lst[ORACLE_CAP];
            int64_t K = in ? blend_list(&S, l, (int32_t)(q % Wl), (int32_t)(q / Wl), p, lst) : 0;
            K = tmin_cut(&S, lst, K);
            double T = 1.0, A = 0.0, C[64], M[64];
            for (int c = 0; c < F; ++c) { C[c] = 0.0; M[c] = 0.0; }
            for (int64_t m = 0; m < K; ++m) {                /* Eqs. (5)-(6), alpha_m = gamma (Q10) */
                const frag_t* f = lst[m];
                fw_t w = frag_weights(&S, f);
                const float* tau = desc + (int64_t)f->i * F;
                for (int c = 0; c < F; ++c) {
                    C[c] += T * w.gamma * (double)tau[c];
                    M[c] += T * w.gamma * fabs((double)tau[c]);
                }
                A += T * w.gamma;                           /* Q16 */
                T *= (1.0 - w.gamma);
            }
            for (int c = 0; c < F; ++c) {
                pyramid[foff + c * plane + q] = C[c];
                if (pyramid_mag) pyramid_mag[foff + c * plane + q] = M[c];
            }
            pyramid[foff + F * plane + q] = A;
            if (pyramid_mag) pyramid_mag[foff + F * plane + q] = A;
            if (kept) {
                for (int m = 0; m < ORACLE_CAP; ++m)
                    kept[p * ORACLE_CAP + m] = m < K ? (int32_t)lst[m]->i : -1;
            }
            if (g_kept_layer) {
                for (int m = 0; m < ORACLE_CAP; ++m)
                    g_kept_layer[p * ORACLE_CAP + m] = (int8_t)(m < K ? (int)lst[m]->l - l : -1);
            }
        }
    }
    if (stats) *stats = st;
    free_scene(&S);
    return 0;
}

/* ---------------------------------------------------------------- backward */

/* Optional export of the per-point screen-space gradients of the last oracle_backward call
 * (SURVEY.md 8(b) SCREEN_GRADS): [n][4+F] doubles (d/dx, d/dy, d/ds in layer-0 pixels, d/dalpha,
 * d/dtau[F]) -- the values the projection chain below consumes -- and their |.| magnitudes. */
static double* g_screen_out = NULL;
static double* g_screen_mag = NULL;

void oracle_set_screen_out(double* screen, double* screen_mag) { g_screen_out = screen; g_screen_mag = screen_mag; }

/* Backward pass (chain rule of Eqs. 2-6; depth order and list membership held
 * constant).  Gradients w.r.t. the raw parameters (Q20), SUMMED
 * into grad (so several views can be accumulated, Q21):
 *   grad     [n][5+F] double, row = (d/dx, d/dy, d/dz, d/ds_w, d/dalpha, d/dtau[F])
 *   grad_mag [n][5+F] double, nullable: the same chain with |.| of every factor
 *            (a scale for the rounding error of any evaluation order)
 *   grad_cam [17] double, nullable: camera gradient (dR row-major, dt, dfx, dfy, dcx, dcy,
 *            df), summed; grad_cam_mag its magnitude scale (nullable)
 * grad_pyramid has the pyramid layout (float).  mask as in oracle_forward.
 */
int oracle_backward(const oracle_camera* cam, int n_layers, int F, int64_t n, const float* pos,
                    const float* sw, const float* alpha, const float* desc,
                    const float* grad_pyramid, double* grad, double* grad_mag, const uint8_t* mask,
                    double* grad_cam, double* grad_cam_mag)
{
    if (n_layers < 1 || n_layers > 16 || F < 1 || F > 64 || n < 0) return -1;
    scene_t S;
    memset(&S, 0, sizeof(S));
    S.cam = cam; S.n_layers = n_layers; S.F = F; S.n = n;
    S.pos = pos; S.sw = sw; S.alpha = alpha; S.desc = desc;
    uint8_t* cmask = coarse_mask(cam, n_layers, mask);
    const int brc = build_lists(&S, cmask ? cmask : mask);
    free(cmask);
    if (brc) { free_scene(&S); return -2; }

    /* screen-space gradients per point: (x, y, s, alpha, tau[F]) and magnitudes */
    int G = 4 + F;
    double* gs = (double*)calloc((size_t)(n ? n : 1) * G, sizeof(double));
    double* ms = (double*)calloc((size_t)(n ? n : 1) * G, sizeof(double));
    if (!gs || !ms) { free(gs); free(ms); free_scene(&S); return -2; }

    for (int l = 0; l < n_layers; ++l) {
        int32_t Wl = layer_w(cam->width, l), Hl = layer_h(cam->height, l);
        int64_t poff = layer_pixel_offset(n_layers, cam->width, cam->height, l);
        int64_t foff = poff * (F + 1);
        int64_t plane = (int64_t)Wl * Hl;
        for (int64_t q = 0; q < plane; ++q) {
            int64_t p = poff + q;
            if (mask && !mask[p]) continue;
            const frag_t* lst[ORACLE_CAP];
            int64_t K = blend_list(&S, l, (int32_t)(q % Wl), (int32_t)(q / Wl), p, lst);
            K = tmin_cut(&S, lst, K);
            if (K == 0) continue;
            double gC[64], gA = (double)grad_pyramid[foff + F * plane + q];
            for (int c = 0; c < F; ++c) gC[c] = (double)grad_pyramid[foff + c * plane + q];
            fw_t w[ORACLE_CAP];
            double T[ORACLE_CAP + 1];
            T[0] = 1.0;
            for (int64_t m = 0; m < K; ++m) {
                w[m] = frag_weights(&S, lst[m]);
                T[m + 1] = T[m] * (1.0 - w[m].gamma);       /* Eq. (6) */
            }
            /* suffix recurrences: B = blend of the fragments behind m (tau and |tau|),
             * bb = the same with tau == 1 (for A) */
            double B[64], MB[64], bb = 0.0;
            for (int c = 0; c < F; ++c) { B[c] = 0.0; MB[c] = 0.0; }
            for (int64_t m = K - 1; m >= 0; --m) {
                const frag_t* f = lst[m];
                const double lscale = ldexp(1.0, -(int)f->l);  /* d x_l / d x = 2^-l, l of the fragment */
                const float* tau = desc + (int64_t)f->i * F;
                double g = w[m].gamma, Tm = T[m];
                /* d out / d gamma_m = T_m (<gC, tau_m - B_m> + gA (1 - bb_m)) */
                double dg = 0.0, mg = 0.0;
                for (int c = 0; c < F; ++c) {
                    dg += gC[c] * ((double)tau[c] - B[c]);
                    mg += fabs(gC[c]) * (fabs((double)tau[c]) + MB[c]);
                }
                dg += gA * (1.0 - bb);
                mg += fabs(gA) * (1.0 + bb);
                dg *= Tm; mg *= Tm;
                double* gi = gs + (int64_t)f->i * G;
                double* mi = ms + (int64_t)f->i * G;
                for (int c = 0; c < F; ++c) {                 /* d C / d tau = T_m gamma_m */
                    gi[4 + c] += Tm * g * gC[c];
                    mi[4 + c] += Tm * g * fabs(gC[c]);
                }
                double a = (double)alpha[f->i];
                gi[3] += dg * w[m].beta * w[m].iota;          /* gamma = beta iota alpha */
                mi[3] += mg * w[m].beta * w[m].iota;
                double gb = dg * w[m].iota * a, mb = mg * w[m].iota * fabs(a);
                double gio = dg * w[m].beta * a, mio = mg * w[m].beta * fabs(a);
                /* beta = wx wy, wx = 1 - |x_l - x_i| : d wx / d x_l = dx ? +1 : -1 */
                gi[0] += gb * w[m].wy * (f->dx ? 1.0 : -1.0) * lscale;
                gi[1] += gb * w[m].wx * (f->dy ? 1.0 : -1.0) * lscale;
                mi[0] += mb * w[m].wy * lscale;
                mi[1] += mb * w[m].wx * lscale;
                gi[2] += gio * w[m].diota;                    /* iota(s), Eq. (4) */
                mi[2] += mio * fabs(w[m].diota);
                for (int c = 0; c < F; ++c) {
                    B[c] = g * (double)tau[c] + (1.0 - g) * B[c];
                    MB[c] = g * fabs((double)tau[c]) + (1.0 - g) * MB[c];
                }
                bb = g + (1.0 - g) * bb;
            }
        }
    }
    /* projection chain (Sec. 3.1, Eq. 2): x = fx p_x / z + cx, y = fy p_y / z + cy,
     * s = f s_w / z, z = p_z, p = R x_w + t. */
    int GO = 5 + F;
    for (int64_t i = 0; i < n; ++i) {
        if (!S.vis[i]) continue;
        const real* pr = S.pr + 4 * i;
        double xs = (double)pr[0], ys = (double)pr[1], z = (double)pr[2], s = (double)pr[3];
        const double* gi = gs + i * G;
        const double* mi = ms + i * G;
        double fx = cam->fx, fy = cam->fy, cx = cam->cx, cy = cam->cy;
        double gp[3], mp[3];
        gp[0] = gi[0] * fx / z;
        gp[1] = gi[1] * fy / z;
        gp[2] = -(gi[0] * (xs - cx) + gi[1] * (ys - cy) + gi[2] * s) / z;
        mp[0] = mi[0] * fx / z;
        mp[1] = mi[1] * fy / z;
        mp[2] = (mi[0] * (fabs(xs) + fabs(cx)) + mi[1] * (fabs(ys) + fabs(cy)) + mi[2] * s) / z;
        double* go = grad + i * GO;
        for (int k = 0; k < 3; ++k) {                         /* d/dx_w = R^T gp */
            go[k] += (double)cam->R[0 * 3 + k] * gp[0] + (double)cam->R[1 * 3 + k] * gp[1]
                   + (double)cam->R[2 * 3 + k] * gp[2];
        }
        go[3] += gi[2] * (double)cam->f / z;                  /* d s / d s_w = f / z */
        go[4] += gi[3];
        for (int c = 0; c < F; ++c) go[5 + c] += gi[4 + c];
        if (grad_cam) {
            /* camera parameters (PAPER.md:92, 268 optimise them):
             * [dR (9, row-major), dt (3), dfx, dfy, dcx, dcy, df], with p = R X + t,
             * x = fx p_x / z + cx, y = fy p_y / z + cy, s = f s_w / z. */
            const float* X = pos + 3 * i;
            double pv[3];
            for (int r = 0; r < 3; ++r)
                pv[r] = (double)cam->R[3 * r] * X[0] + (double)cam->R[3 * r + 1] * X[1]
                      + (double)cam->R[3 * r + 2] * X[2] + (double)cam->t[r];
            for (int a = 0; a < 3; ++a) {
                for (int b = 0; b < 3; ++b) grad_cam[3 * a + b] += gp[a] * (double)X[b];
                grad_cam[9 + a] += gp[a];
            }
            grad_cam[12] += gi[0] * pv[0] / z;
            grad_cam[13] += gi[1] * pv[1] / z;
            grad_cam[14] += gi[0];
            grad_cam[15] += gi[1];
            grad_cam[16] += gi[2] * (double)sw[i] / z;
            if (grad_cam_mag) {
                for (int a = 0; a < 3; ++a) {
                    for (int b = 0; b < 3; ++b) grad_cam_mag[3 * a + b] += mp[a] * fabs((double)X[b]);
                    grad_cam_mag[9 + a] += mp[a];
                }
                grad_cam_mag[12] += mi[0] * fabs(pv[0]) / z;
                grad_cam_mag[13] += mi[1] * fabs(pv[1]) / z;
                grad_cam_mag[14] += mi[0];
                grad_cam_mag[15] += mi[1];
                grad_cam_mag[16] += mi[2] * fabs((double)sw[i]) / z;
            }
        }
        if (grad_mag) {
            double* mo = grad_mag + i * GO;
            for (int k = 0; k < 3; ++k)
                mo[k] += fabs((double)cam->R[k]) * mp[0] + fabs((double)cam->R[3 + k]) * mp[1]
                       + fabs((double)cam->R[6 + k]) * mp[2];
            mo[3] += mi[2] * (double)cam->f / z;
            mo[4] += mi[3];
            for (int c = 0; c < F; ++c) mo[5 + c] += mi[4 + c];
        }
    }
    if (g_screen_out) memcpy(g_screen_out, gs, sizeof(double) * (size_t)n * G);
    if (g_screen_mag) memcpy(g_screen_mag, ms, sizeof(double) * (size_t)n * G);
    free(gs); free(ms);
    free_scene(&S);
    return 0;
}

/* ---------------------------------------------------------------- 4-NN size init */

/* Point-size initialisation, PAPER.md:302 ("Point sizes are initialized with the average
 * distance to the four nearest neighbor"), SURVEY.md 8(f) row 4.  Reading Q25:
 * for point i the K = min(4, #finite - 1) other finite points j with the smallest
 * (d2_ij, j), d2 = ((xj-xi)^2 + (yj-yi)^2) + (zj-zi)^2 evaluated in fp32 with every operation
 * rounded; size_i = (((sqrt d1 + sqrt d2) + sqrt d3) + sqrt d4) / K in fp32 (0 if K = 0 or
 * the point is not finite).  Brute force over all points: O(n) per query.
 *   queries  nullable: query indices (nq of them); NULL = all n points (nq ignored)
 *   size_out [nq] float, nbr_out nullable [nq][4] int32 (-1 padded), in query order */
static int finite3(const float* p) { return isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2]); }

int oracle_knn4(int64_t n, const float* pos, int64_t nq, const int64_t* queries, float* size_out, int32_t* nbr_out)
{
    if (n < 0 || !pos || !size_out) return -1;
    if (!queries) nq = n;
    for (int64_t q = 0; q < nq; ++q) {
        int64_t i = queries ? queries[q] : q;
        float bd[4];
        int64_t bj[4];
        int nb = 0;
        const float* pi = pos + 3 * i;
        if (finite3(pi)) {
            for (int64_t j = 0; j < n; ++j) {
                if (j == i) continue;
                const float* pj = pos + 3 * j;
                if (!finite3(pj)) continue;
                float dx = pj[0] - pi[0], dy = pj[1] - pi[1], dz = pj[2] - pi[2];
                float xx = dx * dx, yy = dy * dy, zz = dz * dz;
                float d2 = xx + yy;
                d2 = d2 + zz;
                /* insert (d2, j) into the ascending top-4 (j increases, so ties keep order) */
                if (nb == 4 && !(d2 < bd[3])) continue;
                int k = nb < 4 ? nb++ : 3;
                while (k > 0 && d2 < bd[k - 1]) { bd[k] = bd[k - 1]; bj[k] = bj[k - 1]; --k; }
                bd[k] = d2; bj[k] = j;
            }
        }
        float s = 0.0f;
        for (int k = 0; k < nb; ++k) s = s + sqrtf(bd[k]);
        size_out[q] = nb ? s / (float)nb : 0.0f;
        if (nbr_out)
            for (int k = 0; k < 4; ++k) nbr_out[4 * q + k] = k < nb ? (int32_t)bj[k] : -1;
    }
    return 0;
}
