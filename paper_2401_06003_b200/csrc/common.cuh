// common.cuh -- shared device definitions of the B200 TRIPS rasterizer.
//
// The "exact block" (projection, layer selection, footprint, beta, gamma) uses explicitly
// rounded intrinsics (__fmul_rn/__fadd_rn/__fdiv_rn/__fsub_rn) so that nvcc can neither
// contract to FMA nor reorder: levels, pixel indices and counts are then bit-identical to
// any IEEE evaluation of the same sequence.  Never compile this
// with --use_fast_math or -ftz=true.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace trips {

constexpr int kTile = 16;                 // pyramid tiles are 16 x 16 pixels
constexpr int kTilePix = kTile * kTile;   // one CTA thread per tile pixel
constexpr int kCap = 16;                  // "clamped to a maximum size of 16"
constexpr int kMaxLayers = 16;
// Kept lists are stored dense per tile, [tile][m][pixel] (16 slots per pixel, 4096 per tile), so
// that a warp's m-th entries are contiguous: the raster stores and the backward loads of keys and
// gamma coalesce (compact per-pixel runs were measured 14% slower in k_raster).
__host__ __device__ constexpr size_t kept_base(int t) { return (size_t)t * kTilePix * kCap; }

constexpr float kEps = 0.25f;             // "at least eps = 0.25"
constexpr uint64_t kKeyMax = ~0ull;
constexpr float kCulled = -1.0f;          // rec.s marker of a culled point

struct LayerGeom {
    int32_t W, H;          // ceil(W0 / 2^l), ceil(H0 / 2^l)   (reading Q8)
    int32_t tiles_x, tiles_y;
    int32_t tile_base;     // first global tile id of this layer
    int32_t pad;
    int64_t pix_off;       // pyramid pixel offset of the layer (pixel order of the export)
    int64_t float_off;     // pyramid float offset = pix_off * (F + 1)
};

struct Cam {
    float fx, fy, cx, cy, f;
    float R[9], t[3];
    float near_plane;
};

// Everything a kernel needs, passed by value (fits the 32 KB kernel-parameter space).
struct Params {
    int32_t n, F, FC, G;              // F features, FC = round_up(F,4), G = 8 + FC
    int32_t n_layers, T;              // layers, total tiles
    float t_min;                      // T_min blend variant (0 = the exact definition)
    int32_t coarse;                   // coarse-layer inclusion depth (0 = the exact definition)
    LayerGeom L[kMaxLayers];
    Cam cam;
    // inputs (caller)
    const float* pos; const float* sw; const float* alpha; const float* desc;
    // workspace
    float4* geo;           // [n]      screen record (x, y, s, alpha); s < 0 marks culled
    float* zbuf;           // [n]      view depth z
    float* tau_copy;       // [n][FC]  padded copy of desc, written only when !tau_direct
    const float* tau;      // [n][FC]  descriptors gathered by raster/backward: the caller's desc
                           //          itself when F % 4 == 0 and it is 16-B aligned (no per-view
                           //          copy), else tau_copy
    int32_t tau_direct;
    uint32_t* hist;        // [C][T]   per-CTA tile counts -> per-CTA offsets within the tile
    uint32_t* cta_vis;     // [C]      visible points per binning CTA (statistics)
    uint32_t* tile_cnt;    // [T]      pairs per tile (k_count's reservations)
    uint32_t* tile_off;    // [T+1]    first pair of each tile's bin; [T] = number of pairs M
    uint32_t* tile_perm;   // [T]      launch order of the per-tile kernels: heaviest bins first
                           //          (nullptr: tile order) -- the long tiles start in the first wave
    uint64_t* bin_key;     // [8n]     (z bits << 32 | i) per (tile, pair), tile-major
    uint16_t* bin_orig;    // [8n]     footprint origin in the tile: (qx0+1) | (qy0+1) << 5
    uint32_t* pix_cnt;     // [T*256]  list length per tile pixel
    uint32_t* pix_meta;    // [T*256]  K (kept-list length; T_min: the cut length)
    uint64_t* kept;        // [T*4096] coarse inclusion only: kept (z, i << 4 | d) keys in blend
                           //          order, [tile][m][pixel]
    uint64_t* kp_key;      // [T*4096] kept (point, tile) pairs of each tile, compact: (z, i) key
    uint32_t* kp_info;     // [T*4096] footprint origin in the tile (bits 0-9, as bin_orig), kept
                           //          corner mask (10-13), slot m of corner c in its pixel's kept
                           //          list (bits 14 + 4c .. 17 + 4c)
    uint32_t* kp_cnt;      // [T]      kept pairs per tile
    uint64_t* own;         // [T][16][256] coarse inclusion only: each pixel's own sorted top-16
    float* kept_gamma;     // [T*4096] gamma of each kept fragment (saved for the backward)
    unsigned long long* stats;  // [8]  n_culled, n_visible, n_pairs, n_frag, n_kept, n_trunc, max_list, n_kept_pairs
};

enum StatIdx { S_CULLED = 0, S_VISIBLE, S_PAIRS, S_FRAG, S_KEPT, S_TRUNC, S_MAXLIST, S_KPAIRS, S_COUNT };

// --------------------------------------------------------------------------- exact block

// Sec. 3.1.  p = R x + t with pinned order ((R0 X + R1 Y) + R2 Z) + t,
// x = (fx p_x) / z + cx, y = (fy p_y) / z + cy, s = (f s_w) / z.  Returns false if culled
// (reading Q14: !(z > near), or x, y, s non-finite, or s < 0).
__device__ __forceinline__ bool project_exact(const Cam& c, float X, float Y, float Z, float sw,
                                              float& xs, float& ys, float& z, float& s)
{
    float p[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        float a = __fmul_rn(c.R[3 * r + 0], X);
        float b = __fmul_rn(c.R[3 * r + 1], Y);
        float d = __fmul_rn(c.R[3 * r + 2], Z);
        float acc = __fadd_rn(a, b);
        acc = __fadd_rn(acc, d);
        p[r] = __fadd_rn(acc, c.t[r]);
    }
    z = p[2];
    if (!(z > c.near_plane)) return false;
    xs = __fadd_rn(__fdiv_rn(__fmul_rn(c.fx, p[0]), z), c.cx);
    ys = __fadd_rn(__fdiv_rn(__fmul_rn(c.fy, p[1]), z), c.cy);
    s = __fdiv_rn(__fmul_rn(c.f, sw), z);
    if (!isfinite(xs) || !isfinite(ys) || !isfinite(s) || s < 0.0f) return false;
    return true;
}

// Layer selection, readings Q1-Q5.  Returns the number of layers (1/2),
// the lowest layer, the weights iota[2] and d iota / d s (right derivative at kinks, Q19).
// Level code: bits 0-3 lowest layer, 0x10 two layers, 0x20 eps branch, 0x40 clamp.
#ifndef TRIPS_LEVELS_SELECT
#define TRIPS_LEVELS_SELECT 1
#endif
struct Levels {
    int n, lo, code;
    float iota[2];
    float diota[2];
};

__device__ __forceinline__ Levels select_levels(float s, int n_layers)
{
#if TRIPS_LEVELS_SELECT
    // branch-free form of the same cases (selects instead of divergent branches; identical values)
    {
        Levels L;
        const bool eps = s < 1.0f;
        const uint32_t bits = __float_as_uint(s);
        const int k = (int)(bits >> 23) - 127;
        const bool clamp = !eps && k >= n_layers - 1;
        const float m = __uint_as_float((bits & 0x007FFFFFu) | 0x3F800000u);
        const float inv = __uint_as_float((uint32_t)(127 - min(max(k, -126), 126)) << 23);
        const bool p2 = !eps && !clamp && m == 1.0f;
        const bool one = eps || clamp || p2;
        L.n = one ? 1 : 2;
        L.lo = eps ? 0 : (clamp ? n_layers - 1 : k);
        L.code = eps ? 0x20 : (clamp ? (0x40 | (n_layers - 1)) : (p2 ? k : (0x10 | k)));
        L.iota[0] = eps ? __fadd_rn(kEps, __fmul_rn(1.0f - kEps, s)) : ((clamp || p2) ? 1.0f : __fsub_rn(2.0f, m));
        L.iota[1] = one ? 0.0f : __fsub_rn(m, 1.0f);
        L.diota[0] = eps ? 1.0f - kEps : (clamp ? 0.0f : -inv);
        L.diota[1] = one ? 0.0f : inv;
        return L;
    }
#endif
    Levels L;
    if (s < 1.0f) {                                  // second case of Eq. (4), reading Q3
        L.n = 1; L.lo = 0; L.code = 0x20;
        L.iota[0] = __fadd_rn(kEps, __fmul_rn(1.0f - kEps, s));
        L.diota[0] = 1.0f - kEps;
        L.iota[1] = 0.0f; L.diota[1] = 0.0f;
        return L;
    }
    const uint32_t bits = __float_as_uint(s);        // s >= 1 and finite: normal number
    const int k = (int)(bits >> 23) - 127;           // floor(log2 s), exact
    if (k >= n_layers - 1) {                         // reading Q5: clamp
        L.n = 1; L.lo = n_layers - 1; L.code = 0x40 | (n_layers - 1);
        L.iota[0] = 1.0f; L.diota[0] = 0.0f; L.iota[1] = 0.0f; L.diota[1] = 0.0f;
        return L;
    }
    const float m = __uint_as_float((bits & 0x007FFFFFu) | 0x3F800000u);   // s / 2^k in [1,2)
    const float inv = __uint_as_float((uint32_t)(127 - k) << 23);         // 2^-k
    L.lo = k;
    if (m == 1.0f) {                                 // reading Q2: s == 2^k
        L.n = 1; L.code = k;
        L.iota[0] = 1.0f; L.diota[0] = -inv; L.iota[1] = 0.0f; L.diota[1] = 0.0f;
        return L;
    }
    // first case of Eq. (4): 1 - |s - 2^L| / (2^(k+1) - 2^k) = 2 - m (L = k), m - 1 (L = k+1)
    L.n = 2; L.code = 0x10 | k;
    L.iota[0] = __fsub_rn(2.0f, m); L.diota[0] = -inv;
    L.iota[1] = __fsub_rn(m, 1.0f); L.diota[1] = inv;
    return L;
}

// 2^-l as an exact float
__device__ __forceinline__ float pow2_neg(int l) { return __uint_as_float((uint32_t)(127 - l) << 23); }

// Footprint of a point in layer l (Eq. 3, readings Q7, Q9): x_l = x * 2^-l; the layer is
// skipped unless -1 <= x_l < W_l and -1 <= y_l < H_l; x0 = floor(x_l), fx = x_l - x0.
struct Foot {
    int x0, y0;
    float fx, fy;
};

__device__ __forceinline__ bool footprint(float xs, float ys, int l, int Wl, int Hl, Foot& f)
{
    const float sc = pow2_neg(l);
    const float xl = __fmul_rn(xs, sc), yl = __fmul_rn(ys, sc);
    if (!(xl >= -1.0f && xl < (float)Wl && yl >= -1.0f && yl < (float)Hl)) return false;
    const float fx0 = floorf(xl), fy0 = floorf(yl);
    f.x0 = (int)fx0; f.y0 = (int)fy0;
    f.fx = __fsub_rn(xl, fx0); f.fy = __fsub_rn(yl, fy0);
    return true;
}

// (point, tile) pairs of a point: for each selected layer the tiles touched by the
// in-bounds pixels of its 2x2 footprint.  Deterministic in (xs, ys, s) so K1 (count) and
// K3 (fill) enumerate identical pairs.  Fixed slots k = 4*layer_sel + 2*dy + dx (no
// dynamic register indexing): slot k is valid iff layer_sel exists, its footprint has
// in-bounds pixels, and the footprint crosses a tile border in x (dx) / y (dy) if set.
struct PointPairs {
    int layer[2];          // layer id, -1 if absent / footprint fully out of bounds
    int x0[2], y0[2];      // footprint origin (floor(x_l), floor(y_l))
    int tx0[2], ty0[2];    // tile of the first in-bounds footprint pixel
    int sx[2], sy[2];      // 1 if the in-bounds footprint spans two tiles in x / y
    int nfrag;             // in-bounds footprint pixels over both layers (= fragments)
};

__device__ __forceinline__ PointPairs point_pairs(const Params& P, float xs, float ys, float s)
{
    PointPairs pp;
    pp.nfrag = 0;
    const Levels lv = select_levels(s, P.n_layers);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        pp.layer[k] = -1;
        pp.x0[k] = pp.y0[k] = pp.tx0[k] = pp.ty0[k] = pp.sx[k] = pp.sy[k] = 0;
        if (k >= lv.n) continue;
        const int l = lv.lo + k;
        const LayerGeom& G = P.L[l];
        Foot f;
        if (!footprint(xs, ys, l, G.W, G.H, f)) continue;
        const int xa = max(f.x0, 0), xb = min(f.x0 + 1, G.W - 1);
        const int ya = max(f.y0, 0), yb = min(f.y0 + 1, G.H - 1);
        if (xa > xb || ya > yb) continue;
        pp.layer[k] = l;
        pp.x0[k] = f.x0; pp.y0[k] = f.y0;
        pp.tx0[k] = xa >> 4; pp.ty0[k] = ya >> 4;
        pp.sx[k] = (xb >> 4) != (xa >> 4);
        pp.sy[k] = (yb >> 4) != (ya >> 4);
        pp.nfrag += (xb - xa + 1) * (yb - ya + 1);
    }
    return pp;
}

// Slot k of a point: returns the global tile id (or -1) and the footprint origin relative
// to that tile, packed as (qx0 + 1) | (qy0 + 1) << 5 with qx0, qy0 in [-1, 15].
__device__ __forceinline__ int pair_slot(const Params& P, const PointPairs& pp, int k, uint32_t& orig)
{
    const int ls = k >> 2, dy = (k >> 1) & 1, dx = k & 1;
    const int l = pp.layer[ls];
    if (l < 0 || (dx && !pp.sx[ls]) || (dy && !pp.sy[ls])) return -1;
    const LayerGeom& G = P.L[l];
    const int tx = pp.tx0[ls] + dx, ty = pp.ty0[ls] + dy;
    orig = (uint32_t)(pp.x0[ls] - tx * 16 + 1) | ((uint32_t)(pp.y0[ls] - ty * 16 + 1) << 5);
    return G.tile_base + ty * G.tiles_x + tx;
}

// Calls fn(tile, orig) for every (point, tile) pair of a point (same pairs as the slot form
// above, without evaluating empty slots): per selected layer, the tiles touched by the
// in-bounds pixels of the 2x2 footprint; orig = footprint origin relative to the tile
// ((qx0 + 1) | (qy0 + 1) << 5) and, in bits 10-13, which of the 4 corners (c = dx + 2 dy) are
// pixels of this tile inside the layer -- computed here, in the memory-bound binning pass,
// instead of per pair in the ALU-bound raster kernel.
#ifndef TRIPS_PAIR_UNROLL
#define TRIPS_PAIR_UNROLL 2
#endif
template <class Fn>
__device__ __forceinline__ void for_each_pair(const Params& P, float xs, float ys, float s, Fn&& fn)
{
    const Levels lv = select_levels(s, P.n_layers);
#if TRIPS_PAIR_UNROLL >= 2
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (k >= lv.n) break;
#else
    for (int k = 0; k < lv.n; ++k) {
#endif
        const int l = lv.lo + k;
        const LayerGeom& G = P.L[l];
        Foot f;
        if (!footprint(xs, ys, l, G.W, G.H, f)) continue;
        const int xa = max(f.x0, 0), xb = min(f.x0 + 1, G.W - 1);
        const int ya = max(f.y0, 0), yb = min(f.y0 + 1, G.H - 1);
        if (xa > xb || ya > yb) continue;
#if TRIPS_PAIR_UNROLL
        // a footprint spans at most 2 x 2 tiles: fixed-trip loops, predicated (as the layer loop)
        const int ty0 = ya >> 4, tx0 = xa >> 4, ny = (yb >> 4) - ty0, nx = (xb >> 4) - tx0;
#pragma unroll
        for (int dy = 0; dy < 2; ++dy)
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                if (dy > ny || dx > nx) continue;
                const int ty = ty0 + dy, tx = tx0 + dx;
#else
        for (int ty = ya >> 4; ty <= (yb >> 4); ++ty)
            for (int tx = xa >> 4; tx <= (xb >> 4); ++tx) {
#endif
                // columns / rows of the footprint inside [xa, xb] and this tile (separable)
                const int cxa = max(xa, tx * 16), cxb = min(xb, tx * 16 + 15);
                const int cya = max(ya, ty * 16), cyb = min(yb, ty * 16 + 15);
                const uint32_t vx = (f.x0 >= cxa ? 1u : 0u) | (f.x0 + 1 <= cxb ? 2u : 0u);
                const uint32_t vy = (f.y0 >= cya ? 1u : 0u) | (f.y0 + 1 <= cyb ? 2u : 0u);
                const uint32_t cm = ((vy & 1u) ? vx : 0u) | ((vy & 2u) ? vx << 2 : 0u);
                fn(G.tile_base + ty * G.tiles_x + tx,
                   (uint32_t)(f.x0 - tx * 16 + 1) | ((uint32_t)(f.y0 - ty * 16 + 1) << 5) | (cm << 10));
            }
    }
}

// u64 compare-exchange: (a, b) <- (min, max)
__device__ __forceinline__ void cswap(uint64_t& a, uint64_t& b)
{
    // one 64-bit compare feeding both selects (nvcc otherwise emits a second, GT, compare)
    uint64_t lo, hi;
    asm("{\n\t.reg .pred p;\n\tsetp.lt.u64 p, %2, %3;\n\tselp.b64 %0, %2, %3, p;\n\tselp.b64 %1, %3, %2, p;\n\t}"
        : "=l"(lo), "=l"(hi) : "l"(a), "l"(b));
    a = lo; b = hi;
}

// Screen record of point i for the blend / backward gathers: rb[0] = (x, y, s, alpha) from the
// per-view record, rb[1 + c] = tau[4c .. 4c+3] from the (view-independent) descriptor rows.
template <int FC>
__device__ __forceinline__ void gather_record(const Params& P, uint32_t i, float4 (&rb)[1 + FC / 4])
{
    rb[0] = __ldg(P.geo + i);
    const float4* tp = reinterpret_cast<const float4*>(P.tau + (size_t)i * FC);
#pragma unroll
    for (int c4 = 0; c4 < FC / 4; ++c4) rb[1 + c4] = __ldg(tp + c4);
}

}  // namespace trips
