// knn.cuh -- point-size initialisation with the mean distance to the 4 nearest neighbours
// ("Point sizes are initialized with the average distance to the four nearest
// neighbor"; reading Q25 in DESIGN.md).
//
// Exact k-NN on a Morton-sorted cloud, sized by the data rather than by the bounding box (the
// uniform grid of round 1 assumed volumetric density: on a surface cloud its cells held hundreds
// of points and a query scanned thousands):
//   1. 45-bit Morton codes of the points quantised to 2^15 steps per axis over the bounding cube
//      (non-finite points get a code above every finite one), stable LSD radix sort (6 x 8 bits,
//      morton.cuh's kernels), points gathered into sorted order;
//   2. one thread per sorted position (so a warp's queries are spatial neighbours): a register
//      top-4 of (d^2, j) over the +-kKnnWin neighbours in sorted order gives an upper bound r on
//      the 4th distance; the box of half-width r (widened for rounding) around the point is a
//      Z-order range query on the sorted codes: scan [code(box min), code(box max)] from a
//      galloping lower_bound, test each code's axis bits against the box, and jump over the
//      stretches of the curve outside it with BIGMIN (Tropf & Herzog) + lower_bound (window
//      positions skipped: already considered).
// Every point j with (d^2, j) below the window's 4th key lies in the box, so the top-4 is exact;
// d^2 and the mean use the pinned fp32 sequence of the definition, so results are bit-identical
// to a brute-force evaluation (tests/test_gpu_knn.py).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "morton.cuh"

namespace trips {

constexpr int kKnnBits = 15;                  // quantisation steps per axis: 2^15
constexpr int kKnnPasses = 6;                 // 45-bit codes + the non-finite marker's bit 47
constexpr uint64_t kKnnNonFinite = (1ull << 48) - 1;
#ifndef TRIPS_KNN_UNION
#define TRIPS_KNN_UNION 6          // warp mode when the union box is <= this x the largest lane box (+64 steps)
#endif
#ifndef TRIPS_KNN_GROUP
#define TRIPS_KNN_GROUP 32         // lanes whose queries share one union box (power of 2; 4 / 8 / 16 measured slower)
#endif
constexpr int kKnnGroup = TRIPS_KNN_GROUP;
#ifndef TRIPS_KNN_WIN
#define TRIPS_KNN_WIN 8
#endif
constexpr int kKnnWin = TRIPS_KNN_WIN;                    // sorted-order neighbours on each side for the bound

struct KnnWs {
    using Key = uint64_t;
    uint64_t* keys[2];        // [n] codes (sorted into keys[0] after the even number of passes)
    uint32_t* vals[2];        // [n] point index (sorted into vals[0])
    uint32_t* hist;           // [256][nblk]
    uint32_t* bsum;           // [ceil(256 nblk / 1024)] segment totals of the histogram scan
    uint32_t* bbox;           // [6] orderable float bits (min xyz, max xyz) of the finite points
    uint32_t* nfin;           // [1] finite points (they sort first)
    float4* pts;              // [n] (x, y, z, index bits) in sorted order
    int n, nblk, last_pass;
};

#ifdef TRIPS_KNN_STATS    // experiment builds only: candidates, lower_bound steps, BIGMIN jumps, boxes
__device__ unsigned long long g_knn_stats[4];
#define TRIPS_KNN_COUNT(k, v) atomicAdd(&g_knn_stats[k], (unsigned long long)(v))
#else
#define TRIPS_KNN_COUNT(k, v) (void)0
#endif

struct KnnQuant {
    double lo[3];
    double scale;             // steps per unit (0 for a single-point extent)
};

__device__ __forceinline__ KnnQuant knn_quant(const uint32_t* bbox)
{
    KnnQuant Q;
    double ext = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const bool any = bbox[a] != 0xffffffffu;
        Q.lo[a] = any ? (double)ord2f(bbox[a]) : 0.0;
        const double hi = any ? (double)ord2f(bbox[3 + a]) : 0.0;
        ext = fmax(ext, hi - Q.lo[a]);
    }
    Q.scale = ext > 0.0 ? (double)(1 << kKnnBits) / ext : 0.0;
    return Q;
}

// quantised coordinate, clamped to [0, 2^kKnnBits - 1] (monotone in v)
__device__ __forceinline__ int knn_q(double v, double lo, double scale)
{
    const double t = floor((v - lo) * scale);
    return t < 0.0 ? 0 : (t > (double)((1 << kKnnBits) - 1) ? (1 << kKnnBits) - 1 : (int)t);
}

__device__ __forceinline__ uint64_t knn_spread(uint32_t v)
{
    uint64_t x = v & 0x1fffffu;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

__device__ __forceinline__ uint64_t knn_code(int qx, int qy, int qz)
{
    return knn_spread((uint32_t)qx) | (knn_spread((uint32_t)qy) << 1) | (knn_spread((uint32_t)qz) << 2);
}

__device__ __forceinline__ bool finite3(float x, float y, float z) { return isfinite(x) && isfinite(y) && isfinite(z); }

__global__ void __launch_bounds__(256) k_knn_codes(KnnWs W, const float* __restrict__ pos)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const KnnQuant Q = knn_quant(W.bbox);
    bool fin = false;
    if (i < W.n) {
        const float x = pos[3 * (size_t)i], y = pos[3 * (size_t)i + 1], z = pos[3 * (size_t)i + 2];
        fin = finite3(x, y, z);
        W.keys[0][i] = fin ? knn_code(knn_q(x, Q.lo[0], Q.scale), knn_q(y, Q.lo[1], Q.scale), knn_q(z, Q.lo[2], Q.scale))
                           : kKnnNonFinite;
        W.vals[0][i] = (uint32_t)i;
    }
    const uint32_t c = __reduce_add_sync(0xffffffffu, fin ? 1u : 0u);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(W.nfin, c);
}

__global__ void __launch_bounds__(256) k_knn_gather(KnnWs W, const float* __restrict__ pos)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= W.n) return;
    const uint32_t i = W.vals[0][k];
    W.pts[k] = make_float4(pos[3 * (size_t)i], pos[3 * (size_t)i + 1], pos[3 * (size_t)i + 2], __uint_as_float(i));
}

// (d2, j) insertion into an ascending register top-4 (lexicographic; j breaks ties)
__device__ __forceinline__ void knn_insert(float (&bd)[4], uint32_t (&bj)[4], float d2, uint32_t j)
{
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const bool lt = d2 < bd[k] || (d2 == bd[k] && j < bj[k]);
        const float td = bd[k];
        const uint32_t tj = bj[k];
        bd[k] = lt ? d2 : td;
        bj[k] = lt ? j : tj;
        d2 = lt ? td : d2;
        j = lt ? tj : j;
    }
}

// first position in [0, nf) whose code is >= c (codes sorted ascending), galloping from `hint`
__device__ __forceinline__ int knn_lower_bound(const uint64_t* __restrict__ codes, int nf, uint64_t c, int hint)
{
    int lo, hi;                                      // answer in (lo, hi]: codes[lo] < c <= codes[hi]
    if (codes[hint] < c) {
        lo = hint;
        int step = 1;
        for (;;) {
            const int p = hint + step;
            if (p >= nf) { hi = nf; break; }
            if (codes[p] >= c) { hi = p; break; }
            lo = p;
            step <<= 1;
        }
    } else {
        hi = hint;
        int step = 1;
        for (;;) {
            const int p = hint - step;
            if (p < 0) { lo = -1; break; }
            if (codes[p] < c) { lo = p; break; }
            hi = p;
            step <<= 1;
        }
    }
    while (hi - lo > 1) {
        const int mid = lo + ((hi - lo) >> 1);
        if (codes[mid] < c) lo = mid; else hi = mid;
    }
    return hi;
}

// Per-axis bits of interleaved codes: masking keeps each axis' order, so a code is inside the
// box [zmin, zmax] (corner codes) iff every axis' masked bits lie between the corners' ones.
constexpr uint64_t kKnnAxis = 0x1249249249249249ull;
__device__ __forceinline__ bool knn_in_box(uint64_t c, uint64_t zmin, uint64_t zmax)
{
    bool in = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const uint64_t m = kKnnAxis << a;
        in = in && (c & m) >= (zmin & m) && (c & m) <= (zmax & m);
    }
    return in;
}

// BIGMIN (Tropf & Herzog, 1981): the smallest code > c inside the box [zmin, zmax], for c inside
// [zmin, zmax] as a number but outside the box; ~0 if there is none.  Walks the bits from the
// top: where c, zmin and zmax disagree it either returns or narrows the box to the half that
// can still hold codes above c ("load 1000" / "load 0111" on that axis' lower bits).
__device__ __forceinline__ uint64_t knn_bigmin(uint64_t c, uint64_t zmin, uint64_t zmax)
{
    uint64_t big = ~0ull;
    // above the highest bit where the corners differ, c, zmin and zmax agree (zmin <= c <= zmax):
    // nothing to do there
    for (int b = 63 - __clzll(zmin ^ zmax); b >= 0; --b) {
        const uint64_t m = 1ull << b;
        const uint64_t axis = kKnnAxis << (b % 3);
        const uint64_t low = axis & (m - 1);             // this axis' bits below b
        const uint64_t at = low | m;                     // ... and b itself
        const int code = ((c & m) ? 4 : 0) | ((zmin & m) ? 2 : 0) | ((zmax & m) ? 1 : 0);
        if (code == 1) {                                 // c 0, min 0, max 1
            big = (zmin & ~at) | m;
            zmax = (zmax & ~at) | low;
        } else if (code == 3) {                          // c 0, min 1, max 1
            return zmin;
        } else if (code == 4) {                          // c 1, min 0, max 0
            return big;
        } else if (code == 5) {                          // c 1, min 0, max 1
            zmin = (zmin & ~at) | m;
        } else if (code == 2 || code == 6) {             // min > max on this axis: cannot happen
            return big;
        }
    }
    return big;
}

__global__ void __launch_bounds__(256) k_knn_query(KnnWs W, float* __restrict__ size_out, int32_t* __restrict__ nbr_out)
{
    constexpr unsigned kAll = 0xffffffffu;
    __shared__ float4 s_stage[8][32];                // per warp: in-box points of one 32-position step
    __shared__ int s_spos[8][32];
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool live = k < W.n;                       // no early return: the warp cooperates below
    const int nf = (int)*W.nfin;
    const uint64_t* __restrict__ codes = W.keys[0];
    const float4* __restrict__ pts = W.pts;
    const float4 p = live ? pts[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    const uint32_t i = __float_as_uint(p.w);
    float bd[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
    uint32_t bj[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
    int nb = 0;
    auto cand_pt = [&](float qx, float qy, float qz, uint32_t jj) {
        const float ddx = __fsub_rn(qx, p.x), ddy = __fsub_rn(qy, p.y), ddz = __fsub_rn(qz, p.z);
        float d2 = __fadd_rn(__fmul_rn(ddx, ddx), __fmul_rn(ddy, ddy));
        d2 = __fadd_rn(d2, __fmul_rn(ddz, ddz));
        ++nb;
        TRIPS_KNN_COUNT(0, 1);
        if (d2 < bd[3] || (d2 == bd[3] && jj < bj[3])) knn_insert(bd, bj, d2, jj);
    };
    auto cand = [&](int j) {
        const float4 q = pts[j];
        cand_pt(q.x, q.y, q.z, __float_as_uint(q.w));
    };
    const bool fin = live && k < nf;
    const int w0 = max(0, k - kKnnWin), w1 = min(nf - 1, k + kKnnWin);
    if (fin)
        for (int j = w0; j <= w1; ++j)
            if (j != k) cand(j);
    // the window holds >= kKnnWin >= 4 others unless it covers every finite point, so bd[3] is
    // finite: every point with a smaller (d^2, j) key lies within r of p (fp32 rounding of d^2
    // covered by the factor), hence inside the quantised box [qlo, qhi] (+-1 step for the
    // quantisation rounding)
    const bool need = fin && (w0 > 0 || w1 < nf - 1);
    int qlo[3] = {0, 0, 0}, qhi[3] = {-1, -1, -1};
    if (need) {
        const KnnQuant Q = knn_quant(W.bbox);
        const double r = sqrt((double)bd[3]) * (1.0 + 1e-5);
        const double pp[3] = {p.x, p.y, p.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            qlo[a] = max(0, knn_q(pp[a] - r, Q.lo[a], Q.scale) - 1);
            qhi[a] = min((1 << kKnnBits) - 1, knn_q(pp[a] + r, Q.lo[a], Q.scale) + 1);
        }
        TRIPS_KNN_COUNT(3, 1);
        TRIPS_KNN_COUNT(1, (uint64_t)(qhi[0] - qlo[0] + 1) * (uint64_t)(qhi[1] - qlo[1] + 1));
    }
    // Warp mode: the 32 queries of a warp are neighbours on the curve, so their boxes overlap.
    // When the union box is compact the warp scans it once, cooperatively (octree cells located in
    // parallel, then 32 consecutive sorted positions per step, coalesced, each in-box point
    // broadcast to every lane).  Otherwise (the warp straddles a far jump of the curve) each lane
    // scans its own box with BIGMIN jumps.  Either way every point of a lane's box is evaluated exactly once (window
    // positions skipped), so the top-4 is exact.
    // groups of kKnnGroup lanes (consecutive sorted positions) cooperate; all sync operations use
    // the group's mask, so the groups of a warp run independently
    constexpr int G = kKnnGroup;
    const int gl = lane & (G - 1), gbase = lane - gl;
    const unsigned gmask = (G == 32) ? kAll : (((1u << G) - 1u) << gbase);
    const unsigned act = __ballot_sync(kAll, need) & gmask;
    if (act) {
        int ulo[3], uhi[3], lext = 0, uext = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            ulo[a] = __reduce_min_sync(gmask, need ? qlo[a] : (1 << kKnnBits));
            uhi[a] = __reduce_max_sync(gmask, need ? qhi[a] : -1);
            lext = max(lext, qhi[a] - qlo[a]);
            uext = max(uext, uhi[a] - ulo[a]);
        }
        lext = __reduce_max_sync(gmask, need ? lext : 0);
        if (uext <= TRIPS_KNN_UNION * lext + 64) {
            // the union box is covered by <= 3 x 3 x 3 aligned octree cells of the smallest size that
            // spans it in 3; each cell is one contiguous code range of the sorted array, located by a
            // lane of the group (parallel lower_bounds); the group then sweeps the cells' ranges G
            // positions at a time, broadcasting the in-box points through shared memory
            const uint64_t zmin = knn_code(ulo[0], ulo[1], ulo[2]), zmax = knn_code(uhi[0], uhi[1], uhi[2]);
            int sh = 0;
            while (sh < kKnnBits && ((uhi[0] >> sh) - (ulo[0] >> sh) > 2 || (uhi[1] >> sh) - (ulo[1] >> sh) > 2 ||
                                     (uhi[2] >> sh) - (ulo[2] >> sh) > 2))
                ++sh;
            const int nx = (uhi[0] >> sh) - (ulo[0] >> sh) + 1, ny = (uhi[1] >> sh) - (ulo[1] >> sh) + 1;
            const int ncell = nx * ny * ((uhi[2] >> sh) - (ulo[2] >> sh) + 1);
            const int k0 = __shfl_sync(gmask, k, __ffs(act) - 1);
            float4* stage = s_stage[threadIdx.x >> 5] + gbase;
            int* spos = s_spos[threadIdx.x >> 5] + gbase;
            constexpr int kRounds = (27 + G - 1) / G;
            int ca[kRounds], cb[kRounds];                            // this lane's cells: [ca, cb)
#pragma unroll
            for (int rr = 0; rr < kRounds; ++rr) {
                ca[rr] = 0;
                cb[rr] = 0;
                const int c = gl + rr * G;
                if (c < ncell) {
                    const int cx = (ulo[0] >> sh) + c % nx, cy = (ulo[1] >> sh) + (c / nx) % ny;
                    const int cz = (ulo[2] >> sh) + c / (nx * ny);
                    const uint64_t base = knn_code(cx << sh, cy << sh, cz << sh);
                    ca[rr] = knn_lower_bound(codes, nf, base, k0);
                    cb[rr] = knn_lower_bound(codes, nf, base + (1ull << (3 * sh)), ca[rr] < nf ? ca[rr] : nf - 1);
                    TRIPS_KNN_COUNT(2, 1);
                }
            }
            for (int cc = 0; cc < ncell; ++cc) {
                int va = 0, vb = 0;
#pragma unroll
                for (int rr = 0; rr < kRounds; ++rr)
                    if (cc / G == rr) { va = ca[rr]; vb = cb[rr]; }
                const int a = __shfl_sync(gmask, va, gbase + cc % G), b = __shfl_sync(gmask, vb, gbase + cc % G);
                for (int j = a; j < b; j += G) {
                    // the in-box points of these G positions are compacted into the group's stage
                    // and read back by every lane of the group (broadcast loads)
                    const int pos = j + gl;
                    const bool inb = pos < b && knn_in_box(codes[pos], zmin, zmax);
                    const unsigned m = (__ballot_sync(gmask, inb) & gmask) >> gbase;
                    if (inb) {
                        const int slot = __popc(m & ((1u << gl) - 1u));
                        stage[slot] = pts[pos];
                        spos[slot] = pos;
                    }
                    __syncwarp(gmask);
                    const int cnt = __popc(m);
                    for (int e = 0; e < cnt; ++e) {
                        const float4 q = stage[e];
                        const int pb = spos[e];
                        if (need && pb != k && (pb < w0 || pb > w1)) cand_pt(q.x, q.y, q.z, __float_as_uint(q.w));
                    }
                    __syncwarp(gmask);
                }
            }
        } else if (need) {
            TRIPS_KNN_COUNT(3, 1000000);                     // (stats builds: fallback lanes, x 1e6)
            // this lane's own box: scan [code(qlo), code(qhi)], jumping over the stretches of the
            // curve outside the box with BIGMIN (the next code >= c inside the box)
            const uint64_t zmin = knn_code(qlo[0], qlo[1], qlo[2]), zmax = knn_code(qhi[0], qhi[1], qhi[2]);
            int j = knn_lower_bound(codes, nf, zmin, k);
            while (j < nf) {
                const uint64_t c = codes[j];
                if (c > zmax) break;
                if (knn_in_box(c, zmin, zmax)) {
                    if (j < w0 || j > w1) cand(j);
                    ++j;
                } else {
                    const uint64_t bm = knn_bigmin(c, zmin, zmax);
                    TRIPS_KNN_COUNT(2, 1);
                    if (bm == ~0ull) break;
                    j = knn_lower_bound(codes, nf, bm, j);
                }
            }
        }
    }
    if (!live) return;
    const int K = nb < 4 ? nb : 4;
    float sz = 0.f;
#pragma unroll
    for (int m = 0; m < 4; ++m)
        if (m < K) sz = __fadd_rn(sz, __fsqrt_rn(bd[m]));
    size_out[i] = K ? __fdiv_rn(sz, (float)K) : 0.f;
    if (nbr_out)
#pragma unroll
        for (int m = 0; m < 4; ++m) nbr_out[4 * (size_t)i + m] = m < K ? (int32_t)bj[m] : -1;
}

}  // namespace trips
