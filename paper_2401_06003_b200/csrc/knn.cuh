// knn.cuh -- point-size initialisation with the mean distance to the 4 nearest neighbours
// ("Point sizes are initialized with the average distance to the four nearest
// neighbor"; reading Q25 in DESIGN.md).
//
// Uniform grid over the cloud's bounding box (about one point per cell), points bucketed per
// cell (count, scan, fill), then one thread per point searches cells ring by ring around its
// own cell with a register top-4 of (d^2, j) and stops once every point outside the scanned
// cube is provably farther than its 4th neighbour.  d^2 and the mean use the pinned fp32
// sequence of the definition, so results are bit-identical to a brute-force evaluation.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace trips {

struct KnnGrid {
    float lo[3];
    float h, inv_h;
    int dim[3];
    int ncell;
};

struct KnnWs {
    int n, cap;               // points, cell capacity (>= ncell)
    uint32_t* bbox;           // [6] orderable float bits (min xyz, max xyz)
    KnnGrid* grid;            // [1]
    uint32_t* cell_of;        // [n]  cell of each point (0xffffffff: not finite)
    uint32_t* cnt;            // [cap + 1] counts -> exclusive offsets
    uint32_t* cur;            // [cap]  fill cursors
    uint32_t* bsum;           // [blocks] scan partials
    float4* pts;              // [n]  (x, y, z, index bits) in cell order
};

__device__ __forceinline__ uint32_t knn_f2ord(float f)
{
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float knn_ord2f(uint32_t o)
{
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__device__ __forceinline__ bool finite3(float x, float y, float z) { return isfinite(x) && isfinite(y) && isfinite(z); }

__global__ void __launch_bounds__(256) k_knn_bbox(KnnWs W, const float* __restrict__ pos)
{
    uint32_t lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0u, 0u, 0u};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < W.n; i += gridDim.x * blockDim.x) {
        const float x = pos[3 * (size_t)i], y = pos[3 * (size_t)i + 1], z = pos[3 * (size_t)i + 2];
        if (!finite3(x, y, z)) continue;
        const float p[3] = {x, y, z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = min(lo[a], knn_f2ord(p[a]));
            hi[a] = max(hi[a], knn_f2ord(p[a]));
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = __reduce_min_sync(0xffffffffu, lo[a]);
        hi[a] = __reduce_max_sync(0xffffffffu, hi[a]);
    }
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(&W.bbox[a], lo[a]);
            atomicMax(&W.bbox[3 + a], hi[a]);
        }
}

// one thread: grid of about one point per cell, at most `cap` cells, at most 2048 per axis
__global__ void k_knn_setup(KnnWs W)
{
    KnnGrid g;
    double ext[3], vol = 1.0, emax = 0.0;
    for (int a = 0; a < 3; ++a) {
        const float lo = W.bbox[a] == 0xffffffffu ? 0.f : knn_ord2f(W.bbox[a]);
        const float hi = W.bbox[a] == 0xffffffffu ? 0.f : knn_ord2f(W.bbox[3 + a]);
        g.lo[a] = lo;
        ext[a] = (double)hi - (double)lo;
        emax = fmax(emax, ext[a]);
    }
    for (int a = 0; a < 3; ++a) vol *= fmax(ext[a], emax * 1e-3 + 1e-30);
    double h = cbrt(vol / fmax((double)W.n, 1.0));
    h = fmax(h, emax / 2048.0);
    h = fmax(h, 1e-30);
    for (int it = 0; it < 64; ++it) {
        double cells = 1.0;
        for (int a = 0; a < 3; ++a) {
            g.dim[a] = (int)fmin(floor(ext[a] / h) + 1.0, 2048.0);
            cells *= g.dim[a];
        }
        if (cells <= (double)W.cap) break;
        h *= 1.26;
    }
    g.h = (float)h;
    g.inv_h = (float)(1.0 / h);
    g.ncell = g.dim[0] * g.dim[1] * g.dim[2];
    *W.grid = g;
}

__device__ __forceinline__ int knn_cell_axis(float v, float lo, float inv_h, int dim)
{
    const int c = (int)floorf((v - lo) * inv_h);
    return c < 0 ? 0 : (c >= dim ? dim - 1 : c);
}

__global__ void __launch_bounds__(256) k_knn_count(KnnWs W, const float* __restrict__ pos)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= W.n) return;
    const KnnGrid g = *W.grid;
    const float x = pos[3 * (size_t)i], y = pos[3 * (size_t)i + 1], z = pos[3 * (size_t)i + 2];
    uint32_t c = 0xffffffffu;
    if (finite3(x, y, z)) {
        const int cx = knn_cell_axis(x, g.lo[0], g.inv_h, g.dim[0]);
        const int cy = knn_cell_axis(y, g.lo[1], g.inv_h, g.dim[1]);
        const int cz = knn_cell_axis(z, g.lo[2], g.inv_h, g.dim[2]);
        c = (uint32_t)((cz * g.dim[1] + cy) * g.dim[0] + cx);
        atomicAdd(&W.cnt[c], 1u);
    }
    W.cell_of[i] = c;
}

// two-level exclusive scan of cnt[0..ncell): per-block sums, then offsets
__global__ void __launch_bounds__(1024) k_knn_scan_a(KnnWs W)
{
    __shared__ uint32_t ws[32];
    const int ncell = W.grid->ncell;
    const int e = blockIdx.x * 1024 + threadIdx.x;
    uint32_t v = e < ncell ? W.cnt[e] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int w = 0; w < 32; ++w) s += ws[w];
        W.bsum[blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(1024) k_knn_scan_b(KnnWs W)
{
    // one CTA: exclusive scan of the block sums (in place)
    __shared__ uint32_t ws[32];
    const int nb = (W.grid->ncell + 1023) / 1024;
    uint32_t carry = 0;
    for (int base = 0; base < nb; base += 1024) {
        const int b = base + threadIdx.x;
        const uint32_t v = b < nb ? W.bsum[b] : 0u;
        uint32_t x = v;
        const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (unsigned)o) x += y;
        }
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = ws[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= (unsigned)o) w += y;
            }
            ws[lane] = w;
        }
        __syncthreads();
        if (b < nb) W.bsum[b] = carry + (warp ? ws[warp - 1] : 0u) + x - v;
        carry += ws[31];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(1024) k_knn_scan_c(KnnWs W)
{
    __shared__ uint32_t ws[32];
    const int ncell = W.grid->ncell;
    const int e = blockIdx.x * 1024 + threadIdx.x;
    const uint32_t v = e < ncell ? W.cnt[e] : 0u;
    uint32_t x = v;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = ws[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (unsigned)o) w += y;
        }
        ws[lane] = w;
    }
    __syncthreads();
    const uint32_t off = W.bsum[blockIdx.x] + (warp ? ws[warp - 1] : 0u) + x - v;
    if (e < ncell) {
        W.cnt[e] = off;
        W.cur[e] = off;
    }
    if (e == ncell - 1) W.cnt[ncell] = off + v;
}

__global__ void __launch_bounds__(256) k_knn_fill(KnnWs W, const float* __restrict__ pos)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= W.n) return;
    const uint32_t c = W.cell_of[i];
    if (c == 0xffffffffu) return;
    const uint32_t p = atomicAdd(&W.cur[c], 1u);
    W.pts[p] = make_float4(pos[3 * (size_t)i], pos[3 * (size_t)i + 1], pos[3 * (size_t)i + 2],
                           __uint_as_float((uint32_t)i));
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

__global__ void __launch_bounds__(256) k_knn_query(KnnWs W, const float* __restrict__ pos, float* __restrict__ size_out,
                                                   int32_t* __restrict__ nbr_out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= W.n) return;
    const KnnGrid g = *W.grid;
    const uint32_t ci = W.cell_of[i];
    float bd[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
    uint32_t bj[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
    int nb = 0;
    if (ci != 0xffffffffu) {
        const float x = pos[3 * (size_t)i], y = pos[3 * (size_t)i + 1], z = pos[3 * (size_t)i + 2];
        const int cx = (int)(ci % (uint32_t)g.dim[0]);
        const int cy = (int)((ci / (uint32_t)g.dim[0]) % (uint32_t)g.dim[1]);
        const int cz = (int)(ci / ((uint32_t)g.dim[0] * (uint32_t)g.dim[1]));
        const int rmax = max(g.dim[0], max(g.dim[1], g.dim[2]));
        for (int r = 0; r <= rmax; ++r) {
            for (int dz = -r; dz <= r; ++dz) {
                const int zz = cz + dz;
                if (zz < 0 || zz >= g.dim[2]) continue;
                for (int dy = -r; dy <= r; ++dy) {
                    const int yy = cy + dy;
                    if (yy < 0 || yy >= g.dim[1]) continue;
                    const bool face = (dz == -r || dz == r || dy == -r || dy == r);
                    for (int dx = -r; dx <= r; dx += (face || r == 0) ? 1 : 2 * r) {
                        const int xx = cx + dx;
                        if (xx < 0 || xx >= g.dim[0]) continue;
                        const uint32_t c = (uint32_t)((zz * g.dim[1] + yy) * g.dim[0] + xx);
                        const uint32_t b = W.cnt[c], e = W.cnt[c + 1];
                        for (uint32_t k = b; k < e; ++k) {
                            const float4 q = W.pts[k];
                            const uint32_t j = __float_as_uint(q.w);
                            if (j == (uint32_t)i) continue;
                            const float ddx = __fsub_rn(q.x, x), ddy = __fsub_rn(q.y, y), ddz = __fsub_rn(q.z, z);
                            float d2 = __fadd_rn(__fmul_rn(ddx, ddx), __fmul_rn(ddy, ddy));
                            d2 = __fadd_rn(d2, __fmul_rn(ddz, ddz));
                            ++nb;
                            if (d2 < bd[3] || (d2 == bd[3] && j < bj[3])) knn_insert(bd, bj, d2, j);
                        }
                    }
                }
            }
            // every point outside the scanned cube is at least `gap` away
            double gap = 1e300;
            const int cc[3] = {cx, cy, cz};
            const float pp[3] = {x, y, z};
            bool covers_all = true;
            for (int a = 0; a < 3; ++a) {
                const double lo_face = (double)g.lo[a] + (double)(cc[a] - r) * g.h;
                const double hi_face = (double)g.lo[a] + (double)(cc[a] + r + 1) * g.h;
                if (cc[a] - r > 0) gap = fmin(gap, (double)pp[a] - lo_face);
                if (cc[a] + r + 1 < g.dim[a]) gap = fmin(gap, hi_face - (double)pp[a]);
                if (cc[a] - r > 0 || cc[a] + r + 1 < g.dim[a]) covers_all = false;
            }
            if (covers_all) break;
            gap -= 1e-4 * g.h;                                 // cell-assignment rounding margin
            if (nb >= 4 && gap > 0 && (double)bd[3] < gap * gap * (1.0 - 1e-5)) break;
        }
    }
    const int K = nb < 4 ? nb : 4;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (k < K) s = __fadd_rn(s, __fsqrt_rn(bd[k]));
    size_out[i] = K ? __fdiv_rn(s, (float)K) : 0.f;
    if (nbr_out)
#pragma unroll
        for (int k = 0; k < 4; ++k) nbr_out[4 * (size_t)i + k] = k < K ? (int32_t)bj[k] : -1;
}

}  // namespace trips
