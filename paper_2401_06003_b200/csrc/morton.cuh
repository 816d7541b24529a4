// morton.cuh -- one-time spatial ordering of a point cloud (trips_morton_order).
//
// Not part of the per-view rasterizer: a data-layout utility.  Every per-view stage
// gathers point records by index and accumulates gradients into per-point rows; when
// consecutive point indices are spatially close (as in MVS / LiDAR captures, and as in the
// spatially sorted batches of the software point rasterizer TRIPS builds on
// [schutz2022software]) those accesses hit the same cache lines and the same tiles.  A
// user applies the permutation once to all per-point parameters (positions, sizes,
// opacities, descriptors and their optimiser state) and trains in that order.
//
// Stable LSD radix sort (4 passes x 8 bits) of 30-bit 3-D Morton codes (10 bits per axis over
// the cloud's bounding box); non-finite points sort last.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace trips {

constexpr int kSortBlock = 4096;            // elements per radix block (256 threads x 16 rounds)

struct MortonWs {
    using Key = uint32_t;
    uint32_t* keys[2];
    uint32_t* vals[2];
    uint32_t* hist;          // [256][nblk] digit-major -> exclusive offsets
    uint32_t* bsum;          // [ceil(256 nblk / 1024)] segment totals of the histogram scan
    uint32_t* bbox;          // [6] orderable float bits: min xyz, max xyz
    int n, nblk;
    int last_pass;           // the scatter of this pass writes the values to final_vals
};

__device__ __forceinline__ uint32_t f2ord(float f)
{
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o)
{
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

template <typename WS>   // any workspace with n and bbox[6] (MortonWs, KnnWs)
__global__ void __launch_bounds__(256) k_bbox(WS W, const float* __restrict__ pos)
{
    uint32_t lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0u, 0u, 0u};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < W.n; i += gridDim.x * blockDim.x) {
        const float p[3] = {pos[3 * (size_t)i], pos[3 * (size_t)i + 1], pos[3 * (size_t)i + 2]};
        if (!isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2])) continue;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const uint32_t o = f2ord(p[a]);
            lo[a] = min(lo[a], o);
            hi[a] = max(hi[a], o);
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

__device__ __forceinline__ uint32_t spread10(uint32_t v)
{
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void __launch_bounds__(256) k_codes(MortonWs W, const float* __restrict__ pos)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= W.n) return;
    float lo[3], ext[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = ord2f(W.bbox[a]);
        ext[a] = fmaxf(ord2f(W.bbox[3 + a]) - lo[a], 1e-30f);
    }
    const float p[3] = {pos[3 * (size_t)i], pos[3 * (size_t)i + 1], pos[3 * (size_t)i + 2]};
    uint32_t code = 0xffffffffu;
    if (isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2])) {
        uint32_t q[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) q[a] = (uint32_t)fminf(fmaxf((p[a] - lo[a]) / ext[a] * 1023.0f, 0.f), 1023.f);
        code = spread10(q[0]) | (spread10(q[1]) << 1) | (spread10(q[2]) << 2);
    }
    W.keys[0][i] = code;
    W.vals[0][i] = (uint32_t)i;
}

// Radix-sort kernels (LSD, 8 bits per pass) over any workspace WS with members Key, keys[2],
// vals[2], hist, n, nblk, last_pass: MortonWs (30-bit codes, 4 passes) and KnnWs (48-bit cell
// codes, 6 passes).
template <typename WS>
__global__ void __launch_bounds__(256) k_sort_hist(WS W, int pass)
{
    __shared__ uint32_t h[256];
    const int blk = blockIdx.x;
    h[threadIdx.x] = 0;
    __syncthreads();
    const typename WS::Key* keys = W.keys[pass & 1];
    for (int j = 0; j < kSortBlock / 256; ++j) {
        const int e = blk * kSortBlock + j * 256 + threadIdx.x;
        if (e < W.n) atomicAdd(&h[(keys[e] >> (8 * pass)) & 255u], 1u);
    }
    __syncthreads();
    W.hist[(size_t)threadIdx.x * W.nblk + blk] = h[threadIdx.x];
}

// Exclusive scan of the digit-major histogram (digit d, block b) in place, in three launches:
// k_sort_scan_blocks scans 1024-entry segments and records their totals, k_sort_scan_top scans
// the totals (one CTA), k_sort_scan_add adds each segment's offset.  (A single CTA walking the
// ~500k entries at C4 size took ~0.45 ms per pass.)
__device__ __forceinline__ uint32_t sort_block_excl_scan(uint32_t v, uint32_t* ws, uint32_t* total)
{
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
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
    *total = ws[31];
    return (warp ? ws[warp - 1] : 0u) + x - v;
}

template <typename WS>
__global__ void __launch_bounds__(1024) k_sort_scan_blocks(WS W)
{
    __shared__ uint32_t ws[32];
    const int total = 256 * W.nblk;
    const int e = blockIdx.x * 1024 + threadIdx.x;
    const uint32_t v = e < total ? W.hist[e] : 0u;
    uint32_t tot;
    const uint32_t ex = sort_block_excl_scan(v, ws, &tot);
    if (e < total) W.hist[e] = ex;
    if (threadIdx.x == 0) W.bsum[blockIdx.x] = tot;
}

template <typename WS>
__global__ void __launch_bounds__(1024) k_sort_scan_top(WS W)
{
    __shared__ uint32_t ws[32];
    const int nseg = (256 * W.nblk + 1023) / 1024;
    uint32_t carry = 0;
    for (int base = 0; base < nseg; base += 1024) {
        const int e = base + threadIdx.x;
        const uint32_t v = e < nseg ? W.bsum[e] : 0u;
        uint32_t tot;
        const uint32_t ex = sort_block_excl_scan(v, ws, &tot);
        if (e < nseg) W.bsum[e] = carry + ex;
        carry += tot;
        __syncthreads();
    }
}

template <typename WS>
__global__ void __launch_bounds__(1024) k_sort_scan_add(WS W)
{
    const int total = 256 * W.nblk;
    const int e = blockIdx.x * 1024 + threadIdx.x;
    if (e < total) W.hist[e] += W.bsum[blockIdx.x];
}

// Stable scatter: rounds of 256 consecutive elements; rank = elements of the same digit in
// earlier rounds + earlier warps of this round + earlier lanes of this warp.
template <typename WS>
__global__ void __launch_bounds__(256) k_sort_scatter(WS W, int pass, uint32_t* final_vals)
{
    __shared__ uint32_t base[256];           // next output position per digit
    __shared__ uint32_t wcnt[8][256];
    const int blk = blockIdx.x;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    base[threadIdx.x] = W.hist[(size_t)threadIdx.x * W.nblk + blk];
    using Key = typename WS::Key;
    const Key* kin = W.keys[pass & 1];
    const uint32_t* vin = W.vals[pass & 1];
    Key* kout = W.keys[(pass + 1) & 1];
    uint32_t* vout = (pass == W.last_pass && final_vals) ? final_vals : W.vals[(pass + 1) & 1];
    for (int j = 0; j < kSortBlock / 256; ++j) {
#pragma unroll
        for (int w = 0; w < 8; ++w) wcnt[w][threadIdx.x] = 0;
        __syncthreads();
        const int e = blk * kSortBlock + j * 256 + threadIdx.x;
        const bool ok = e < W.n;
        const Key k = ok ? kin[e] : Key(0);
        const int d = ok ? (int)((k >> (8 * pass)) & 255u) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (ok && lane == (unsigned)(__ffs(peers) - 1)) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        if (ok) {
            uint32_t pre = 0;
            for (int w = 0; w < (int)warp; ++w) pre += wcnt[w][d];
            const uint32_t p = base[d] + pre + __popc(peers & ((1u << lane) - 1u));
            kout[p] = k;
            vout[p] = vin[e];
        }
        __syncthreads();
        uint32_t add = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) add += wcnt[w][threadIdx.x];
        base[threadIdx.x] += add;
        __syncthreads();
    }
}

}  // namespace trips
