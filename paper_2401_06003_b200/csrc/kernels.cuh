// kernels.cuh -- rasterization and backward kernels of the B200 TRIPS rasterizer
// (DESIGN.md "Kernels"); binning.cuh holds the collecting/splatting stages.
//
//   k_raster   per tile (CTA of 256 = 16x16 pixel threads): streams the tile's (point, tile)
//              pairs in chunks, builds the per-pixel fragment lists in shared memory
//              (counting sort by pixel), keeps the 16 smallest (z, i) keys per pixel in
//              registers with Batcher odd-even sorting/merging networks, blends front to back
//              and stores the sorted kept lists and their gamma.
//                                                 ("combined sorting and accumulation", 290-295)
//   k_backward per tile pixel: T_m from the saved gamma_m, reverse replay with suffix
//              recurrences, screen -> world chain per fragment, 16-byte vector reductions
//              (red.global.add.v4.f32) into the packed gradient rows.
#pragma once
#include "binning.cuh"

namespace trips {

#ifndef TRIPS_CHUNK
#define TRIPS_CHUNK 1024
#endif
#ifndef TRIPS_BLEND_BATCH
#define TRIPS_BLEND_BATCH 4
#endif
#ifndef TRIPS_RASTER_CTAS
#define TRIPS_RASTER_CTAS 3
#endif
#ifndef TRIPS_THR_SKIP0
#define TRIPS_THR_SKIP0 1
#endif
#ifndef TRIPS_BLEND_REG
#define TRIPS_BLEND_REG 0
#endif
#ifndef TRIPS_PF_UNROLL
#define TRIPS_PF_UNROLL 2
#endif

#ifndef TRIPS_RED_CLOBBER
#define TRIPS_RED_CLOBBER 1
#endif
#ifndef TRIPS_BWD_CTAS
#define TRIPS_BWD_CTAS 4
#endif
constexpr int kChunk = TRIPS_CHUNK;         // (point, tile) pairs staged per K4 iteration
constexpr int kPairsPerThread = kChunk / kTilePix;
constexpr int kPfUnroll = TRIPS_PF_UNROLL;      // bin pairs loaded together in k_raster phase F
#ifndef TRIPS_BWD_SLOTS
#define TRIPS_BWD_SLOTS 4
#endif
constexpr int kBwdSlots = TRIPS_BWD_SLOTS;      // kept pairs per thread held in registers across k_backward_pairs' phases
#ifndef TRIPS_BWD_BATCH
#define TRIPS_BWD_BATCH 4
#endif
constexpr int kBatch = TRIPS_BWD_BATCH;     // record gathers issued together (memory-level parallelism)
constexpr int kBlendBatch = TRIPS_BLEND_BATCH;  // same in k_raster's blend (register budget: 3 CTAs/SM)
// wide descriptors hold FC / 4 float4 per gathered record: fewer records in flight keeps them in
// registers (F > 8 spilled kilobytes per thread at the F = 4 batch sizes)
template <int FC> __host__ __device__ constexpr int blend_batch() { return FC <= 8 ? kBlendBatch : (FC <= 16 ? 2 : 1); }
template <int FC> __host__ __device__ constexpr int bwd_slots() { return FC <= 8 ? kBwdSlots : (FC <= 16 ? 2 : 1); }

// Experiment builds only (-DTRIPS_PHASE_CLOCK): per-phase clock64 accumulation of k_raster
// (thread 0 of each CTA, after a barrier), read with trips_debug_phase_clocks().
#ifdef TRIPS_PHASE_CLOCK
__device__ unsigned long long g_pclk[8];
#define TRIPS_PCLK_START long long _pc_t = clock64()
#define TRIPS_PCLK(k)                                                                            \
    do {                                                                                         \
        __syncthreads();                                                                         \
        if (threadIdx.x == 0) {                                                                  \
            const long long _n = clock64();                                                      \
            atomicAdd(&g_pclk[k], (unsigned long long)(_n - _pc_t));                             \
            _pc_t = _n;                                                                          \
        }                                                                                        \
    } while (0)
#else
#define TRIPS_PCLK_START (void)0
#define TRIPS_PCLK(k) (void)0
#endif

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d)
{
#ifdef TRIPS_EXP_NORED      // experiment builds only (tools/variants.sh): measure without the reductions
    if (a == 1.2345e-38f) *addr = b + c + d;
#elif TRIPS_RED_CLOBBER
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
                 :: "l"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
#else
    // no "memory" clobber: nothing in the kernel reads the gradient rows, so the compiler may
    // move the next fragments' record loads above these reductions
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
                 :: "l"(addr), "f"(a), "f"(b), "f"(c), "f"(d));
#endif
}

// --------------------------------------------------------------------------- networks

// Sorting networks (ascending) on t[0..N), verified exhaustively with the 0-1 principle
// (tests/test_networks.py): 5 comparators for 4 keys, 19 for 8 (Batcher odd-even merge sort),
// 39 for 12 and 60 for 16 (the best known sizes; TRIPS_NET16 = 0 selects Batcher's 63).
#ifndef TRIPS_NET16
#define TRIPS_NET16 1
#endif
#ifndef TRIPS_NET_SIZES
#define TRIPS_NET_SIZES 2        // network sizes k_raster phase C picks from: 2 = {8, 16}, 4 = {4, 8, 12, 16} (measured slower: +11 us)
#endif
template <int N>
__device__ __forceinline__ void sort_small(uint64_t (&t)[16]);

template <>
__device__ __forceinline__ void sort_small<4>(uint64_t (&t)[16])
{
    cswap(t[0], t[1]); cswap(t[2], t[3]); cswap(t[0], t[2]); cswap(t[1], t[3]); cswap(t[1], t[2]);
}

template <>
__device__ __forceinline__ void sort_small<12>(uint64_t (&t)[16])
{
    cswap(t[0], t[8]); cswap(t[1], t[7]); cswap(t[2], t[6]); cswap(t[3], t[11]); cswap(t[4], t[10]); cswap(t[5], t[9]);
    cswap(t[0], t[1]); cswap(t[2], t[5]); cswap(t[3], t[4]); cswap(t[6], t[9]); cswap(t[7], t[8]); cswap(t[10], t[11]);
    cswap(t[0], t[2]); cswap(t[1], t[6]); cswap(t[5], t[10]); cswap(t[9], t[11]);
    cswap(t[0], t[3]); cswap(t[1], t[2]); cswap(t[4], t[6]); cswap(t[5], t[7]); cswap(t[8], t[11]); cswap(t[9], t[10]);
    cswap(t[1], t[4]); cswap(t[3], t[5]); cswap(t[6], t[8]); cswap(t[7], t[10]);
    cswap(t[1], t[3]); cswap(t[2], t[5]); cswap(t[6], t[9]); cswap(t[8], t[10]);
    cswap(t[2], t[3]); cswap(t[4], t[5]); cswap(t[6], t[7]); cswap(t[8], t[9]);
    cswap(t[4], t[6]); cswap(t[5], t[7]);
    cswap(t[3], t[4]); cswap(t[5], t[6]); cswap(t[7], t[8]);
}

template <>
__device__ __forceinline__ void sort_small<8>(uint64_t (&t)[16])
{
    cswap(t[0], t[1]); cswap(t[2], t[3]); cswap(t[0], t[2]); cswap(t[1], t[3]); cswap(t[1], t[2]);
    cswap(t[4], t[5]); cswap(t[6], t[7]); cswap(t[4], t[6]); cswap(t[5], t[7]); cswap(t[5], t[6]);
    cswap(t[0], t[4]); cswap(t[2], t[6]); cswap(t[2], t[4]); cswap(t[1], t[5]); cswap(t[3], t[7]);
    cswap(t[3], t[5]); cswap(t[1], t[2]); cswap(t[3], t[4]); cswap(t[5], t[6]);
}

template <>
__device__ __forceinline__ void sort_small<16>(uint64_t (&t)[16])
{
#if TRIPS_NET16
    cswap(t[0], t[13]); cswap(t[1], t[12]); cswap(t[2], t[15]); cswap(t[3], t[14]); cswap(t[4], t[8]); cswap(t[5], t[6]); cswap(t[7], t[11]); cswap(t[9], t[10]);
    cswap(t[0], t[5]); cswap(t[1], t[7]); cswap(t[2], t[9]); cswap(t[3], t[4]); cswap(t[6], t[13]); cswap(t[8], t[14]); cswap(t[10], t[15]); cswap(t[11], t[12]);
    cswap(t[0], t[1]); cswap(t[2], t[3]); cswap(t[4], t[5]); cswap(t[6], t[8]); cswap(t[7], t[9]); cswap(t[10], t[11]); cswap(t[12], t[13]); cswap(t[14], t[15]);
    cswap(t[0], t[2]); cswap(t[1], t[3]); cswap(t[4], t[10]); cswap(t[5], t[11]); cswap(t[6], t[7]); cswap(t[8], t[9]); cswap(t[12], t[14]); cswap(t[13], t[15]);
    cswap(t[1], t[2]); cswap(t[3], t[12]); cswap(t[4], t[6]); cswap(t[5], t[7]); cswap(t[8], t[10]); cswap(t[9], t[11]); cswap(t[13], t[14]);
    cswap(t[1], t[4]); cswap(t[2], t[6]); cswap(t[5], t[8]); cswap(t[7], t[10]); cswap(t[9], t[13]); cswap(t[11], t[14]);
    cswap(t[2], t[4]); cswap(t[3], t[6]); cswap(t[9], t[12]); cswap(t[11], t[13]);
    cswap(t[3], t[5]); cswap(t[6], t[8]); cswap(t[7], t[9]); cswap(t[10], t[12]);
    cswap(t[3], t[4]); cswap(t[5], t[6]); cswap(t[7], t[8]); cswap(t[9], t[10]); cswap(t[11], t[12]);
    cswap(t[6], t[7]); cswap(t[8], t[9]);
#else
    cswap(t[0], t[1]); cswap(t[2], t[3]); cswap(t[0], t[2]); cswap(t[1], t[3]); cswap(t[1], t[2]);
    cswap(t[4], t[5]); cswap(t[6], t[7]); cswap(t[4], t[6]); cswap(t[5], t[7]); cswap(t[5], t[6]);
    cswap(t[0], t[4]); cswap(t[2], t[6]); cswap(t[2], t[4]); cswap(t[1], t[5]); cswap(t[3], t[7]);
    cswap(t[3], t[5]); cswap(t[1], t[2]); cswap(t[3], t[4]); cswap(t[5], t[6]);
    cswap(t[8], t[9]); cswap(t[10], t[11]); cswap(t[8], t[10]); cswap(t[9], t[11]); cswap(t[9], t[10]);
    cswap(t[12], t[13]); cswap(t[14], t[15]); cswap(t[12], t[14]); cswap(t[13], t[15]); cswap(t[13], t[14]);
    cswap(t[8], t[12]); cswap(t[10], t[14]); cswap(t[10], t[12]); cswap(t[9], t[13]); cswap(t[11], t[15]);
    cswap(t[11], t[13]); cswap(t[9], t[10]); cswap(t[11], t[12]); cswap(t[13], t[14]);
    cswap(t[0], t[8]); cswap(t[4], t[12]); cswap(t[4], t[8]); cswap(t[2], t[10]); cswap(t[6], t[14]);
    cswap(t[6], t[10]); cswap(t[2], t[4]); cswap(t[6], t[8]); cswap(t[10], t[12]); cswap(t[1], t[9]);
    cswap(t[5], t[13]); cswap(t[5], t[9]); cswap(t[3], t[11]); cswap(t[7], t[15]); cswap(t[7], t[11]);
    cswap(t[3], t[5]); cswap(t[7], t[9]); cswap(t[11], t[13]); cswap(t[1], t[2]); cswap(t[3], t[4]);
    cswap(t[5], t[6]); cswap(t[7], t[8]); cswap(t[9], t[10]); cswap(t[11], t[12]); cswap(t[13], t[14]);
#endif
}

// r (sorted asc, 16) <- the 16 smallest of r U t, t sorted asc in t[0..N) (N = 8 or 16):
// bitonic split (min against reversed t) + bitonic clean.
template <int N>
__device__ __forceinline__ void merge_keep16(uint64_t (&r)[16], const uint64_t (&t)[16])
{
#pragma unroll
    for (int j = 16 - N; j < 16; ++j) r[j] = r[j] < t[15 - j] ? r[j] : t[15 - j];
#pragma unroll
    for (int d = 8; d > 0; d >>= 1)
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if ((i & d) == 0) cswap(r[i], r[i + d]);
}

// Phase C step: the next min(rem, N) keys of this pixel's chunk list (k[0..)) are sorted with
// the N-key network and merged into the running top-16 r (or become it when `first`).
template <int N>
__device__ __forceinline__ void group_top16(uint64_t (&r)[16], const uint64_t* k, uint32_t rem, bool first)
{
    uint64_t tk[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) tk[j] = (j < N && (uint32_t)j < rem) ? k[j] : kKeyMax;
    sort_small<N>(tk);
    if (first) {
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = tk[j];
    } else {
        merge_keep16<N>(r, tk);
    }
}

// Exclusive prefix of one u32 per thread over a 256-thread tile CTA with a single barrier:
// warp-inclusive shuffle scan, warp totals through shared memory, each thread adds the totals of
// the warps before it.  `s_warp` (>= 8 u32) must not be rewritten before the next barrier.
__device__ __forceinline__ uint32_t tile_excl_scan(uint32_t v, uint32_t* s_warp)
{
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    uint32_t pre = 0;
#pragma unroll
    for (int w = 0; w < kTilePix / 32 - 1; ++w) pre += (w < (int)warp) ? s_warp[w] : 0u;
    return pre + x - v;
}

// --------------------------------------------------------------------------- fragment weights

// gamma of point record r0 = (x, y, s, alpha) at pixel (px, py) of layer l (Eq. 3):
// beta = wx wy with wx = 1 - |x_l - px|, iota from Eq. (4) for layer l.
struct FragW {
    float gamma, beta, iota, diota, wx, wy;
    int dx, dy;
};

__device__ __forceinline__ FragW frag_weights(float4 r0, int l, int n_layers, int px, int py)
{
    FragW w;
    const Levels lv = select_levels(r0.z, n_layers);
    const int sel = l - lv.lo;                       // 0 or 1
    w.iota = sel ? lv.iota[1] : lv.iota[0];
    w.diota = sel ? lv.diota[1] : lv.diota[0];
    const float sc = pow2_neg(l);
    const float xl = __fmul_rn(r0.x, sc), yl = __fmul_rn(r0.y, sc);
    const float x0 = floorf(xl), y0 = floorf(yl);
    const float fx = __fsub_rn(xl, x0), fy = __fsub_rn(yl, y0);
    w.dx = px - (int)x0;
    w.dy = py - (int)y0;
    w.wx = w.dx ? fx : __fsub_rn(1.0f, fx);
    w.wy = w.dy ? fy : __fsub_rn(1.0f, fy);
    w.beta = __fmul_rn(w.wx, w.wy);
    w.gamma = __fmul_rn(__fmul_rn(w.beta, w.iota), r0.w);
    return w;
}

struct TileCoord {
    int l, tx, ty;
};

__device__ __forceinline__ TileCoord tile_coord(const Params& P, int t)
{
    int l = 0;
#pragma unroll 1
    while (l + 1 < P.n_layers && t >= P.L[l + 1].tile_base) ++l;
    const int loc = t - P.L[l].tile_base;
    TileCoord c;
    c.l = l;
    c.ty = loc / P.L[l].tiles_x;
    c.tx = loc - c.ty * P.L[l].tiles_x;
    return c;
}

// --------------------------------------------------------------------------- K4 raster

// Dynamic shared memory of k_raster: the per-chunk fragment keys.  (Reusing it after the last
// chunk to stage the kept records for the blend with one cp.async wave was measured slower:
// 64 KB per CTA shrinks L1 -- profiles/r01_v2.md.)
// After the last chunk the buffer holds the 16 x 256 sorted kept keys (phase D / F), so it is at
// least 32 KB whatever the chunk size.
__host__ __device__ constexpr int raster_keys_smem() { return kChunk * 32 > kCap * kTilePix * 8 ? kChunk * 32 : kCap * kTilePix * 8; }

__host__ __device__ constexpr int raster_dyn_smem() { return raster_keys_smem(); }

// MODE: kRasterPlain (the definition), kRasterTmin (T_min variant, Q17) or kRasterOwn
// (coarse-layer inclusion, Q22: phases A-C only; the pixel's own sorted top-16 goes to P.own
// and k_coarse_blend merges it with its ancestors' lists and blends).
enum RasterMode { kRasterPlain = 0, kRasterTmin = 1, kRasterOwn = 2 };

__device__ __forceinline__ void emit_kept_pairs(const Params& P, int t, uint32_t b0, uint32_t M, const uint64_t* s_kk,
                                                const uint64_t* s_thr, uint32_t* s_ctr);


template <int FC, int MODE>
__global__ void __launch_bounds__(kTilePix, TRIPS_RASTER_CTAS) k_raster(Params P, float* __restrict__ pyramid, int save)
{
    constexpr bool COARSE = MODE == kRasterOwn;
    constexpr bool TMIN = MODE == kRasterTmin;
    extern __shared__ __align__(16) uint64_t s_dyn[];
    uint64_t* s_keys = s_dyn;                        // [kChunk * 4] fragment keys of a chunk
    __shared__ uint32_t s_cnt[kTilePix];
    __shared__ uint32_t s_base[kTilePix];
    __shared__ uint32_t s_rej[kTilePix];             // fragments rejected by the threshold
    __shared__ uint64_t s_thr[kTilePix];             // per-pixel 16th smallest key so far
    __shared__ uint32_t s_warp[32];

    const int t = P.tile_perm ? (int)__ldg(P.tile_perm + blockIdx.x) : (int)blockIdx.x;
    const TileCoord tc = tile_coord(P, t);
    const LayerGeom& G = P.L[tc.l];
    const int tid = threadIdx.x;
    const int lx = tid & (kTile - 1), ly = tid >> 4;
    const int x_lo = tc.tx * kTile, y_lo = tc.ty * kTile;
    const int px = x_lo + lx, py = y_lo + ly;
    const bool valid = px < G.W && py < G.H;
    const uint32_t b0 = P.tile_off[t], b1 = P.tile_off[t + 1];

    uint64_t r[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = kKeyMax;
    uint32_t total = 0;

    s_thr[tid] = kKeyMax;
    TRIPS_PCLK_START;
    // Chunks interleave the bin (chunk ch takes positions ch, ch + nch, ...): a pixel's
    // fragments then spread evenly over the chunks whatever the point order, which balances
    // the per-pixel merge work inside a chunk and lets the 16th-key threshold of earlier
    // chunks reject most fragments of later ones.
    const uint32_t M = b1 - b0;
    const uint32_t nch = (M + kChunk - 1) / kChunk;
    for (uint32_t ch = 0; ch < nch; ++ch) {
        const int m = (int)((M - ch + nch - 1) / nch);
        const uint32_t c0 = b0 + ch;                 // element j of this chunk: c0 + j * nch
        s_cnt[tid] = 0;
        s_rej[tid] = 0;
        __syncthreads();
        // phase A: this chunk's pairs -> fragments of this tile (footprint origin in the bin).
        // Lanes of a warp take pairs 8 apart: consecutive bin entries of a spatially ordered
        // cloud hit the same pixels, and same-address shared atomics within a warp serialise.
        uint32_t fq[kPairsPerThread][4];             // (q | rank << 8), 0xffffffff = none
        const int jl = (tid & 31) * 8 + (tid >> 5);
        // all of this thread's pair loads issued before the first shared-memory atomic (a
        // generic-pointer load cannot be hoisted across them); keys stay live for phase B
        uint64_t pk[kPairsPerThread];
        uint32_t po[kPairsPerThread];
#pragma unroll
        for (int k = 0; k < kPairsPerThread; ++k) {
            const int j = jl + k * kTilePix;
            pk[k] = j < m ? __ldg(reinterpret_cast<const unsigned long long*>(P.bin_key) + c0 + (size_t)j * nch) : 0ull;
            po[k] = j < m ? __ldg(P.bin_orig + c0 + (size_t)j * nch) : 0u;
        }
#pragma unroll
        for (int k = 0; k < kPairsPerThread; ++k) {
#pragma unroll
            for (int c = 0; c < 4; ++c) fq[k][c] = 0xffffffffu;
            const int j = jl + k * kTilePix;
            if (j < m) {
                const uint64_t key = pk[k];
                const uint32_t o = po[k];
                const int q0 = (int)(o & 31u) - 1 + ((int)((o >> 5) & 31u) - 1) * kTile;   // may be < 0
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (o & (1u << (10 + c))) {               // corner inside this tile and layer
                        const uint32_t q = (uint32_t)(q0 + (c & 1) + (c >> 1) * kTile);
                        if (TRIPS_THR_SKIP0 && ch == 0) {
                            // first chunk: no pixel holds 16 keys yet, nothing can be rejected
                            const uint32_t rank = atomicAdd(&s_cnt[q], 1u);
                            fq[k][c] = q | (rank << 8);
                        } else if (key >= s_thr[q]) {
                            // cannot enter this pixel's top-16 any more (keys are unique):
                            // counted for the list length, never sorted
                            atomicAdd(&s_rej[q], 1u);
                        } else {
                            const uint32_t rank = atomicAdd(&s_cnt[q], 1u);
                            fq[k][c] = q | (rank << 8);
                        }
                    }
                }
            }
        }
        __syncthreads();
        TRIPS_PCLK(0);
        const uint32_t my_cnt = s_cnt[tid];
        const uint32_t my_base = tile_excl_scan(my_cnt, s_warp);
        s_base[tid] = my_base;
        __syncthreads();
        TRIPS_PCLK(1);
        // phase B: counting-sort scatter by pixel (keys re-read from L1 instead of being held
        // in registers across the scan)
#pragma unroll
        for (int k = 0; k < kPairsPerThread; ++k) {
            const int j = jl + k * kTilePix;
            if (j < m) {
                const uint64_t key = pk[k];
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (fq[k][c] != 0xffffffffu) s_keys[s_base[fq[k][c] & 0xffu] + (fq[k][c] >> 8)] = key;
            }
        }
        __syncthreads();
        TRIPS_PCLK(2);
        // phase C: merge this pixel's new fragments into its running top-16.  Network sizes are
        // chosen per warp (8 when no lane of the warp has more than 8 keys left in the group).
        const uint32_t wcnt = __reduce_max_sync(0xffffffffu, my_cnt);
        for (uint32_t g = 0; g < wcnt; g += 16) {
            const uint32_t rem = my_cnt > g ? my_cnt - g : 0u;
            const bool first = __all_sync(0xffffffffu, total == 0 && g == 0);
            const uint32_t wrem = __reduce_max_sync(0xffffffffu, rem);
#if TRIPS_NET_SIZES == 4
            if (wrem <= 4u) group_top16<4>(r, s_keys + my_base + g, rem, first);
            else if (wrem <= 8u) group_top16<8>(r, s_keys + my_base + g, rem, first);
            else if (wrem <= 12u) group_top16<12>(r, s_keys + my_base + g, rem, first);
            else group_top16<16>(r, s_keys + my_base + g, rem, first);
#else
            if (wrem <= 8u) group_top16<8>(r, s_keys + my_base + g, rem, first);
            else group_top16<16>(r, s_keys + my_base + g, rem, first);
#endif
        }
        total += my_cnt + s_rej[tid];
        s_thr[tid] = r[15];                          // 16th smallest key so far (MAX if < 16)
        if (ch + 1 < nch) __syncthreads();           // shared buffers are reused by the next chunk only
        TRIPS_PCLK(3);
    }

    if constexpr (COARSE) {
        P.pix_cnt[(size_t)t * kTilePix + tid] = valid ? total : 0u;
        const int Ko = valid ? (int)min(total, (uint32_t)kCap) : 0;
        // [tile][m][pixel] so that a warp's m-th keys are contiguous (coalesced both ways)
        uint64_t* op = P.own + (size_t)t * kTilePix * kCap + tid;
#pragma unroll
        for (int mm = 0; mm < kCap; ++mm)
            if (mm < Ko) op[(size_t)mm * kTilePix] = r[mm];
        return;
    }

#if !TRIPS_BLEND_REG
    // The sorted top-16 moves to the (now free) chunk buffer, [m][pixel]: the blend reads its
    // indices from there and phase F binary-searches it, so the 16 key registers die here.
    __syncthreads();                                 // other lanes may still read s_keys (phase C)
    uint64_t* s_kk = s_keys;                         // 16 x 256 keys (= kChunk * 4)
#pragma unroll
    for (int mm = 0; mm < kCap; ++mm) s_kk[mm * kTilePix + tid] = r[mm];   // kKeyMax beyond K
#endif

    // phase D: front-to-back blend of the kept list (Eqs. 5-6; alpha_m := gamma_m, Q10).
    // Record gathers are issued kBatch at a time.  Without a following backward the loop
    // stops once T == 0 exactly (later terms vanish); with one, every gamma_m is needed.
    const int K = valid ? (int)min(total, (uint32_t)kCap) : 0;
    constexpr int KS = kTilePix;                     // [tile][m][pixel]: entry m at kidx + m * KS
    TRIPS_PCLK(4);
    const size_t kidx = kept_base(t) + (size_t)tid;
    float C[FC];
#pragma unroll
    for (int c = 0; c < FC; ++c) C[c] = 0.f;
    float A = 0.f, T = 1.f;
    // T_min variant (0 = the exact definition): the kept list ends with
    // the fragment after which the fp32 transmittance drops below t_min
    int Keff = K;
    constexpr int kBB = blend_batch<FC>();
#pragma unroll
    for (int b = 0; b < kCap / kBB; ++b) {
        if (b * kBB >= Keff || (!save && T == 0.f)) break;
        float4 rb[kBB][1 + FC / 4];
#pragma unroll
        for (int u = 0; u < kBB; ++u) {
            const int mm = b * kBB + u;
#if TRIPS_BLEND_REG
            const uint32_t ii = (uint32_t)(mm < K ? r[mm] : r[0]);
#else
            const uint32_t ii = (uint32_t)s_kk[(mm < K ? mm : 0) * kTilePix + tid];
#endif
            gather_record<FC>(P, ii, rb[u]);
        }
#pragma unroll
        for (int u = 0; u < kBB; ++u) {
            const int mm = b * kBB + u;
            if (mm < Keff) {
                const FragW w = frag_weights(rb[u][0], tc.l, P.n_layers, px, py);
                const float tg = T * w.gamma;
#pragma unroll
                for (int c4 = 0; c4 < FC / 4; ++c4) {
                    const float4 tau = rb[u][1 + c4];
                    C[4 * c4 + 0] = fmaf(tg, tau.x, C[4 * c4 + 0]);
                    C[4 * c4 + 1] = fmaf(tg, tau.y, C[4 * c4 + 1]);
                    C[4 * c4 + 2] = fmaf(tg, tau.z, C[4 * c4 + 2]);
                    C[4 * c4 + 3] = fmaf(tg, tau.w, C[4 * c4 + 3]);
                }
                A += tg;
                T = __fmul_rn(T, __fsub_rn(1.0f, w.gamma));      // pinned: decides the T_min cut
                if (save) P.kept_gamma[kidx + (size_t)mm * KS] = w.gamma;
                if (TMIN && T < P.t_min) Keff = mm + 1;
            }
        }
    }
    if (valid) {
        const int64_t plane = (int64_t)G.W * G.H;
        float* out = pyramid + G.float_off + (int64_t)py * G.W + px;
#pragma unroll
        for (int c = 0; c < FC; ++c)
            if (c < P.F) out[c * plane] = C[c];
        out[P.F * plane] = A;
    }
    TRIPS_PCLK(5);

    // phase E: per-pixel metadata
    P.pix_cnt[(size_t)t * kTilePix + tid] = valid ? total : 0u;
    P.pix_meta[(size_t)t * kTilePix + tid] = (uint32_t)Keff;
    TRIPS_PCLK(6);
    if (!save) return;
#ifdef TRIPS_EXP_NOPF
    if (tid == 0) P.kp_cnt[t] = 0;
    return;
#endif

    // phase F: the sorted kept lists stored as the tile's kept (point, tile) pairs
    // (emit_kept_pairs)
#if TRIPS_BLEND_REG
    __syncthreads();                                 // other lanes may still read s_keys (phase C)
    uint64_t* s_kk = s_keys;                         // 16 x 256 keys (= kChunk * 4)
#pragma unroll
    for (int mm = 0; mm < kCap; ++mm) s_kk[mm * kTilePix + tid] = r[mm];   // kKeyMax beyond K
#endif
    // per-pixel kept threshold: the Keff-th key (a key of this pixel is kept iff <= it)
    s_thr[tid] = Keff > 0 ? s_kk[(Keff - 1) * kTilePix + tid] : 0ull;
    if (tid == 0) s_warp[0] = 0;
    __syncthreads();
    emit_kept_pairs(P, t, b0, M, s_kk, s_thr, s_warp);
    TRIPS_PCLK(7);
}

// Kept (point, tile) pairs of tile t: a pair of the bin is kept at corner c iff its key is among
// the first Keff keys of that corner's pixel; its slot m there is the key's rank (binary search of
// the pixel's sorted list).  A point's <= 4 kept fragments in the tile then travel together: the
// backward gathers its record and reduces its gradient once per pair instead of once per fragment
// (2.8x fewer scattered L2 operations at C4).  s_kk: [m][pixel] sorted kept keys (any key > the
// kept ones beyond Keff), s_thr: per-pixel Keff-th key (0 if Keff = 0), *s_ctr zeroed; all threads
// call after a barrier.
__device__ __forceinline__ void emit_kept_pairs(const Params& P, int t, uint32_t b0, uint32_t M, const uint64_t* s_kk,
                                                const uint64_t* s_thr, uint32_t* s_ctr)
{
    const int tid = threadIdx.x;
    const size_t kpb = kept_base(t);
    const unsigned long long* bk = reinterpret_cast<const unsigned long long*>(P.bin_key) + b0;
    const uint16_t* bo = P.bin_orig + b0;
    for (uint32_t j0 = tid; j0 < M; j0 += kPfUnroll * kTilePix) {
        uint64_t key[kPfUnroll];
        uint32_t o[kPfUnroll];
#pragma unroll
        for (int u = 0; u < kPfUnroll; ++u) {
            const uint32_t j = j0 + u * kTilePix;
            key[u] = j < M ? __ldg(bk + j) : kKeyMax;
            o[u] = j < M ? __ldg(bo + j) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kPfUnroll; ++u) {
            const int q0 = (int)(o[u] & 31u) - 1 + ((int)((o[u] >> 5) & 31u) - 1) * kTile;
            uint32_t info = o[u] & 0x3ffu;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int q = q0 + (c & 1) + (c >> 1) * kTile;
                if ((o[u] & (1u << (10 + c))) && key[u] <= s_thr[q]) {
                    const uint64_t* L = s_kk + q;
                    int p = 0;
                    p += L[(p + 7) * kTilePix] < key[u] ? 8 : 0;
                    p += L[(p + 3) * kTilePix] < key[u] ? 4 : 0;
                    p += L[(p + 1) * kTilePix] < key[u] ? 2 : 0;
                    p += L[p * kTilePix] < key[u] ? 1 : 0;
                    info |= (1u << (10 + c)) | ((uint32_t)p << (14 + 4 * c));
                }
            }
            if (info & 0x3c00u) {
                const uint32_t slot = atomicAdd(s_ctr, 1u);
                P.kp_key[kpb + slot] = key[u];
                P.kp_info[kpb + slot] = info;
            }
        }
    }
    __syncthreads();
    if (tid == 0) P.kp_cnt[t] = *s_ctr;
}

// --------------------------------------------------------------------------- K4c coarse blend

// Coarse-layer inclusion (reading Q22).  One thread
// per pyramid pixel (l, x, y): merges the own sorted top-16 lists of (l + d, x >> d, y >> d),
// d = 0..D, into the top-16 of their union.  Keys become (z, i << 4 | d) so that the networks
// order by (z, i, d) -- the same point's fragment in a finer layer first (i < 2^28 by the plan
// limit).  The top-16 of a union is inside the union of the top-16s, so the own lists suffice.
// Then the front-to-back blend of k_raster phase D, each fragment weighted in its own layer and
// pixel; kept lists [tile][m][pixel] as in k_raster.
template <int FC>
__global__ void __launch_bounds__(kTilePix) k_coarse_blend(Params P, float* __restrict__ pyramid, int save)
{
    const int t = P.tile_perm ? (int)__ldg(P.tile_perm + blockIdx.x) : (int)blockIdx.x;
    const TileCoord tc = tile_coord(P, t);
    const LayerGeom& G = P.L[tc.l];
    const int tid = threadIdx.x;
    const int px = tc.tx * kTile + (tid & (kTile - 1)), py = tc.ty * kTile + (tid >> 4);
    const bool valid = px < G.W && py < G.H;
    const int D = min(P.coarse, P.n_layers - 1 - tc.l);

    uint64_t r[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = kKeyMax;
    int K = 0;
    for (int d = 0; d <= D; ++d) {
        const LayerGeom& A = P.L[tc.l + d];
        const int ax = px >> d, ay = py >> d;
        const size_t at = (size_t)(A.tile_base + (ay >> 4) * A.tiles_x + (ax >> 4));
        const int aq = (ay & (kTile - 1)) * kTile + (ax & (kTile - 1));
        const int kd = valid ? (int)min(__ldg(P.pix_cnt + at * kTilePix + aq), (uint32_t)kCap) : 0;
        if (__all_sync(0xffffffffu, kd == 0)) continue;
        K += kd;
        const unsigned long long* op = reinterpret_cast<const unsigned long long*>(P.own) + at * kTilePix * kCap + aq;
        uint64_t tk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint64_t k = j < kd ? __ldg(op + (size_t)j * kTilePix) : kKeyMax;
            tk[j] = j < kd ? ((k & 0xffffffff00000000ull) | ((k & 0xffffffffull) << 4) | (uint64_t)d) : kKeyMax;
        }
        merge_keep16<16>(r, tk);
    }
    K = min(K, kCap);

    // dense kept lists, [tile][m][pixel] (stride kTilePix between a pixel's entries)
    const size_t kidx = kept_base(t) + (size_t)tid;
    float C[FC];
#pragma unroll
    for (int c = 0; c < FC; ++c) C[c] = 0.f;
    float A = 0.f, T = 1.f;
    int Keff = K;
    constexpr int kBB = blend_batch<FC>();
#pragma unroll
    for (int b = 0; b < kCap / kBB; ++b) {
        if (b * kBB >= Keff || (!save && T == 0.f)) break;
        float4 rb[kBB][1 + FC / 4];
#pragma unroll
        for (int u = 0; u < kBB; ++u) {
            const int mm = b * kBB + u;
            const uint32_t ii = (uint32_t)(mm < K ? r[mm] : r[0]) >> 4;
            gather_record<FC>(P, ii, rb[u]);
        }
#pragma unroll
        for (int u = 0; u < kBB; ++u) {
            const int mm = b * kBB + u;
            if (mm < Keff) {
                const int d = (int)(r[mm] & 15u);
                const FragW w = frag_weights(rb[u][0], tc.l + d, P.n_layers, px >> d, py >> d);
                const float tg = T * w.gamma;
#pragma unroll
                for (int c4 = 0; c4 < FC / 4; ++c4) {
                    const float4 tau = rb[u][1 + c4];
                    C[4 * c4 + 0] = fmaf(tg, tau.x, C[4 * c4 + 0]);
                    C[4 * c4 + 1] = fmaf(tg, tau.y, C[4 * c4 + 1]);
                    C[4 * c4 + 2] = fmaf(tg, tau.z, C[4 * c4 + 2]);
                    C[4 * c4 + 3] = fmaf(tg, tau.w, C[4 * c4 + 3]);
                }
                A += tg;
                T = __fmul_rn(T, __fsub_rn(1.0f, w.gamma));
                if (save) P.kept_gamma[kidx + (size_t)mm * kTilePix] = w.gamma;
                if (T < P.t_min) Keff = mm + 1;
            }
        }
    }
    if (valid) {
        const int64_t plane = (int64_t)G.W * G.H;
        float* out = pyramid + G.float_off + (int64_t)py * G.W + px;
#pragma unroll
        for (int c = 0; c < FC; ++c)
            if (c < P.F) out[c * plane] = C[c];
        out[P.F * plane] = A;
    }
    P.pix_meta[(size_t)t * kTilePix + tid] = (uint32_t)Keff;
    if (save) {
        uint64_t* kp = P.kept + kidx;
#pragma unroll
        for (int mm = 0; mm < kCap; ++mm)
            if (mm < Keff) kp[(size_t)mm * kTilePix] = r[mm];
    }
}

// --------------------------------------------------------------------------- K5 backward

// Caller's gradient buffers (trips_splat_backward): pos_size [n] float4 (dL/dx, dL/dy, dL/dz,
// dL/ds_w), opacity [n], desc [n][F] (vector reductions when the rows allow it: desc_vec = 4 for
// F % 4 == 0 and 16-B aligned rows, 2 for F % 2 == 0 and 8-B aligned, else 1).  `screen`
// (debug export only) receives the screen-space gradients [n][4 + F] instead.
struct GradOut {
    float* pos_size;
    float* opacity;
    float* desc;
    float* screen;
    int desc_vec;
};

__device__ __forceinline__ void red_add_v2(float* addr, float a, float b)
{
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" :: "l"(addr), "f"(a), "f"(b));
}
__device__ __forceinline__ void red_add_f32(float* addr, float a)
{
    asm volatile("red.global.add.f32 [%0], %1;" :: "l"(addr), "f"(a));
}

// Screen-space gradient of one point in one view (gxs, gys, gs: d/dx, d/dy, d/ds in layer-0
// pixels; galpha; gtau[F]) -> world space through the projection chain (Eq. 2, Sec. 3.1), added
// to the caller's buffers with vector reductions; CAM: camera partials into cg.  SCREEN (debug
// export): the screen-space values are added to go.screen instead.
template <int FC, bool CAM, bool SCREEN>
__device__ __forceinline__ void point_reduce(const Params& P, uint32_t i, float4 r0, float z, float gxs, float gys,
                                             float gs, float galpha, const float (&gtau)[FC], const GradOut& go,
                                             float (&cg)[CAM ? 17 : 1])
{
    if (SCREEN) {
        float* d = go.screen + (size_t)i * (4 + P.F);
        atomicAdd(d + 0, gxs); atomicAdd(d + 1, gys); atomicAdd(d + 2, gs); atomicAdd(d + 3, galpha);
#pragma unroll
        for (int c = 0; c < FC; ++c)
            if (c < P.F) atomicAdd(d + 4 + c, gtau[c]);
        return;
    }
    const Cam& cam = P.cam;
    const float iz = 1.0f / z;
    const float gpx = gxs * cam.fx * iz, gpy = gys * cam.fy * iz;
    const float gpz = -(gxs * (r0.x - cam.cx) + gys * (r0.y - cam.cy) + gs * r0.z) * iz;
    const float gX = cam.R[0] * gpx + cam.R[3] * gpy + cam.R[6] * gpz;
    const float gY = cam.R[1] * gpx + cam.R[4] * gpy + cam.R[7] * gpz;
    const float gZ = cam.R[2] * gpx + cam.R[5] * gpy + cam.R[8] * gpz;
    const float gsw = gs * cam.f * iz;
    if (CAM) {
        // p = (px, py, z) from the screen record, X = R^T (p - t)
        const float pxv = (r0.x - cam.cx) * z / cam.fx, pyv = (r0.y - cam.cy) * z / cam.fy;
        const float q0 = pxv - cam.t[0], q1 = pyv - cam.t[1], q2 = z - cam.t[2];
        const float Xw[3] = {cam.R[0] * q0 + cam.R[3] * q1 + cam.R[6] * q2,
                             cam.R[1] * q0 + cam.R[4] * q1 + cam.R[7] * q2,
                             cam.R[2] * q0 + cam.R[5] * q1 + cam.R[8] * q2};
        const float gpv[3] = {gpx, gpy, gpz};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
#pragma unroll
            for (int b = 0; b < 3; ++b) cg[3 * a + b] = fmaf(gpv[a], Xw[b], cg[3 * a + b]);
            cg[9 + a] += gpv[a];
        }
        cg[12] = fmaf(gxs, pxv * iz, cg[12]);
        cg[13] = fmaf(gys, pyv * iz, cg[13]);
        cg[14] += gxs;
        cg[15] += gys;
        cg[16] = fmaf(gs, r0.z / cam.f, cg[16]);
    }
    red_add_v4(go.pos_size + (size_t)i * 4, gX, gY, gZ, gsw);
    red_add_f32(go.opacity + i, galpha);
    float* dr = go.desc + (size_t)i * P.F;
    if (go.desc_vec == 4) {
#pragma unroll
        for (int c4 = 0; c4 < FC / 4; ++c4) red_add_v4(dr + 4 * c4, gtau[4 * c4], gtau[4 * c4 + 1], gtau[4 * c4 + 2], gtau[4 * c4 + 3]);
    } else if (go.desc_vec == 2) {
#pragma unroll
        for (int c2 = 0; c2 < FC / 2; ++c2)
            if (2 * c2 < P.F) red_add_v2(dr + 2 * c2, gtau[2 * c2], gtau[2 * c2 + 1]);
    } else {
#pragma unroll
        for (int c = 0; c < FC; ++c)
            if (c < P.F) red_add_f32(dr + c, gtau[c]);
    }
}

// Block reduction of the 17 camera-gradient partials, 17 atomics per tile (all threads call).
__device__ __forceinline__ void camera_block_reduce(float (&cg)[17], float* grad_cam)
{
    __shared__ float s_cg[kTilePix / 32][17];
    const int tid = threadIdx.x;
#pragma unroll
    for (int k = 0; k < 17; ++k) {
        float v = cg[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((tid & 31) == 0) s_cg[tid >> 5][k] = v;
    }
    __syncthreads();
    if (tid < 17) {
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < kTilePix / 32; ++w) v += s_cg[w][tid];
        if (v != 0.f) atomicAdd(grad_cam + tid, v);
    }
}

// Pair-wise backward (non-coarse): one CTA per tile, three phases over the tile's kept pairs
// (written by k_raster phase F) and its pixels.
//   P1 per kept pair: gather tau_i once; for each kept corner (pixel q, slot m) c = <gC_q, tau_i>
//   P2 per pixel: T_m from the saved gamma_m (Eq. 6) and the reverse suffix recurrence
//      dL/dgamma_m = T_m (c_m - S_m + gA (1 - b_m)),  S_{m-1} = gamma_m c_m + (1 - gamma_m) S_m,
//      b_{m-1} = gamma_m + (1 - gamma_m) b_m  (division-free)
//   P3 per kept pair: gather the screen record once, sum the chain of Eq. (3)-(4) over its kept
//      corners (beta = wx wy, iota(s)) and dL/dtau = sum T_m gamma_m gC_q, then ONE world-space
//      reduction set per pair (point_reduce).
template <int FC, bool CAM, bool SCREEN>
__global__ void __launch_bounds__(kTilePix, TRIPS_BWD_CTAS) k_backward_pairs(Params P, const float* __restrict__ gpyr,
                                                                             GradOut go, float* __restrict__ grad_cam)
{
    // [channel][pixel] upstream gradient of the tile (static shared memory stays <= 48 KB up to
    // FC = 12; wider descriptors read it from the pyramid through L1 instead)
    constexpr bool kGs = FC <= 12;
    __shared__ float s_g[kGs ? FC * kTilePix : 1];
    __shared__ float s_c[kCap * kTilePix];           // [m][pixel] c_m, then dL/dgamma_m
    __shared__ float s_tg[kCap * kTilePix];          // [m][pixel] T_m gamma_m
    const int t = P.tile_perm ? (int)__ldg(P.tile_perm + blockIdx.x) : (int)blockIdx.x;
    const TileCoord tc = tile_coord(P, t);           // kernel parameters only: no memory round trip
    const LayerGeom& G = P.L[tc.l];
    const int tid = threadIdx.x;
    const int x_lo = tc.tx * kTile, y_lo = tc.ty * kTile;
    const int px = x_lo + (tid & (kTile - 1)), py = y_lo + (tid >> 4);
    const int64_t plane = (int64_t)G.W * G.H;
    // the CTA's independent loads go out together (one memory round trip instead of three):
    // the tile's kept-pair count, this pixel's kept-list length and its upstream gradient
    const uint32_t npair = __ldg(P.kp_cnt + t);
    const int K = (int)(__ldg(P.pix_meta + (size_t)t * kTilePix + tid) & 31u);
    float gv[kGs ? FC : 1];
    float gA = 0.f;
    if (px < G.W && py < G.H) {
        const float* gp = gpyr + G.float_off + (int64_t)py * G.W + px;
        if constexpr (kGs) {
#pragma unroll
            for (int c = 0; c < FC; ++c) gv[c] = c < P.F ? __ldg(gp + c * plane) : 0.f;
        }
        gA = __ldg(gp + P.F * plane);
    } else if constexpr (kGs) {
#pragma unroll
        for (int c = 0; c < FC; ++c) gv[c] = 0.f;
    }
    if (npair == 0) return;                          // uniform: nothing kept in this tile
    const float* gtile = gpyr + G.float_off + (int64_t)y_lo * G.W + x_lo;   // pixel q at (q & 15) + (q >> 4) W
    auto gC = [&](int f, int q) -> float {
        if constexpr (kGs) return s_g[f * kTilePix + q];
        else return f < P.F ? __ldg(gtile + f * plane + (int64_t)(q >> 4) * G.W + (q & (kTile - 1))) : 0.f;
    };
    if constexpr (kGs) {
#pragma unroll
        for (int c = 0; c < FC; ++c) s_g[c * kTilePix + tid] = gv[c];
    }
    const size_t kpb = kept_base(t);
    const unsigned long long* kkey = reinterpret_cast<const unsigned long long*>(P.kp_key) + kpb;
    const uint32_t* kinfo = P.kp_info + kpb;
    constexpr int kBS = bwd_slots<FC>();
    uint64_t rkey[kBS];
    uint32_t rinfo[kBS];
#pragma unroll
    for (int u = 0; u < kBS; ++u) {            // issued before the barrier
        const uint32_t j = tid + u * kTilePix;
        rkey[u] = j < npair ? __ldg(kkey + j) : 0ull;
        rinfo[u] = j < npair ? __ldg(kinfo + j) : 0u;            // no corner bits: inert
    }
    __syncthreads();

    // P1: c = <gC_q, tau_i> for every kept corner.  The first kBS pairs of each thread keep
    // their key, info and screen record in registers for P3 (all their loads are issued before
    // the first use); pairs beyond kBS * 256 (dense tiles) are re-read in P3.
    auto corners_c = [&](uint32_t info, const float4 (&tb)[FC / 4]) {
        const int q0 = (int)(info & 31u) - 1 + ((int)((info >> 5) & 31u) - 1) * kTile;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (info & (1u << (10 + c))) {
                const int q = q0 + (c & 1) + (c >> 1) * kTile;
                const int m = (int)((info >> (14 + 4 * c)) & 15u);
                float d = 0.f;
#pragma unroll
                for (int c4 = 0; c4 < FC / 4; ++c4) {
                    d = fmaf(gC(4 * c4 + 0, q), tb[c4].x, d);
                    d = fmaf(gC(4 * c4 + 1, q), tb[c4].y, d);
                    d = fmaf(gC(4 * c4 + 2, q), tb[c4].z, d);
                    d = fmaf(gC(4 * c4 + 3, q), tb[c4].w, d);
                }
                s_c[m * kTilePix + q] = d;
            }
        }
    };
    float4 rgeo[kBS];
    {
        float4 rtau[kBS][FC / 4];
#pragma unroll
        for (int u = 0; u < kBS; ++u) {
            const uint32_t i = (uint32_t)rkey[u];
            if (rinfo[u]) {
                const float4* tp = reinterpret_cast<const float4*>(P.tau + (size_t)i * FC);
#pragma unroll
                for (int c4 = 0; c4 < FC / 4; ++c4) rtau[u][c4] = __ldg(tp + c4);
                rgeo[u] = __ldg(P.geo + i);
            }
        }
#pragma unroll
        for (int u = 0; u < kBS; ++u)
            if (rinfo[u]) corners_c(rinfo[u], rtau[u]);
    }
    for (uint32_t j = tid + kBS * kTilePix; j < npair; j += kTilePix) {
        const uint32_t i = (uint32_t)__ldg(kkey + j);
        const uint32_t info = __ldg(kinfo + j);
        float4 tb[FC / 4];
        const float4* tp = reinterpret_cast<const float4*>(P.tau + (size_t)i * FC);
#pragma unroll
        for (int c4 = 0; c4 < FC / 4; ++c4) tb[c4] = __ldg(tp + c4);
        corners_c(info, tb);
    }
    __syncthreads();

    // P2: per pixel, T_m and the reverse suffix recurrence
    if (K > 0) {
        const float* gm = P.kept_gamma + kpb + tid;
        float gam[kCap];
#pragma unroll
        for (int mm = 0; mm < kCap; ++mm) gam[mm] = mm < K ? __ldg(gm + mm * kTilePix) : 0.f;
        float Tm[kCap];
        float T = 1.f;
#pragma unroll
        for (int mm = 0; mm < kCap; ++mm) { Tm[mm] = T; T = T * (1.0f - gam[mm]); }
        float S = 0.f, bb = 0.f;
#pragma unroll
        for (int mm = kCap - 1; mm >= 0; --mm) {
            if (mm < K) {
                const float g = gam[mm];
                const float c = s_c[mm * kTilePix + tid];
                s_c[mm * kTilePix + tid] = Tm[mm] * (c - S + gA * (1.0f - bb));
                s_tg[mm * kTilePix + tid] = Tm[mm] * g;
                S = g * c + (1.0f - g) * S;
                bb = g + (1.0f - g) * bb;
            }
        }
    }
    __syncthreads();

    // P3: per kept pair, the chain summed over its kept corners, one reduction set
    float cg[CAM ? 17 : 1];
#pragma unroll
    for (int k = 0; k < (CAM ? 17 : 1); ++k) cg[k] = 0.f;
    const float sc = pow2_neg(tc.l);
    auto pair_chain = [&](uint64_t key, uint32_t info, float4 r0) {
        const uint32_t i = (uint32_t)key;
        const float z = __uint_as_float((uint32_t)(key >> 32));
        const Levels lv = select_levels(r0.z, P.n_layers);
        const bool upper = tc.l != lv.lo;                // this tile's layer is the point's second one
        const float iota = upper ? lv.iota[1] : lv.iota[0];
        const float diota = upper ? lv.diota[1] : lv.diota[0];
        const float xl = __fmul_rn(r0.x, sc), yl = __fmul_rn(r0.y, sc);
        const float fx = __fsub_rn(xl, floorf(xl)), fy = __fsub_rn(yl, floorf(yl));
        const int q0 = (int)(info & 31u) - 1 + ((int)((info >> 5) & 31u) - 1) * kTile;
        float gbx = 0.f, gby = 0.f, gal = 0.f;
        float gt[FC];
#pragma unroll
        for (int c = 0; c < FC; ++c) gt[c] = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (info & (1u << (10 + c))) {
                const int q = q0 + (c & 1) + (c >> 1) * kTile;
                const int m = (int)((info >> (14 + 4 * c)) & 15u);
                const float dg = s_c[m * kTilePix + q];
                const float tg = s_tg[m * kTilePix + q];
                const float wx = (c & 1) ? fx : __fsub_rn(1.0f, fx);
                const float wy = (c & 2) ? fy : __fsub_rn(1.0f, fy);
                const float beta = wx * wy;
                gal = fmaf(dg, beta, gal);                   // * iota at the end
                // d beta / d x_l = wy * (dx ? +1 : -1), d beta / d y_l = wx * (dy ? +1 : -1)
                gbx = fmaf(dg, (c & 1) ? wy : -wy, gbx);     // * iota alpha 2^-l
                gby = fmaf(dg, (c & 2) ? wx : -wx, gby);
#pragma unroll
                for (int f = 0; f < FC; ++f) gt[f] = fmaf(tg, gC(f, q), gt[f]);
            }
        }
        const float ia = iota * r0.w;
        const float gxs = gbx * ia * sc, gys = gby * ia * sc;
        const float gs = gal * r0.w * diota;             // d gamma / d iota = beta alpha
        const float galpha = gal * iota;                 // d gamma / d alpha = beta iota
        point_reduce<FC, CAM, SCREEN>(P, i, r0, z, gxs, gys, gs, galpha, gt, go, cg);
    };
#pragma unroll
    for (int u = 0; u < kBS; ++u)
        if (rinfo[u]) pair_chain(rkey[u], rinfo[u], rgeo[u]);
    for (uint32_t j = tid + kBS * kTilePix; j < npair; j += kTilePix) {
        const uint64_t key = __ldg(kkey + j);
        pair_chain(key, __ldg(kinfo + j), __ldg(P.geo + (uint32_t)key));
    }
    if constexpr (CAM) camera_block_reduce(cg, grad_cam);
}

// Per-pixel backward over the kept (z, i << 4 | d) lists of coarse-layer inclusion (reading Q22):
// the blended fragments of a pixel come from several layers and tiles, so they are replayed per
// pixel and reduced per fragment.
template <int FC, bool CAM, bool SCREEN>
__global__ void __launch_bounds__(kTilePix, FC <= 4 ? 3 : 2) k_backward_coarse(Params P, const float* __restrict__ gpyr,
                                                       GradOut go, float* __restrict__ grad_cam)
{
    const int t = P.tile_perm ? (int)__ldg(P.tile_perm + blockIdx.x) : (int)blockIdx.x;
    const TileCoord tc = tile_coord(P, t);
    const LayerGeom& G = P.L[tc.l];
    const int tid = threadIdx.x;
    const int px = tc.tx * kTile + (tid & (kTile - 1)), py = tc.ty * kTile + (tid >> 4);
    const uint32_t meta = P.pix_meta[(size_t)t * kTilePix + tid];
    const int K = (int)(meta & 31u);
    if (!CAM && K == 0) return;
    const size_t kidx = kept_base(t) + (size_t)tid;
    const uint64_t* kp = P.kept + kidx;
    const float* gm = P.kept_gamma + kidx;
    constexpr int KS = kTilePix;                     // entry stride ([tile][m][pixel])
    float cg[CAM ? 17 : 1];
#pragma unroll
    for (int k = 0; k < (CAM ? 17 : 1); ++k) cg[k] = 0.f;

    // upstream gradient of this pixel: gC (F channels) and gA
    const int64_t plane = (int64_t)G.W * G.H;
    const float* gp = gpyr + G.float_off + (int64_t)py * G.W + px;
    float gC[FC];
#pragma unroll
    for (int c = 0; c < FC; ++c) gC[c] = (K > 0 && c < P.F) ? __ldg(gp + c * plane) : 0.f;
    const float gA = K > 0 ? __ldg(gp + P.F * plane) : 0.f;

    // T_m from the saved gamma_m (Eq. 6) -- no record gathers
    float gam[kCap], Tm[kCap];
    float T = 1.f;
#pragma unroll
    for (int mm = 0; mm < kCap; ++mm) {
        gam[mm] = mm < K ? __ldg(gm + mm * KS) : 0.f;
        Tm[mm] = T;
        T = T * (1.0f - gam[mm]);
    }
    // reverse replay with suffix recurrences (division-free):
    //   dL/dgamma_m = T_m (<gC, tau_m - B_m> + gA (1 - b_m)),
    //   B_{m-1} = gamma_m tau_m + (1 - gamma_m) B_m,   b_{m-1} = gamma_m + (1 - gamma_m) b_m
    float B[FC];
#pragma unroll
    for (int c = 0; c < FC; ++c) B[c] = 0.f;
    float bb = 0.f;
#pragma unroll
    for (int b = kCap / kBatch - 1; b >= 0; --b) {
        if (b * kBatch >= K) continue;
        float4 rb[kBatch][1 + FC / 4];
        uint64_t kb[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int mm = min(b * kBatch + u, K - 1);
            kb[u] = __ldg(reinterpret_cast<const unsigned long long*>(kp) + mm * KS);
            const uint32_t iu = (uint32_t)kb[u] >> 4;
            gather_record<FC>(P, iu, rb[u]);
        }
#pragma unroll
        for (int u = kBatch - 1; u >= 0; --u) {
            const int mm = b * kBatch + u;
            if (mm >= K) continue;
            const uint32_t i = (uint32_t)kb[u] >> 4;
            const int d = (int)(kb[u] & 15u);
            const float sc = pow2_neg(tc.l + d);
            const float z = __uint_as_float((uint32_t)(kb[u] >> 32));
            const float4 r0 = rb[u][0];
            const FragW w = frag_weights(r0, tc.l + d, P.n_layers, px >> d, py >> d);
            const float g = gam[mm], tm = Tm[mm];
            float tau[FC];
#pragma unroll
            for (int c4 = 0; c4 < FC / 4; ++c4) {
                tau[4 * c4 + 0] = rb[u][1 + c4].x; tau[4 * c4 + 1] = rb[u][1 + c4].y;
                tau[4 * c4 + 2] = rb[u][1 + c4].z; tau[4 * c4 + 3] = rb[u][1 + c4].w;
            }
            float dg = gA * (1.0f - bb);
#pragma unroll
            for (int c = 0; c < FC; ++c) dg = fmaf(gC[c], tau[c] - B[c], dg);
            dg *= tm;
            const float tg = tm * g;
            const float galpha = dg * w.beta * w.iota;
            const float gbeta = dg * w.iota * r0.w;
            const float giota = dg * w.beta * r0.w;
            const float gxs = gbeta * w.wy * (w.dx ? 1.f : -1.f) * sc;
            const float gys = gbeta * w.wx * (w.dy ? 1.f : -1.f) * sc;
            const float gs = giota * w.diota;
            float gt[FC];
#pragma unroll
            for (int c = 0; c < FC; ++c) gt[c] = tg * gC[c];
            point_reduce<FC, CAM, SCREEN>(P, i, r0, z, gxs, gys, gs, galpha, gt, go, cg);
#pragma unroll
            for (int c = 0; c < FC; ++c) B[c] = g * tau[c] + (1.0f - g) * B[c];
            bb = g + (1.0f - g) * bb;
        }
    }
    if constexpr (CAM) camera_block_reduce(cg, grad_cam);
}

// --------------------------------------------------------------------------- export

__global__ void __launch_bounds__(kTilePix) k_export(Params P, int what, void* dst)
{
    const int t = P.tile_perm ? (int)__ldg(P.tile_perm + blockIdx.x) : (int)blockIdx.x;
    const TileCoord tc = tile_coord(P, t);
    const LayerGeom& G = P.L[tc.l];
    const int tid = threadIdx.x;
    const int px = tc.tx * kTile + (tid & (kTile - 1)), py = tc.ty * kTile + (tid >> 4);
    const bool valid = px < G.W && py < G.H;
    const int64_t pidx = G.pix_off + (int64_t)py * G.W + px;
    if (what == 1) {
        if (valid) static_cast<uint32_t*>(dst)[pidx] = P.pix_cnt[(size_t)t * kTilePix + tid];
        return;
    }
    int32_t* o = static_cast<int32_t*>(dst);
    if (P.coarse) {
        if (!valid) return;
        const uint32_t meta = P.pix_meta[(size_t)t * kTilePix + tid];
        const int K = (int)(meta & 31u);
        const uint64_t* kp = P.kept + kept_base(t) + tid;
        for (int m = 0; m < kCap; ++m) {
            const uint32_t lo = (uint32_t)kp[m * kTilePix];
            o[pidx * kCap + m] = m < K ? (what == 3 ? (int32_t)(lo & 15u) : (int32_t)(lo >> 4)) : -1;
        }
        return;
    }
    // plain / T_min: the kept lists are stored as kept (point, tile) pairs (k_raster phase F)
    if (valid)
        for (int m = 0; m < kCap; ++m) o[pidx * kCap + m] = -1;
    __syncthreads();
    const uint32_t npair = P.kp_cnt[t];
    for (uint32_t j = tid; j < npair; j += kTilePix) {
        const uint32_t i = (uint32_t)P.kp_key[kept_base(t) + j];
        const uint32_t info = P.kp_info[kept_base(t) + j];
        const int qx0 = (int)(info & 31u) - 1, qy0 = (int)((info >> 5) & 31u) - 1;
        for (int c = 0; c < 4; ++c) {
            if (!(info & (1u << (10 + c)))) continue;
            const int m = (int)((info >> (14 + 4 * c)) & 15u);
            const int64_t q = G.pix_off + (int64_t)(tc.ty * kTile + qy0 + (c >> 1)) * G.W + (tc.tx * kTile + qx0 + (c & 1));
            o[q * kCap + m] = what == 3 ? 0 : (int32_t)i;
        }
    }
}

}  // namespace trips
