// kernels.cuh -- the five kernels of the B200 TRIPS rasterizer.
//
//   K1 k_project   per point: Sec. 3.1 projection + Eq. (2) size + Eq. (4) layers, writes the
//                  point's 16-B-aligned screen record, counts (point, tile) pairs per 16x16
//                  pyramid tile with warp-aggregated atomics.          ("collecting")
//   K2 k_scan      one CTA: exclusive scan of the per-tile pair counts (and of the per-tile
//                  kept-list capacity).                                ("offset scan")
//   K3 k_bin       per point: same pair enumeration, warp-aggregated cursor atomics, writes the
//                  point index into its tiles' bins.                   ("splatting")
//   K4 k_raster    per tile (CTA of 256 = 16x16 pixel threads): stages chunks of the tile's
//                  points, builds the per-pixel fragment lists in shared memory (counting sort
//                  by pixel), keeps the 16 smallest (z, i) keys per pixel in registers with
//                  sorting/merging networks, then blends front to back and stores the sorted
//                  kept lists.                     ("combined sorting and accumulation", 290-295)
//   K5 k_backward  per tile pixel: replays the kept list (forward for T_m, then reverse suffix
//                  recurrences), chains screen-space gradients to world space per fragment and
//                  accumulates with 16-byte vector reductions (red.global.add.v4.f32).
#pragma once
#include "common.cuh"

namespace trips {

constexpr int kChunk = 512;                 // (point, tile) pairs staged per K4 iteration
constexpr int kPairsPerThread = kChunk / kTilePix;

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt()
{
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d)
{
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
                 :: "l"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// Block-wide exclusive scan of one u32 per thread (256 threads).  Returns the exclusive
// prefix; *total receives the block sum.  Uses `warp_sums` (>= 8 u32 of shared memory).
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t* warp_sums, uint32_t* total)
{
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kTilePix / 32; ++w) {
        const uint32_t ws = warp_sums[w];
        wpre += (w < (int)warp) ? ws : 0u;
        tot += ws;
    }
    __syncthreads();                        // warp_sums may be reused by the caller
    *total = tot;
    return wpre + x - v;
}

// --------------------------------------------------------------------------- K1 project

template <int FC>
__global__ void __launch_bounds__(256) k_project(Params P, int8_t* __restrict__ level_out,
                                                 float* __restrict__ proj_out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = i < P.n;
    int tiles[8];
    int np = 0, nf = 0;
    bool vis = false;
    if (in) {
        const float X = P.pos[3 * (size_t)i + 0], Y = P.pos[3 * (size_t)i + 1], Z = P.pos[3 * (size_t)i + 2];
        const float sw = P.sw[i];
        float xs = 0.f, ys = 0.f, z = 0.f, s = 0.f;
        vis = project_exact(P.cam, X, Y, Z, sw, xs, ys, z, s);
        int code = -1;
        if (vis) {
            np = enumerate_pairs(P, xs, ys, s, tiles, &nf);
            code = select_levels(s, P.n_layers).code;
        }
        float4* r = reinterpret_cast<float4*>(P.rec + (size_t)i * P.RS);
        r[0] = make_float4(vis ? xs : 0.f, vis ? ys : 0.f, vis ? s : kCulled, P.alpha[i]);
        const float* d = P.desc + (size_t)i * P.F;
#pragma unroll
        for (int c = 0; c < FC / 4; ++c) {
            float v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = (4 * c + j < P.F) ? d[4 * c + j] : 0.f;
            r[1 + c] = make_float4(v[0], v[1], v[2], v[3]);
        }
        P.zbuf[i] = vis ? z : __int_as_float(0x7f800000);
        if (level_out) level_out[i] = (int8_t)code;
        if (proj_out) {
            const float nan = __int_as_float(0x7fc00000);
            reinterpret_cast<float4*>(proj_out)[i] = vis ? make_float4(xs, ys, z, s) : make_float4(nan, nan, nan, nan);
        }
    }
    // warp-aggregated per-tile pair counts
    const unsigned lane = lane_id();
    const int wmax = __reduce_max_sync(0xffffffffu, np);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k >= wmax) break;
        const int t = k < np ? tiles[k] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, t);
        if (t >= 0 && lane == (unsigned)(__ffs(peers) - 1)) atomicAdd(&P.tile_cnt[t], (uint32_t)__popc(peers));
    }
    // statistics
    const unsigned nvis = __popc(__ballot_sync(0xffffffffu, in && vis));
    const unsigned ncul = __popc(__ballot_sync(0xffffffffu, in && !vis));
    if (lane == 0) {
        if (nvis) atomicAdd(&P.stats[S_VISIBLE], (unsigned long long)nvis);
        if (ncul) atomicAdd(&P.stats[S_CULLED], (unsigned long long)ncul);
    }
}

// --------------------------------------------------------------------------- K2 scan

__global__ void __launch_bounds__(1024) k_scan(Params P)
{
    __shared__ uint32_t s_a[32], s_b[32];
    const int T = P.T;
    const int per = (T + blockDim.x - 1) / blockDim.x;
    const int b = threadIdx.x * per, e = min(T, b + per);
    uint32_t sa = 0, sb = 0;
    for (int t = b; t < e; ++t) {
        const uint32_t c = P.tile_cnt[t];
        sa += c;
        sb += min(4u * c, (uint32_t)(kTilePix * kCap));
    }
    // block exclusive scan of (sa, sb)
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t xa = sa, xb = sb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
        if (lane >= (unsigned)o) { xa += ya; xb += yb; }
    }
    if (lane == 31) { s_a[warp] = xa; s_b[warp] = xb; }
    __syncthreads();
    if (warp == 0) {
        uint32_t wa = s_a[lane], wb = s_b[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, wa, o), yb = __shfl_up_sync(0xffffffffu, wb, o);
            if (lane >= (unsigned)o) { wa += ya; wb += yb; }
        }
        s_a[lane] = wa; s_b[lane] = wb;            // inclusive warp totals
    }
    __syncthreads();
    uint32_t pa = (warp ? s_a[warp - 1] : 0u) + xa - sa;
    uint32_t pb = (warp ? s_b[warp - 1] : 0u) + xb - sb;
    for (int t = b; t < e; ++t) {
        const uint32_t c = P.tile_cnt[t];
        P.tile_off[t] = pa;
        P.tile_cur[t] = pa;
        P.tile_kbase[t] = pb;
        pa += c;
        pb += min(4u * c, (uint32_t)(kTilePix * kCap));
    }
    if (threadIdx.x == blockDim.x - 1) {
        P.tile_off[T] = pa;
        P.tile_kbase[T] = pb;
        P.stats[S_PAIRS] = pa;
    }
}

// --------------------------------------------------------------------------- K3 bin

__global__ void __launch_bounds__(256) k_bin(Params P)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int tiles[8];
    int np = 0;
    if (i < P.n) {
        const float4 r = reinterpret_cast<const float4*>(P.rec + (size_t)i * P.RS)[0];
        if (r.z >= 0.f) np = enumerate_pairs(P, r.x, r.y, r.z, tiles, nullptr);
    }
    const unsigned lane = lane_id();
    const int wmax = __reduce_max_sync(0xffffffffu, np);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k >= wmax) break;
        const int t = k < np ? tiles[k] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, t);
        if (t >= 0) {
            const int leader = __ffs(peers) - 1;
            uint32_t base = 0;
            if (lane == (unsigned)leader) base = atomicAdd(&P.tile_cur[t], (uint32_t)__popc(peers));
            base = __shfl_sync(peers, base, leader);
            P.bins[base + __popc(peers & lanemask_lt())] = (uint32_t)i;
        }
    }
}

// --------------------------------------------------------------------------- K4 raster

// Sorting network (bitonic, ascending) over 16 u64 keys held in registers.
__device__ __forceinline__ void sort16(uint64_t (&t)[16])
{
#pragma unroll
    for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    if ((i & k) == 0) cswap(t[i], t[l]);
                    else cswap(t[l], t[i]);
                }
            }
}

// r (sorted asc) <- the 16 smallest of r U t (both sorted asc): bitonic split + clean.
__device__ __forceinline__ void merge16(uint64_t (&r)[16], const uint64_t (&t)[16])
{
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = r[j] < t[15 - j] ? r[j] : t[15 - j];
#pragma unroll
    for (int d = 8; d > 0; d >>= 1)
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if ((i & d) == 0) cswap(r[i], r[i + d]);
}

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

template <int FC>
__global__ void __launch_bounds__(kTilePix, 2) k_raster(Params P, float* __restrict__ pyramid, int save)
{
    __shared__ uint64_t s_keys[kChunk * 4];
    __shared__ uint32_t s_cnt[kTilePix];
    __shared__ uint32_t s_base[kTilePix];
    __shared__ uint32_t s_warp[32];

    const int t = blockIdx.x;
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

    for (uint32_t c0 = b0; c0 < b1; c0 += kChunk) {
        const int m = (int)min((uint32_t)kChunk, b1 - c0);
        s_cnt[tid] = 0;
        __syncthreads();
        // phase A: stage this chunk's points, compute their fragments in this tile
        uint64_t fk[kPairsPerThread][4];
        uint32_t fq[kPairsPerThread][4];             // (q | rank << 8), 0xffffffff = none
#pragma unroll
        for (int k = 0; k < kPairsPerThread; ++k) {
#pragma unroll
            for (int c = 0; c < 4; ++c) fq[k][c] = 0xffffffffu;
            const int j = tid + k * kTilePix;
            if (j < m) {
                const uint32_t i = P.bins[c0 + j];
                const float4 r0 = reinterpret_cast<const float4*>(P.rec + (size_t)i * P.RS)[0];
                const float z = P.zbuf[i];
                const uint64_t key = ((uint64_t)__float_as_uint(z) << 32) | i;
                Foot f;
                if (footprint(r0.x, r0.y, tc.l, G.W, G.H, f)) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int qx = f.x0 + (c & 1), qy = f.y0 + (c >> 1);
                        if (qx >= x_lo && qx < x_lo + kTile && qx < G.W && qy >= y_lo && qy < y_lo + kTile &&
                            qy < G.H) {
                            const uint32_t q = (uint32_t)((qy - y_lo) * kTile + (qx - x_lo));
                            const uint32_t rank = atomicAdd(&s_cnt[q], 1u);
                            fk[k][c] = key;
                            fq[k][c] = q | (rank << 8);
                        }
                    }
                }
            }
        }
        __syncthreads();
        uint32_t chunk_total;
        const uint32_t my_cnt = s_cnt[tid];
        const uint32_t my_base = block_excl_scan256(my_cnt, s_warp, &chunk_total);
        s_base[tid] = my_base;
        __syncthreads();
        // phase B: counting-sort scatter by pixel
#pragma unroll
        for (int k = 0; k < kPairsPerThread; ++k)
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (fq[k][c] != 0xffffffffu) s_keys[s_base[fq[k][c] & 0xffu] + (fq[k][c] >> 8)] = fk[k][c];
        __syncthreads();
        // phase C: merge this pixel's new fragments into its running top-16
        for (uint32_t g = 0; g < my_cnt; g += 16) {
            uint64_t tk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) tk[j] = (g + j < my_cnt) ? s_keys[my_base + g + j] : kKeyMax;
            sort16(tk);
            merge16(r, tk);
        }
        total += my_cnt;
        __syncthreads();
    }

    // phase D: front-to-back blend of the kept list (Eqs. 5-6; alpha_m := gamma_m, Q10)
    const int K = valid ? (int)min(total, (uint32_t)kCap) : 0;
    float C[FC];
#pragma unroll
    for (int c = 0; c < FC; ++c) C[c] = 0.f;
    float A = 0.f, T = 1.f;
#pragma unroll
    for (int mm = 0; mm < kCap; ++mm) {
        if (mm < K && T > 0.f) {                        // T == 0 exactly: later terms vanish
            const uint32_t i = (uint32_t)r[mm];
            const float4* rp = reinterpret_cast<const float4*>(P.rec + (size_t)i * P.RS);
            const float4 r0 = rp[0];
            const FragW w = frag_weights(r0, tc.l, P.n_layers, px, py);
            const float tg = T * w.gamma;
#pragma unroll
            for (int c4 = 0; c4 < FC / 4; ++c4) {
                const float4 tau = rp[1 + c4];
                C[4 * c4 + 0] = fmaf(tg, tau.x, C[4 * c4 + 0]);
                C[4 * c4 + 1] = fmaf(tg, tau.y, C[4 * c4 + 1]);
                C[4 * c4 + 2] = fmaf(tg, tau.z, C[4 * c4 + 2]);
                C[4 * c4 + 3] = fmaf(tg, tau.w, C[4 * c4 + 3]);
            }
            A += tg;
            T = T * (1.0f - w.gamma);
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

    // phase E: store the sorted kept lists and per-pixel metadata
    uint32_t ktot;
    const uint32_t koff = block_excl_scan256((uint32_t)K, s_warp, &ktot);
    P.pix_cnt[(size_t)t * kTilePix + tid] = valid ? total : 0u;
    P.pix_meta[(size_t)t * kTilePix + tid] = (koff << 5) | (uint32_t)K;
    if (save) {
        uint64_t* kp = P.kept + P.tile_kbase[t] + koff;
#pragma unroll
        for (int mm = 0; mm < kCap; ++mm)
            if (mm < K) kp[mm] = r[mm];
    }
    // statistics (n_frag, n_kept, n_trunc, max_list)
    const uint32_t vt = valid ? total : 0u;
    const uint32_t wf = __reduce_add_sync(0xffffffffu, vt);
    const uint32_t wtr = __popc(__ballot_sync(0xffffffffu, vt > (uint32_t)kCap));
    const uint32_t wmx = __reduce_max_sync(0xffffffffu, vt);
    if (lane_id() == 0) {
        if (wf) atomicAdd(&P.stats[S_FRAG], (unsigned long long)wf);
        if (wtr) atomicAdd(&P.stats[S_TRUNC], (unsigned long long)wtr);
        if (wmx) atomicMax(&P.stats[S_MAXLIST], (unsigned long long)wmx);
    }
    if (tid == 0 && ktot) atomicAdd(&P.stats[S_KEPT], (unsigned long long)ktot);
}

// --------------------------------------------------------------------------- K5 backward

template <int FC>
__global__ void __launch_bounds__(kTilePix) k_backward(Params P, const float* __restrict__ gpyr,
                                                       float* __restrict__ grad)
{
    const int t = blockIdx.x;
    const TileCoord tc = tile_coord(P, t);
    const LayerGeom& G = P.L[tc.l];
    const int tid = threadIdx.x;
    const int px = tc.tx * kTile + (tid & (kTile - 1)), py = tc.ty * kTile + (tid >> 4);
    const uint32_t meta = P.pix_meta[(size_t)t * kTilePix + tid];
    const int K = (int)(meta & 31u);
    if (K == 0) return;
    const uint64_t* kp = P.kept + P.tile_kbase[t] + (meta >> 5);

    // upstream gradient of this pixel: gC (F channels) and gA
    const int64_t plane = (int64_t)G.W * G.H;
    const float* gp = gpyr + G.float_off + (int64_t)py * G.W + px;
    float gC[FC];
#pragma unroll
    for (int c = 0; c < FC; ++c) gC[c] = (c < P.F) ? gp[c * plane] : 0.f;
    const float gA = gp[P.F * plane];

    // forward replay: gamma_m and T_m (Eq. 6)
    float gam[kCap], Tm[kCap];
    float T = 1.f;
#pragma unroll
    for (int mm = 0; mm < kCap; ++mm) {
        gam[mm] = 0.f; Tm[mm] = 0.f;
        if (mm < K) {
            const uint32_t i = (uint32_t)kp[mm];
            const float4 r0 = reinterpret_cast<const float4*>(P.rec + (size_t)i * P.RS)[0];
            const FragW w = frag_weights(r0, tc.l, P.n_layers, px, py);
            gam[mm] = w.gamma;
            Tm[mm] = T;
            T = T * (1.0f - w.gamma);
        }
    }
    // reverse replay with suffix recurrences (division-free)
    float B[FC];
#pragma unroll
    for (int c = 0; c < FC; ++c) B[c] = 0.f;
    float bb = 0.f;
    const float sc = pow2_neg(tc.l);
    const Cam& cam = P.cam;
#pragma unroll
    for (int mm = kCap - 1; mm >= 0; --mm) {
        if (mm < K) {
            const uint64_t key = kp[mm];
            const uint32_t i = (uint32_t)key;
            const float z = __uint_as_float((uint32_t)(key >> 32));
            const float4* rp = reinterpret_cast<const float4*>(P.rec + (size_t)i * P.RS);
            const float4 r0 = rp[0];
            const FragW w = frag_weights(r0, tc.l, P.n_layers, px, py);
            const float g = gam[mm], tm = Tm[mm];
            float tau[FC];
#pragma unroll
            for (int c4 = 0; c4 < FC / 4; ++c4) {
                const float4 v = rp[1 + c4];
                tau[4 * c4 + 0] = v.x; tau[4 * c4 + 1] = v.y; tau[4 * c4 + 2] = v.z; tau[4 * c4 + 3] = v.w;
            }
            // d out / d gamma_m = T_m (<gC, tau_m - B_m> + gA (1 - b_m))
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
            // projection chain (Eq. 2, Sec. 3.1)
            const float iz = 1.0f / z;
            const float gpx = gxs * cam.fx * iz, gpy = gys * cam.fy * iz;
            const float gpz = -(gxs * (r0.x - cam.cx) + gys * (r0.y - cam.cy) + gs * r0.z) * iz;
            const float gX = cam.R[0] * gpx + cam.R[3] * gpy + cam.R[6] * gpz;
            const float gY = cam.R[1] * gpx + cam.R[4] * gpy + cam.R[7] * gpz;
            const float gZ = cam.R[2] * gpx + cam.R[5] * gpy + cam.R[8] * gpz;
            const float gsw = gs * cam.f * iz;
            float* grow = grad + (size_t)i * P.G;
            red_add_v4(grow, gX, gY, gZ, gsw);
            // (alpha, tau[0..FC-1]) in 16-B chunks
            float v[FC + 4];
            v[0] = galpha;
#pragma unroll
            for (int c = 0; c < FC; ++c) v[1 + c] = tg * gC[c];
            v[FC + 1] = 0.f; v[FC + 2] = 0.f; v[FC + 3] = 0.f;
#pragma unroll
            for (int c4 = 0; c4 < (FC + 4) / 4; ++c4)
                if (4 * c4 < P.F + 1) red_add_v4(grow + 4 + 4 * c4, v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
            // suffix recurrences
#pragma unroll
            for (int c = 0; c < FC; ++c) B[c] = g * tau[c] + (1.0f - g) * B[c];
            bb = g + (1.0f - g) * bb;
        }
    }
}

// --------------------------------------------------------------------------- export

__global__ void __launch_bounds__(kTilePix) k_export(Params P, int what, void* dst)
{
    const int t = blockIdx.x;
    const TileCoord tc = tile_coord(P, t);
    const LayerGeom& G = P.L[tc.l];
    const int tid = threadIdx.x;
    const int px = tc.tx * kTile + (tid & (kTile - 1)), py = tc.ty * kTile + (tid >> 4);
    if (px >= G.W || py >= G.H) return;
    const int64_t pidx = G.pix_off + (int64_t)py * G.W + px;
    if (what == 1) {
        static_cast<uint32_t*>(dst)[pidx] = P.pix_cnt[(size_t)t * kTilePix + tid];
    } else {
        const uint32_t meta = P.pix_meta[(size_t)t * kTilePix + tid];
        const int K = (int)(meta & 31u);
        const uint64_t* kp = P.kept + P.tile_kbase[t] + (meta >> 5);
        int32_t* o = static_cast<int32_t*>(dst) + pidx * kCap;
        for (int m = 0; m < kCap; ++m) o[m] = m < K ? (int32_t)(uint32_t)kp[m] : -1;
    }
}

}  // namespace trips
