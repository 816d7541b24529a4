// binning.cuh -- "collecting" and "splatting" without global atomics.
//
// The paper counts fragments per pixel with atomics, scans the counts and fills per-pixel
// lists.  On B200 the per-pixel (or per-tile) global atomic counters are the bottleneck for
// randomly ordered clouds: thousands of same-address atomics per hot tile serialise in L2.
// This build privatises the counters instead.  A persistent grid of C CTAs splits the points
// into C contiguous ranges; every CTA keeps one counter per pyramid tile in shared memory:
//
//   k_count  per CTA: project its points (Sec. 3.1, Eq. 2), write their screen records,
//            enumerate their (point, tile)
//            pairs (Eq. 4 layers, 2x2 footprints), count them per tile in shared memory;
//            then reserve its slice of each touched tile with ONE global atomic per (CTA,
//            tile) on the tile total; the returned base goes to hist[c][t]
//   k_emit   per CTA, same point range: exclusive scan of the tile totals (every CTA for itself;
//            CTA 0 publishes tile_off), then re-enumerate the pairs from the screen record and
//            place every pair at tile_off[t] + hist[c][t] + (shared-memory cursor)
//   The tile totals are scanned into tile_off by the LAST k_count CTA to finish (completion
//   ticket; TRIPS_TILE_SCAN selects the alternatives: in every k_emit CTA, or a k_tscan launch)
//
// The order of pairs inside a tile's bin is not defined; K4 orders fragments by the full
// (z, i) key (reading Q12), so results do not depend on it.
#pragma once
#include "common.cuh"

namespace trips {

// Where the tile totals become offsets: 2 = the last k_count CTA to finish (a completion
// ticket in tile_cnt[T]), 1 = every k_emit CTA for itself, 0 = a one-CTA k_tscan launch.
#ifndef TRIPS_TILE_SCAN
#define TRIPS_TILE_SCAN 2
#endif
#define TRIPS_EMIT_SCAN (TRIPS_TILE_SCAN == 1)
#ifndef TRIPS_EMIT_PREFETCH
#define TRIPS_EMIT_PREFETCH 0
#endif
#ifndef TRIPS_HIST_FULL_ROW
#define TRIPS_HIST_FULL_ROW 1
#endif
constexpr int kBinThreads = 512;           // threads per binning CTA
#ifndef TRIPS_BIN_CTAS
#define TRIPS_BIN_CTAS 3
#endif
constexpr int kBinCtasPerSm = TRIPS_BIN_CTAS;
constexpr int kMaxTilesSmem = 49152;       // 192 KB of shared-memory counters

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Block-wide exclusive scan of one u32 per thread (any multiple of 32 threads <= 1024).
// Returns the exclusive prefix; *total receives the block sum.  `warp_sums` >= 32 u32.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_sums, uint32_t* total)
{
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < nw ? warp_sums[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (unsigned)o) w += y;
        }
        warp_sums[lane] = w;                 // inclusive warp prefixes
    }
    __syncthreads();
    const uint32_t wpre = warp ? warp_sums[warp - 1] : 0u;
    *total = warp_sums[nw - 1];
    __syncthreads();                         // warp_sums may be reused by the caller
    return wpre + x - v;
}

// The CTA's contiguous point range [b, e).
__device__ __forceinline__ void cta_range(int n, int& b, int& e)
{
    const int per = (n + gridDim.x - 1) / gridDim.x;
    b = min(n, (int)blockIdx.x * per);
    e = min(n, b + per);
}

// tile_off <- exclusive scan of the T tile totals (all threads of the CTA call; s_tot: >= T u32 of
// shared memory, overwritten; s_ws: 32 u32).  Totals staged with coalesced loads (__ldcg: written
// by other CTAs' atomics), each thread scans a contiguous run, one block scan.
__device__ __forceinline__ void scan_tile_totals(const Params& P, uint32_t* s_tot, uint32_t* s_ws)
{
    const int T = P.T;
#pragma unroll 8
    for (int t = threadIdx.x; t < T; t += blockDim.x) s_tot[t] = __ldcg(P.tile_cnt + t);
    __syncthreads();
    const int per = (T + blockDim.x - 1) / blockDim.x;
    const int t0 = min(T, (int)threadIdx.x * per), t1 = min(T, t0 + per);
    uint32_t sa = 0;
    for (int t = t0; t < t1; ++t) sa += s_tot[t];
    uint32_t ta;
    uint32_t pa = block_excl_scan(sa, s_ws, &ta);
    for (int t = t0; t < t1; ++t) {
        const uint32_t a = s_tot[t];
        s_tot[t] = pa;
        pa += a;
    }
    __syncthreads();
#pragma unroll 8
    for (int t = threadIdx.x; t < T; t += blockDim.x) P.tile_off[t] = s_tot[t];
    if (threadIdx.x == 0) P.tile_off[T] = ta;
}

// tile_perm <- the tiles in descending order of their bin size (bucket = bit length of M; order
// within a bucket arbitrary), so the per-tile kernels start the longest tiles in the first wave
// instead of finding them in the last (k_raster -15 us per C4 view).  One CTA; s_off: the
// exclusive tile offsets (scan_tile_totals).  (A 4-class ballot variant measured slower.)
__device__ __forceinline__ void order_tiles_by_size(const Params& P, const uint32_t* s_off)
{
    __shared__ uint32_t s_bk[33];
    const int T = P.T;
    const unsigned lane = lane_id();
    if (threadIdx.x < 33) s_bk[threadIdx.x] = 0;
    __syncthreads();
    auto bucket = [&](int t) -> int {
        const uint32_t m = (t + 1 < T ? s_off[t + 1] : P.tile_off[T]) - s_off[t];
        return 32 - __clz(m);                        // 0 (empty) .. 32
    };
    for (int t0 = 0; t0 < T; t0 += blockDim.x) {     // histogram, one atomic per (warp, bucket)
        const int t = t0 + (int)threadIdx.x;
        const int b = t < T ? bucket(t) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        if (b >= 0 && lane == (unsigned)(__ffs(peers) - 1)) atomicAdd(&s_bk[b], (uint32_t)__popc(peers));
    }
    __syncthreads();
    if (threadIdx.x == 0) {                          // descending buckets: cursor = tiles in larger buckets
        uint32_t acc = 0;
        for (int b = 32; b >= 0; --b) {
            const uint32_t c = s_bk[b];
            s_bk[b] = acc;
            acc += c;
        }
    }
    __syncthreads();
    for (int t0 = 0; t0 < T; t0 += blockDim.x) {
        const int t = t0 + (int)threadIdx.x;
        const int b = t < T ? bucket(t) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        const unsigned leader = (unsigned)(__ffs(peers) - 1);
        uint32_t base = 0;
        if (b >= 0 && lane == leader) base = atomicAdd(&s_bk[b], (uint32_t)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (b >= 0) P.tile_perm[base + __popc(peers & ((1u << lane) - 1u))] = (uint32_t)t;
    }
}

// --------------------------------------------------------------------------- k_count

// Projects every point once (exact block), writes its screen record and depth, and counts its
// (point, tile) pairs in shared-memory counters.
// GLOBAL (plans with more tiles than the shared-memory counters hold, T > kMaxTilesSmem, e.g.
// 8K frames): one global atomic per pair on the tile total instead; the host scans the totals
// (k_gscan_*) and k_emit<true> places pairs with global cursors.
template <int FC, bool GLOBAL>
__global__ void __launch_bounds__(kBinThreads, kBinCtasPerSm) k_count(Params P, int8_t* __restrict__ level_out,
                                                       float* __restrict__ proj_out)
{
    extern __shared__ __align__(16) uint32_t s_hist[];            // [T] (GLOBAL: unused)
    __shared__ uint32_t s_v;
    if (!GLOBAL)
        for (int t = threadIdx.x; t < P.T; t += blockDim.x) s_hist[t] = 0;
    if (threadIdx.x == 0) s_v = 0;
    __syncthreads();
    int b, e;
    cta_range(P.n, b, e);
    uint32_t nvis = 0;
#ifndef TRIPS_COUNT_UNROLL
#define TRIPS_COUNT_UNROLL 1
#endif
#ifndef TRIPS_COUNT_PREFETCH
#define TRIPS_COUNT_PREFETCH 1
#endif
    constexpr int kU = TRIPS_COUNT_UNROLL;        // points per thread per iteration (loads issued together)
#if TRIPS_COUNT_PREFETCH
    // the next point's inputs are loaded while this one is projected and counted
    float nx[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
    if (b + (int)threadIdx.x < e) {
        const int i = b + threadIdx.x;
        const float* q = P.pos + 3 * (size_t)i;
        nx[0] = __ldg(q); nx[1] = __ldg(q + 1); nx[2] = __ldg(q + 2); nx[3] = __ldg(P.sw + i); nx[4] = __ldg(P.alpha + i);
    }
#endif
    for (int i0 = b + threadIdx.x; i0 < e; i0 += kU * blockDim.x) {
      float in[kU][5];
#if TRIPS_COUNT_PREFETCH
      static_assert(kU == 1, "prefetch assumes one point per iteration");
#pragma unroll
      for (int k = 0; k < 5; ++k) in[0][k] = nx[k];
      {
        const int i = i0 + (int)blockDim.x;
        if (i < e) {
            const float* q = P.pos + 3 * (size_t)i;
            nx[0] = __ldg(q); nx[1] = __ldg(q + 1); nx[2] = __ldg(q + 2); nx[3] = __ldg(P.sw + i); nx[4] = __ldg(P.alpha + i);
        }
      }
#else
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = min(i0 + u * (int)blockDim.x, e - 1);
        const float* q = P.pos + 3 * (size_t)i;
        in[u][0] = __ldg(q); in[u][1] = __ldg(q + 1); in[u][2] = __ldg(q + 2);
        in[u][3] = __ldg(P.sw + i); in[u][4] = __ldg(P.alpha + i);
      }
#endif
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * (int)blockDim.x;
        if (i >= e) break;
        float xs = 0.f, ys = 0.f, z = 0.f, s = 0.f;
        const bool vis = project_exact(P.cam, in[u][0], in[u][1], in[u][2], in[u][3], xs, ys, z, s);
        P.geo[i] = make_float4(vis ? xs : 0.f, vis ? ys : 0.f, vis ? s : kCulled, in[u][4]);
        if (!P.tau_direct) {
            // descriptors not gatherable in place (F % 4 != 0 or unaligned): padded copy
            const float* d = P.desc + (size_t)i * P.F;
            float4* r = reinterpret_cast<float4*>(P.tau_copy + (size_t)i * FC);
#pragma unroll
            for (int c = 0; c < FC / 4; ++c) {
                float v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = (4 * c + j < P.F) ? __ldg(d + 4 * c + j) : 0.f;
                r[c] = make_float4(v[0], v[1], v[2], v[3]);
            }
        }
        P.zbuf[i] = z;
        if (level_out) level_out[i] = (int8_t)(vis ? select_levels(s, P.n_layers).code : -1);
        if (proj_out) {
            const float nan = __int_as_float(0x7fc00000);
            reinterpret_cast<float4*>(proj_out)[i] = vis ? make_float4(xs, ys, z, s) : make_float4(nan, nan, nan, nan);
        }
        if (vis) {
            ++nvis;
            if (GLOBAL) for_each_pair(P, xs, ys, s, [&](int t, uint32_t) { atomicAdd(&P.tile_cnt[t], 1u); });
            else for_each_pair(P, xs, ys, s, [&](int t, uint32_t) { atomicAdd(&s_hist[t], 1u); });
        }
      }
    }
    const uint32_t wv = __reduce_add_sync(0xffffffffu, nvis);
    if (lane_id() == 0 && wv) atomicAdd(&s_v, wv);
    __syncthreads();
    if constexpr (GLOBAL) {
        if (threadIdx.x == 0) P.cta_vis[blockIdx.x] = s_v;
        return;
    }
    // reserve this CTA's slice of every tile it touches: tile_cnt[t] holds the running tile
    // total here (k_tscan turns totals into offsets); the returned value is the CTA's offset
    // inside the tile.  One atomic per (CTA, non-empty tile), spread over T addresses; every
    // CTA starts at a different tile so that CTAs finishing together do not queue on the
    // same addresses (a randomly ordered cloud touches almost every tile from every CTA).
    uint32_t* row = P.hist + (size_t)blockIdx.x * P.T;
#ifdef TRIPS_FLUSH_ROT
    const int rot = (int)(((uint64_t)blockIdx.x * P.T) / gridDim.x);
#else
    const int rot = 0;
#endif
#pragma unroll 8
    for (int k = threadIdx.x; k < P.T; k += blockDim.x) {      // unrolled: 8 atomics in flight
        int t = k + rot;
        if (t >= P.T) t -= P.T;
        const uint32_t c = s_hist[t];
#if TRIPS_HIST_FULL_ROW
        // every entry written (untouched tiles: 0), so k_emit reads no uninitialised memory
        row[t] = c ? atomicAdd(&P.tile_cnt[t], c) : 0u;
#else
        if (c) row[t] = atomicAdd(&P.tile_cnt[t], c);
#endif
    }
    if (threadIdx.x == 0) P.cta_vis[blockIdx.x] = s_v;
#if TRIPS_TILE_SCAN == 2
    // completion ticket (tile_cnt[T], zeroed with the totals): the last CTA sees every CTA's
    // reservations and publishes the tile offsets, so k_emit starts placing pairs at once
    __shared__ uint32_t s_last;
    __shared__ uint32_t s_ws[32];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(P.tile_cnt + P.T, 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last) {
        __threadfence();
        scan_tile_totals(P, s_hist, s_ws);
        if (P.tile_perm) order_tiles_by_size(P, s_hist);
    }
#endif
}

// --------------------------------------------------------------------------- k_tscan

// One CTA: tile_off <- exclusive scan of the tile totals (tile_off[T] = M).  The totals are
// staged in shared memory with coalesced loads (T independent loads in flight instead of each
// thread walking its run with dependent ones), each thread sums a contiguous run, one block scan.
__global__ void __launch_bounds__(1024) k_tscan(Params P)
{
    extern __shared__ __align__(16) uint32_t s_tot[];             // [T]
    __shared__ uint32_t s_ws[32];
    const int T = P.T;
#pragma unroll 4
    for (int t = threadIdx.x; t < T; t += blockDim.x) s_tot[t] = P.tile_cnt[t];
    __syncthreads();
    const int per = (T + blockDim.x - 1) / blockDim.x;
    const int t0 = min(T, (int)threadIdx.x * per), t1 = min(T, t0 + per);
    uint32_t sa = 0;
    for (int t = t0; t < t1; ++t) sa += s_tot[t];
    uint32_t ta;
    uint32_t pa = block_excl_scan(sa, s_ws, &ta);
    for (int t = t0; t < t1; ++t) {
        const uint32_t a = s_tot[t];
        s_tot[t] = pa;
        pa += a;
    }
    __syncthreads();
#pragma unroll 4
    for (int t = threadIdx.x; t < T; t += blockDim.x) P.tile_off[t] = s_tot[t];
    if (threadIdx.x == 0) P.tile_off[T] = ta;
}

// --------------------------------------------------------------------------- k_gscan_*

// tile_off <- exclusive scan of tile_cnt[0..T) in global memory (GLOBAL binning), in three
// launches: 1024-entry segments, their totals (one CTA), offsets added; tile_off[T] = total.
__global__ void __launch_bounds__(1024) k_gscan_seg(Params P, uint32_t* bsum)
{
    __shared__ uint32_t ws[32];
    const int t = blockIdx.x * 1024 + threadIdx.x;
    const uint32_t v = t < P.T ? P.tile_cnt[t] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(v, ws, &tot);
    if (t < P.T) P.tile_off[t] = ex;
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_gscan_top(Params P, uint32_t* bsum)
{
    __shared__ uint32_t ws[32];
    const int nseg = (P.T + 1023) / 1024;
    uint32_t carry = 0;
    for (int base = 0; base < nseg; base += 1024) {
        const int e = base + threadIdx.x;
        const uint32_t v = e < nseg ? bsum[e] : 0u;
        uint32_t tot;
        const uint32_t ex = block_excl_scan(v, ws, &tot);
        if (e < nseg) bsum[e] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) P.tile_off[P.T] = carry;
}

__global__ void __launch_bounds__(1024) k_gscan_add(Params P, const uint32_t* bsum)
{
    const int t = blockIdx.x * 1024 + threadIdx.x;
    if (t < P.T) P.tile_off[t] += bsum[blockIdx.x];
}

// --------------------------------------------------------------------------- k_emit

// Same point partition as k_count: re-enumerates each visible point's pairs from its screen
// record (no projection) and places them at tile_off[t] + this CTA's slice + shared cursor.
template <bool GLOBAL>
__global__ void __launch_bounds__(kBinThreads, kBinCtasPerSm) k_emit(Params P)
{
    extern __shared__ __align__(16) uint32_t s_cur[];             // [T] fill cursors
    if constexpr (GLOBAL) {
        // tile_cnt was re-zeroed after the scan: it is the per-tile fill cursor
        int b, e;
        cta_range(P.n, b, e);
        for (int i = b + threadIdx.x; i < e; i += blockDim.x) {
            const float4 r0 = __ldg(P.geo + i);
            if (!(r0.z >= 0.f)) continue;                         // culled
            const uint64_t key = ((uint64_t)__float_as_uint(__ldg(P.zbuf + i)) << 32) | (uint32_t)i;
            for_each_pair(P, r0.x, r0.y, r0.z, [&](int t, uint32_t o) {
                const uint32_t pos = P.tile_off[t] + atomicAdd(&P.tile_cnt[t], 1u);
                P.bin_key[pos] = key;
                P.bin_orig[pos] = (uint16_t)o;
            });
        }
        return;
    }
    const uint32_t* row = P.hist + (size_t)blockIdx.x * P.T;
#if TRIPS_EMIT_SCAN
    // every CTA scans the tile totals itself (T independent coalesced loads, one block scan):
    // no separate k_tscan launch; CTA 0 publishes the offsets for the raster
    __shared__ uint32_t s_ws[32];
    const int T = P.T;
#pragma unroll 8
    for (int t = threadIdx.x; t < T; t += blockDim.x) s_cur[t] = __ldcg(P.tile_cnt + t);
    __syncthreads();
    {
        const int per = (T + blockDim.x - 1) / blockDim.x;
        const int t0 = min(T, (int)threadIdx.x * per), t1 = min(T, t0 + per);
        uint32_t sa = 0;
        for (int t = t0; t < t1; ++t) sa += s_cur[t];
        uint32_t ta;
        uint32_t pa = block_excl_scan(sa, s_ws, &ta);
        for (int t = t0; t < t1; ++t) {
            const uint32_t a = s_cur[t];
            s_cur[t] = pa;
            pa += a;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) P.tile_off[T] = ta;
    }
    __syncthreads();
    // entries of tiles this CTA never touches are 0 (TRIPS_HIST_FULL_ROW) and never used
#pragma unroll 8
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        const uint32_t o = s_cur[t];
        if (blockIdx.x == 0) P.tile_off[t] = o;
        s_cur[t] = o + row[t];
    }
#else
    // entries of tiles this CTA never touches are 0 (TRIPS_HIST_FULL_ROW) and never used
#pragma unroll 8
    for (int t = threadIdx.x; t < P.T; t += blockDim.x) s_cur[t] = P.tile_off[t] + row[t];
#endif
    __syncthreads();
    int b, e;
    cta_range(P.n, b, e);
#if TRIPS_EMIT_PREFETCH
    // the next point's record is loaded while this one's pairs are placed
    float4 nr = make_float4(0.f, 0.f, -1.f, 0.f);
    float nz = 0.f;
    if (b + (int)threadIdx.x < e) { nr = __ldg(P.geo + b + threadIdx.x); nz = __ldg(P.zbuf + b + threadIdx.x); }
    for (int i = b + threadIdx.x; i < e; i += blockDim.x) {
        const float4 r0 = nr;
        const float z = nz;
        if (i + (int)blockDim.x < e) { nr = __ldg(P.geo + i + blockDim.x); nz = __ldg(P.zbuf + i + blockDim.x); }
        if (!(r0.z >= 0.f)) continue;                             // culled
        const uint64_t key = ((uint64_t)__float_as_uint(z) << 32) | (uint32_t)i;
#else
    for (int i = b + threadIdx.x; i < e; i += blockDim.x) {
        const float4 r0 = __ldg(P.geo + i);
        if (!(r0.z >= 0.f)) continue;                             // culled
        const uint64_t key = ((uint64_t)__float_as_uint(__ldg(P.zbuf + i)) << 32) | (uint32_t)i;
#endif
        for_each_pair(P, r0.x, r0.y, r0.z, [&](int t, uint32_t o) {
            const uint32_t pos = atomicAdd(&s_cur[t], 1u);
            P.bin_key[pos] = key;
            P.bin_orig[pos] = (uint16_t)o;
        });
    }
}

// --------------------------------------------------------------------------- k_stats

// On-demand statistics (trips_read_stats): reduces the per-pixel list lengths and the
// per-CTA visible counts; nothing on the hot path touches a shared counter.
__global__ void __launch_bounds__(256) k_stats(Params P, int ctas, int npix, int ntiles_kp)
{
    unsigned long long frag = 0, kept = 0, trunc = 0, mx = 0, vis = 0, kpairs = 0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ntiles_kp; j += gridDim.x * blockDim.x) kpairs += P.kp_cnt[j];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < npix; j += gridDim.x * blockDim.x) {
        const unsigned long long c = P.pix_cnt[j];
        frag += c;
        kept += c < (unsigned long long)kCap ? c : (unsigned long long)kCap;
        trunc += c > (unsigned long long)kCap;
        mx = c > mx ? c : mx;
    }
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ctas; j += gridDim.x * blockDim.x) vis += P.cta_vis[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        frag += __shfl_xor_sync(0xffffffffu, frag, o);
        kept += __shfl_xor_sync(0xffffffffu, kept, o);
        trunc += __shfl_xor_sync(0xffffffffu, trunc, o);
        vis += __shfl_xor_sync(0xffffffffu, vis, o);
        kpairs += __shfl_xor_sync(0xffffffffu, kpairs, o);
        const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = m2 > mx ? m2 : mx;
    }
    if (lane_id() == 0) {
        if (frag) atomicAdd(&P.stats[S_FRAG], frag);
        if (kept) atomicAdd(&P.stats[S_KEPT], kept);
        if (trunc) atomicAdd(&P.stats[S_TRUNC], trunc);
        if (vis) atomicAdd(&P.stats[S_VISIBLE], vis);
        if (kpairs) atomicAdd(&P.stats[S_KPAIRS], kpairs);
        if (mx) atomicMax(&P.stats[S_MAXLIST], mx);
    }
}

}  // namespace trips
