// decoder.cuh -- the gated-convolution decoder over the image pyramid:
// "a single gated convolution in each layer with a self-bypass connection and a feature size of
// 32 ... a bilinear upsampling operation for all layers except the final one, merging the output
// with the subsequent level" (Fig. fig:conv; readings D1-D8 in DESIGN.md).
//
// Per layer l (coarsest first), three steps on the GPU:
//   k_dec_prep   X_l[y][x][64] fp16 (NHWC): channels 0-31 = bilinear 2x upsampling of y_{l+1}
//                (half-pixel centres, edge-clamped, cropped), 32-32+F = the pyramid layer's F
//                features + opacity, the rest 0 (memory-bound elementwise pass);
//   k_dec_conv   the 3x3 gated convolution + 1x1 bypass as ONE implicit GEMM on the tcgen05
//                tensor cores: D[128 pixels][96] += A_tap[128][64] . B_tap[96][64]^T over the 9
//                taps, where A_tap is the row segment of X_l shifted by the tap (a TMA box of the
//                3-D tensor map: out-of-image taps are zero-filled by the TMA unit = the conv's
//                zero padding) and B_tap the packed weights [f (32) | g (32) | bypass (32, centre
//                tap only)]; fp16 operands, fp32 accumulators in TMEM.  Epilogue straight from
//                TMEM: y = ELU(f + bf) * sigmoid(g + bg) + bypass, stored fp32 NHWC -- or, at the
//                finest layer, the 1x1 output projection Wo y + bo, stored planar [out][H][W];
//   (k_dec_pack  once per call: the flat fp32 parameter vector -> the packed fp16 B operands.)
//
// k_dec_conv is warp-specialised and persistent (one CTA per SM): warp 0 issues the TMA loads of
// the A taps into a 4-stage ring (mbarrier full/empty pairs), warp 1 issues the tcgen05.mma
// (one elected lane, 4 x K16 per tap), warps 2-9 drain the accumulator (double-buffered in TMEM,
// 2 x 96 columns; two warps per TMEM lane quarter, 16 hidden channels each) while the next tile's
// MMAs run.  The B operands of all 9 taps (108 KB) stay
// resident in shared memory for the whole launch.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace trips {

constexpr int kDecHidden = 32;             // "a feature size of 32"
constexpr int kDecXC = 64;                 // X channels: 32 upsampled + F + 1 pyramid, zero-padded
constexpr int kDecN = 96;                  // GEMM N: f (32) | g (32) | bypass (32)
constexpr int kDecM = 128;                 // pixels per tile (one UMMA M)
constexpr int kDecTaps = 9;
#ifndef TRIPS_DEC_STAGES
#define TRIPS_DEC_STAGES 6
#endif
constexpr int kDecStages = TRIPS_DEC_STAGES;    // A-tap ring depth (smem: 108 KB B + 16 KB per stage)
constexpr int kDecABytes = kDecM * kDecXC * 2;          // 16 KB per tap
constexpr int kDecBBytes = kDecN * kDecXC * 2;          // 12 KB per tap
#ifndef TRIPS_DEC_EPI16
#define TRIPS_DEC_EPI16 1
#endif
// EPI16: 16 epilogue warps, 4 per TMEM lane quarter, each taking every 4th tile whole (32 channels,
// in two 16-channel chunks); else 8 warps, 2 per lane quarter, 16 channels each of every tile
constexpr int kDecEpiWarps = TRIPS_DEC_EPI16 ? 16 : 8;
constexpr int kDecEpiPerTile = TRIPS_DEC_EPI16 ? 4 : 8;  // warps that arrive on a tile's tempty
constexpr int kDecThreads = 64 + 32 * kDecEpiWarps;     // TMA warp, MMA warp, epilogue warps
constexpr int kDecMaxOut = 32;
#ifndef TRIPS_DEC_ROWS
#define TRIPS_DEC_ROWS 1           // 1: row boxes reused across taps and tiles; 0: one box per tap
#endif
#ifndef TRIPS_DEC_BO
#define TRIPS_DEC_BO 0             // descriptor base_offset for row-shifted operands (0 or the address phase)
#endif
constexpr int kDecRowPix = kDecM + 2;                   // a row box: the tile's 128 pixels + 1 halo each side
constexpr int kDecRowBytes = kDecRowPix * kDecXC * 2;   // 16640 B written by the TMA
constexpr int kDecRowSlot = 17 * 1024;                  // slots 1024-B aligned (swizzle phase)
#ifndef TRIPS_DEC_ACC
#define TRIPS_DEC_ACC 4
#endif
constexpr int kDecAcc = TRIPS_DEC_ACC;                  // TMEM accumulators in flight (x 96 columns)
constexpr int kDecTmemCols = kDecAcc * 96 <= 256 ? 256 : 512;
#ifndef TRIPS_DEC_SLOTS
#define TRIPS_DEC_SLOTS 4            // 6 (prefetch 3 rows ahead) measured 0.525 vs 0.511 ms per frame
#endif
constexpr int kDecRowSlots = TRIPS_DEC_SLOTS;           // rows y-1, y, y+1 in use + the next ones loading
constexpr int kDecMdone = 4;                            // per-tile MMA-completion barriers (tile mod 4)
constexpr int kDecSmem = TRIPS_DEC_ROWS ? 1024 + kDecTaps * kDecBBytes + kDecRowSlots * kDecRowSlot + 256
                                        : 1024 + kDecTaps * kDecBBytes + kDecStages * kDecABytes + 256;

// ----------------------------------------------------------------------------- PTX wrappers

__device__ __forceinline__ uint32_t dec_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void dec_mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(dec_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void dec_mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(dec_smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void dec_mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(dec_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void dec_mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra WAIT_%=;\n\t}" :: "r"(dec_smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void dec_tma_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2)
{
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 :: "r"(dec_smem_u32(dst)), "l"(map), "r"(dec_smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void dec_tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 :: "r"(dec_smem_u32(dst)), "l"(map), "r"(dec_smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void dec_tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void dec_tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand in the canonical 128-byte-swizzled layout (8-row groups of 128-byte rows,
// 1024 B apart; the TMA box writes exactly this): start >> 4, LBO = 1 (unused for swizzled
// K-major), SBO = 1024 B >> 4, version 1 (sm_100), layout SWIZZLE_128B (2).
__device__ __forceinline__ uint64_t dec_desc(uint32_t saddr)
{
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3fffu) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
#if TRIPS_DEC_BO
    d |= (uint64_t)((saddr >> 7) & 7u) << 49;        // start not on a 1024-B swizzle repeat: its phase
#endif
    return d;
}
// instruction descriptor, kind::f16: D f32 (bits 4-5 = 1), A = B = f16 (0), both K-major,
// N >> 3 at bits 17-22, M >> 4 at bits 24-28
constexpr uint32_t kDecIdesc = (1u << 4) | ((uint32_t)(kDecN >> 3) << 17) | ((uint32_t)(kDecM >> 4) << 24);
// the bypass block (columns 64-95) is non-zero only in the centre tap: the other 8 taps issue N = 64
#ifndef TRIPS_DEC_N64
#define TRIPS_DEC_N64 1
#endif
constexpr uint32_t kDecIdesc64 = (1u << 4) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(kDecM >> 4) << 24);

__device__ __forceinline__ void dec_umma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate,
                                         uint32_t idesc = kDecIdesc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void dec_umma_commit(uint64_t* bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(dec_smem_u32(bar)) : "memory");
}
// 32 lanes x 16 consecutive fp32 columns: thread t of the warp gets lane (base + t), columns c..c+15
// (no wait: the caller issues tcgen05.wait::ld once after all its loads)
__device__ __forceinline__ void dec_tmem_ld16(uint32_t taddr, uint32_t (&r)[16])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                 "%14, %15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
}
__device__ __forceinline__ void dec_tmem_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ----------------------------------------------------------------------------- parameters

struct DecLayer {
    int32_t H, W;                  // layer size
    int32_t Hc, Wc;                // next-coarser layer size (0 at the coarsest)
    int64_t pyr_off;               // float offset of the layer in the planar pyramid
    int64_t prm_off;               // float offset of the layer's block in the flat parameters
    int32_t C;                     // input channels of the block (F + 1 coarsest, 32 + F + 1 else)
    int32_t coarsest;
};

struct DecParams {
    int32_t n_layers, F, out_ch;
    int32_t xc;                    // X channels stored: 48 when F + 1 <= 16, else 64 (TMA reads 64, the
                                   // channels beyond xc come back zero-filled and their K steps are skipped)
    DecLayer L[16];
    int64_t prm_out;               // float offset of Wo [out][32], bo [out]
    const float* prm;              // flat fp32 parameters (oracle/decoder.py param_layout)
    const float* pyramid;          // the rasterizer's planar pyramid
    __half* wpack;                 // [n][9][96][64] packed B operands
    __half* X;                     // [H_l][W_l][64] current layer input
    float* Y[2];                   // [H_l][W_l][32] hidden outputs (ping-pong by layer parity)
    float* out;                    // [out][H][W]
};

// k_dec_pack: B[l][t][n][k] = Wf / Wg (3x3 tap t = (dy+1)*3 + (dx+1)) or Wb (centre tap), with
// the block's input channel c at X channel k = c (32 + c at the coarsest layer: no upsampled part).
__global__ void __launch_bounds__(256) k_dec_pack(DecParams D)
{
    const int64_t total = (int64_t)D.n_layers * kDecTaps * kDecN * kDecXC;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e % kDecXC);
        const int n = (int)((e / kDecXC) % kDecN);
        const int t = (int)((e / (kDecXC * kDecN)) % kDecTaps);
        const int l = (int)(e / ((int64_t)kDecXC * kDecN * kDecTaps));
        const DecLayer& L = D.L[l];
        const int c = L.coarsest ? k - kDecHidden : k;
        float v = 0.f;
        if (c >= 0 && c < L.C) {
            const float* P = D.prm + L.prm_off;
            const int64_t wsz = (int64_t)kDecHidden * L.C * 9;
            if (n < 32) v = P[((int64_t)n * L.C + c) * 9 + t];                                   // Wf
            else if (n < 64) v = P[wsz + kDecHidden + ((int64_t)(n - 32) * L.C + c) * 9 + t];    // Wg
            else if (t == 4) v = P[2 * (wsz + kDecHidden) + (int64_t)(n - 64) * L.C + c];       // Wb
        }
        D.wpack[e] = __float2half_rn(v);
    }
}

// k_dec_prep: X_l (see the header).  One CTA per 32 x 16 output block: the block's source
// region of y_{l+1} (at most 18 x 10 pixels x 32 channels) is staged in shared memory with
// coalesced 16-byte loads, so every source value leaves L2 once instead of once per output pixel
// that interpolates it; then one thread per (pixel, 8-channel group) writes 16 bytes of X_l.
constexpr int kPrepW = 32, kPrepH = 16;
constexpr int kPrepSW = kPrepW / 2 + 2, kPrepSH = kPrepH / 2 + 2;
#ifndef TRIPS_PREP_UNIFORM
#define TRIPS_PREP_UNIFORM 1
#endif
// UNIFORM: items ordered group-major (a warp's 32 items share the channel group: no divergence
// between the interpolated and the pyramid groups); source pixels padded to 36 floats in shared
// memory so that the 16 distinct source pixels of a warp's float4 reads spread over the banks
constexpr int kPrepSP = TRIPS_PREP_UNIFORM ? kDecHidden + 4 : kDecHidden;   // floats per staged pixel
template <int NG>   // 16-byte channel groups per pixel: D.xc / 8
__global__ void __launch_bounds__(256) k_dec_prep(DecParams D, int l)
{
    __shared__ __align__(16) float s_y[kPrepSH * kPrepSW * kPrepSP];
    __shared__ int4 s_src[kPrepW * kPrepH];          // per output pixel: its 4 source offsets in s_y
    __shared__ float2 s_lw[kPrepW * kPrepH];         // and its bilinear weights (lx, ly)
    const DecLayer& L = D.L[l];
    const int npx = L.H * L.W;                       // < 2^31 / 8 (checked on the host)
    const int x0 = blockIdx.x * kPrepW, y0 = blockIdx.y * kPrepH;
    // source window: rows sy0 .. sy0 + SH - 1 (clamped into the layer), same for columns
    const int sx0 = max(0, x0 / 2 - 1), sy0 = max(0, y0 / 2 - 1);
    if (!L.coarsest) {
        const float* Yc = D.Y[(l + 1) & 1];
        for (int e = threadIdx.x; e < kPrepSH * kPrepSW * (kDecHidden / 4); e += blockDim.x) {
            const int c4 = e & (kDecHidden / 4 - 1);
            const int px = e >> 3;
            const int ry = px / kPrepSW, rx = px - ry * kPrepSW;
            const int sy = min(sy0 + ry, L.Hc - 1), sx = min(sx0 + rx, L.Wc - 1);
            reinterpret_cast<float4*>(s_y + px * kPrepSP)[c4] =
                __ldg(reinterpret_cast<const float4*>(Yc + ((int64_t)sy * L.Wc + sx) * kDecHidden) + c4);
        }
        // the interpolation setup once per output pixel (bilinear 2x, half-pixel centres: output i
        // samples (i + 0.5) / 2 - 0.5 >= 0, clamped), shared by its 4 channel groups
        for (int q = threadIdx.x; q < kPrepW * kPrepH; q += blockDim.x) {
            const int y = y0 + q / kPrepW, x = x0 + (q & (kPrepW - 1));
            const float sy = fmaxf((y + 0.5f) * 0.5f - 0.5f, 0.f), sx = fmaxf((x + 0.5f) * 0.5f - 0.5f, 0.f);
            const int iy0 = min((int)sy, L.Hc - 1), ix0 = min((int)sx, L.Wc - 1);
            const int iy1 = min(iy0 + 1, L.Hc - 1), ix1 = min(ix0 + 1, L.Wc - 1);
            s_src[q] = make_int4(((iy0 - sy0) * kPrepSW + (ix0 - sx0)) * kPrepSP, ((iy0 - sy0) * kPrepSW + (ix1 - sx0)) * kPrepSP,
                                 ((iy1 - sy0) * kPrepSW + (ix0 - sx0)) * kPrepSP, ((iy1 - sy0) * kPrepSW + (ix1 - sx0)) * kPrepSP);
            s_lw[q] = make_float2(sx - (float)ix0, sy - (float)iy0);
        }
        __syncthreads();
    }
    for (int it = threadIdx.x; it < kPrepW * kPrepH * NG; it += blockDim.x) {
#if TRIPS_PREP_UNIFORM
        const int grp = it / (kPrepW * kPrepH);      // warp-uniform
        const int q = it - grp * (kPrepW * kPrepH);
#else
        const int q = it / NG;                       // compile-time divisor
        const int grp = it - q * NG;
#endif
        const int y = y0 + q / kPrepW, x = x0 + (q & (kPrepW - 1));
        if (y >= L.H || x >= L.W) continue;
        const int p = y * L.W + x;
        float v[8];
        if (grp < kDecHidden / 8) {
            if (L.coarsest) {
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = 0.f;
            } else {
                const int4 so = s_src[q];
                const float2 w = s_lw[q];
                const float4* a = reinterpret_cast<const float4*>(s_y + so.x + grp * 8);
                const float4* b = reinterpret_cast<const float4*>(s_y + so.y + grp * 8);
                const float4* c = reinterpret_cast<const float4*>(s_y + so.z + grp * 8);
                const float4* d = reinterpret_cast<const float4*>(s_y + so.w + grp * 8);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float4 A = a[h], B = b[h], C = c[h], Dd = d[h];
                    const float r0[4] = {A.x, A.y, A.z, A.w}, r1[4] = {B.x, B.y, B.z, B.w};
                    const float r2[4] = {C.x, C.y, C.z, C.w}, r3[4] = {Dd.x, Dd.y, Dd.z, Dd.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float top = r0[j] * (1.f - w.x) + r1[j] * w.x;
                        const float bot = r2[j] * (1.f - w.x) + r3[j] * w.x;
                        v[4 * h + j] = top * (1.f - w.y) + bot * w.y;
                    }
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int ch = (grp * 8 + j) - kDecHidden;
                v[j] = ch <= D.F ? __ldg(D.pyramid + L.pyr_off + (int64_t)ch * npx + p) : 0.f;
            }
        }
        __half2 h2[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) h2[j] = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
        *reinterpret_cast<uint4*>(D.X + (int64_t)p * (NG * 8) + grp * 8) = *reinterpret_cast<uint4*>(h2);
    }
}

// fast-math activations (ex2.approx based): |error| ~ 1e-7 absolute, far inside the fp16-operand
// tolerance of the decoder (D8)
__device__ __forceinline__ float dec_elu(float v) { return v > 0.f ? v : __expf(v) - 1.f; }
__device__ __forceinline__ float dec_sigmoid(float v) { return __fdividef(1.f, 1.f + __expf(-v)); }

// k_dec_conv: see the header.  tmX: 3-D map of X_l {64 ch, W, H}, box {64, 128, 1}, SWIZZLE_128B;
// tmB: 2-D map of the packed weights {64, n * 9 * 96}, box {64, 96}, SWIZZLE_128B.
__global__ void __launch_bounds__(kDecThreads, 1) k_dec_conv(const __grid_constant__ CUtensorMap tmX,
                                                            const __grid_constant__ CUtensorMap tmB, DecParams D, int l)
{
    extern __shared__ __align__(1024) uint8_t dec_smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dec_smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sB = smem;                                           // 9 x 12 KB
    uint8_t* sA = smem + kDecTaps * kDecBBytes;                   // tap stages x 16 KB | row slots x 17 KB
    uint64_t* bars = reinterpret_cast<uint64_t*>(sA + (TRIPS_DEC_ROWS ? kDecRowSlots * kDecRowSlot : kDecStages * kDecABytes));
    uint64_t* full = bars;                                        // [stages]
    uint64_t* empty = bars + kDecStages;                          // [stages]
    uint64_t* tfull = bars + 2 * kDecStages;                      // [kDecAcc]
    uint64_t* tempty = tfull + kDecAcc;                           // [kDecAcc]
    uint64_t* bbar = tempty + kDecAcc;                            // weights loaded
    uint64_t* mdone = bbar + 1;                                   // [4] MMAs of tile it (mod 4) finished
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mdone + kDecMdone);

    const DecLayer& L = D.L[l];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int xt = (L.W + kDecM - 1) / kDecM;
    const int ntiles = L.H * xt;
#if TRIPS_DEC_ROWS
    // each CTA takes a contiguous run of the column-segment-major tile order: consecutive rows of
    // one 128-pixel column, so the row boxes y, y + 1 of a tile are rows of the next one too
    const int per = (ntiles + gridDim.x - 1) / gridDim.x;
    const int tile0 = blockIdx.x * per, tile1 = min(ntiles, tile0 + per), tstep = 1;
    auto tile_y = [&](int tile) { return tile % L.H; };
    auto tile_x0 = [&](int tile) { return (tile / L.H) * kDecM; };
#else
    const int tile0 = blockIdx.x, tile1 = ntiles, tstep = gridDim.x;
    auto tile_y = [&](int tile) { return tile / xt; };
    auto tile_x0 = [&](int tile) { return (tile % xt) * kDecM; };
#endif

    // epilogue constants in shared memory (broadcast reads instead of per-element L1 loads):
    // bf [32], bg [32], then at the finest layer Wo [out_ch][32], bo [out_ch]
    __shared__ __align__(16) float s_epi[2 * kDecHidden + kDecMaxOut * kDecHidden + kDecMaxOut];
    {
        const float* Pl = D.prm + L.prm_off;
        const int64_t wsz = (int64_t)kDecHidden * L.C * 9;
        for (int e = threadIdx.x; e < 2 * kDecHidden; e += kDecThreads)
            s_epi[e] = e < kDecHidden ? Pl[wsz + e] : Pl[2 * wsz + kDecHidden + (e - kDecHidden)];
        if (l == 0)
            for (int e = threadIdx.x; e < D.out_ch * (kDecHidden + 1); e += kDecThreads)
                s_epi[2 * kDecHidden + e] = D.prm[D.prm_out + e];       // Wo rows then bo, as stored
    }
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kDecStages; ++s) { dec_mbar_init(full + s, 1); dec_mbar_init(empty + s, 1); }
        for (int a = 0; a < kDecAcc; ++a) {
            dec_mbar_init(tfull + a, 1);
            dec_mbar_init(tempty + a, kDecEpiPerTile);
        }
        for (int a = 0; a < kDecMdone; ++a) dec_mbar_init(mdone + a, 1);
        dec_mbar_init(bbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {      // TMEM: kDecAcc accumulators x 96 columns (256 or 512 allocated)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(dec_smem_u32(tmem_slot)), "n"(kDecTmemCols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    dec_tc_fence_before();
    __syncthreads();
    dec_tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---- TMA producer: the weights once, then the 9 shifted A boxes of every tile
            dec_mbar_expect_tx(bbar, kDecTaps * kDecBBytes);
            for (int t = 0; t < kDecTaps; ++t) dec_tma_2d(sB + t * kDecBBytes, &tmB, bbar, 0, (l * kDecTaps + t) * kDecN);
#if TRIPS_DEC_ROWS
            // row boxes {64 ch, 130 px, 1 row} at (x0 - 1, r) in slot (r + 1) mod kDecRowSlots; a slot is reloaded once
            // the MMAs of the last tile that read it have finished
            int skey[kDecRowSlots], slast[kDecRowSlots];
#pragma unroll
            for (int q = 0; q < kDecRowSlots; ++q) { skey[q] = -1; slast[q] = -1; }
            int it = 0;
            for (int tile = tile0; tile < tile1; tile += tstep, ++it) {
                const int y = tile_y(tile), x0 = tile_x0(tile);
#pragma unroll
                for (int dy = -1; dy <= 1; ++dy) {
                    const int r = y + dy, sl = (r + 1) % kDecRowSlots;
                    const int key = (x0 / kDecM) * (L.H + 2) + (r + 1);
                    if (skey[sl] != key) {
                        if (slast[sl] >= 0) {
                            // MMAs complete in issue order; a barrier of tile it - 4 or later has
                            // not wrapped (its next phase is a tile not loaded yet)
                            const int w = max(slast[sl], it - kDecMdone);
                            dec_mbar_wait(mdone + (w & (kDecMdone - 1)), (uint32_t)(w / kDecMdone) & 1u);
                        }
                        dec_mbar_expect_tx(full + sl, kDecRowBytes);
                        dec_tma_3d(sA + sl * kDecRowSlot, &tmX, full + sl, 0, x0 - 1, r);
                        skey[sl] = key;
                    }
                    slast[sl] = it;
                }
            }
#else
            int s = 0;
            uint32_t ph = 0;
            for (int tile = tile0; tile < tile1; tile += tstep) {
                const int y = tile_y(tile), x0 = tile_x0(tile);
                for (int t = 0; t < kDecTaps; ++t) {
                    dec_mbar_wait(empty + s, ph ^ 1);
                    dec_mbar_expect_tx(full + s, kDecABytes);
                    dec_tma_3d(sA + s * kDecABytes, &tmX, full + s, 0, x0 + (t % 3) - 1, y + (t / 3) - 1);
                    if (++s == kDecStages) { s = 0; ph ^= 1; }
                }
            }
#endif
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---- MMA issuer
            dec_mbar_wait(bbar, 0);
#if TRIPS_DEC_ROWS
            int skey[kDecRowSlots];
            uint32_t snl[kDecRowSlots];
#pragma unroll
            for (int q = 0; q < kDecRowSlots; ++q) { skey[q] = -1; snl[q] = 0; }
            int it = 0;
            for (int tile = tile0; tile < tile1; tile += tstep, ++it) {
                const int acc = it % kDecAcc;
                const uint32_t aph = (uint32_t)(it / kDecAcc) & 1u;
                const int y = tile_y(tile), x0 = tile_x0(tile);
                dec_mbar_wait(tempty + acc, aph ^ 1);
                uint32_t rowa[3];
#pragma unroll
                for (int dy = -1; dy <= 1; ++dy) {            // the producer's slot bookkeeping, replayed
                    const int r = y + dy, sl = (r + 1) % kDecRowSlots;
                    const int key = (x0 / kDecM) * (L.H + 2) + (r + 1);
                    if (skey[sl] != key) {
                        skey[sl] = key;
                        dec_mbar_wait(full + sl, snl[sl] & 1u);
                        ++snl[sl];
                    }
                    rowa[dy + 1] = dec_smem_u32(sA + sl * kDecRowSlot);
                }
                dec_tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * kDecN);
#pragma unroll
                for (int tt = 0; tt < kDecTaps; ++tt) {
                    // tap (dy, dx): the row box of y + dy from pixel dx + 1 on (one 128-B row per pixel).
                    // N64: the centre tap first, over all 96 columns (it initialises the bypass block),
                    // then the other taps over the 64 gate/feature columns only
                    const int t = TRIPS_DEC_N64 ? (tt == 0 ? 4 : (tt <= 4 ? tt - 1 : tt)) : tt;
                    const uint32_t idesc = (TRIPS_DEC_N64 && tt > 0) ? kDecIdesc64 : kDecIdesc;
                    const uint32_t a0 = rowa[t / 3] + 128u * (uint32_t)(t % 3), b0 = dec_smem_u32(sB + t * kDecBBytes);
#pragma unroll
                    for (int k = 0; k < kDecXC / 16; ++k)
                        if (16 * k < D.xc) dec_umma(d, dec_desc(a0 + 32 * k), dec_desc(b0 + 32 * k), (tt | k) ? 1u : 0u, idesc);
                }
                dec_umma_commit(mdone + (it & (kDecMdone - 1)));   // row slots read by this tile may be reused
                dec_umma_commit(tfull + acc);                 // accumulator ready for the epilogue
            }
#else
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (int tile = tile0; tile < tile1; tile += tstep, ++it) {
                const int acc = it % kDecAcc;
                const uint32_t aph = (uint32_t)(it / kDecAcc) & 1u;
                dec_mbar_wait(tempty + acc, aph ^ 1);
                dec_tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * kDecN);
                for (int t = 0; t < kDecTaps; ++t) {
                    dec_mbar_wait(full + s, ph);
                    dec_tc_fence_after();
                    const uint32_t a0 = dec_smem_u32(sA + s * kDecABytes), b0 = dec_smem_u32(sB + t * kDecBBytes);
#pragma unroll
                    for (int k = 0; k < kDecXC / 16; ++k)    // K16 steps: +32 B inside the swizzle atom
                        if (16 * k < D.xc) dec_umma(d, dec_desc(a0 + 32 * k), dec_desc(b0 + 32 * k), (t | k) ? 1u : 0u);
                    dec_umma_commit(empty + s);               // smem slot free once these MMAs finish
                    if (++s == kDecStages) { s = 0; ph ^= 1; }
                }
                dec_umma_commit(tfull + acc);                 // accumulator ready for the epilogue
            }
#endif
        }
#if TRIPS_DEC_EPI16
    } else {
        // ---- epilogue warps 2-17: TMEM lane quarter q = warp % 4 (tile rows 32 q ..); warp slot
        // h = (warp - 2) / 4 takes tiles it = h (mod 4) whole, so four tiles drain concurrently
        static_assert(kDecAcc % 4 == 0, "EPI16 assigns accumulator it % 4 to warp slot it % 4");
        const int q = warp & 3, h = (warp - 2) >> 2;
        const bool last = l == 0;
        float* Yo = D.Y[l & 1];
        int it = 0;
        for (int tile = tile0; tile < tile1; tile += tstep, ++it) {
            if ((it & 3) != h) continue;
            const int acc = it % kDecAcc;
            const uint32_t aph = (uint32_t)(it / kDecAcc) & 1u;
            dec_mbar_wait(tfull + acc, aph);
            dec_tc_fence_after();
            const int y = tile_y(tile), x = tile_x0(tile) + 32 * q + lane;
            const int64_t p = (int64_t)y * L.W + x;
            const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * kDecN);
            float o[32];
#pragma unroll
            for (int hc = 0; hc < 2; ++hc) {
                uint32_t f[16], g[16], b[16];
                dec_tmem_ld16(ta + 16 * hc, f);
                dec_tmem_ld16(ta + 32 + 16 * hc, g);
                dec_tmem_ld16(ta + 64 + 16 * hc, b);
                dec_tmem_wait();
                if (hc == 1) {
                    dec_tc_fence_before();
                    __syncwarp();
                    if (lane == 0) dec_mbar_arrive(tempty + acc);    // TMEM buffer may be refilled
                }
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    o[16 * hc + c] = dec_elu(__uint_as_float(f[c]) + s_epi[16 * hc + c]) *
                                         dec_sigmoid(__uint_as_float(g[c]) + s_epi[kDecHidden + 16 * hc + c]) +
                                     __uint_as_float(b[c]);
                if (!last && x < L.W) {
                    float4* dst = reinterpret_cast<float4*>(Yo + p * kDecHidden + 16 * hc);
#pragma unroll
                    for (int c4 = 0; c4 < 4; ++c4)
                        dst[c4] = make_float4(o[16 * hc + 4 * c4], o[16 * hc + 4 * c4 + 1], o[16 * hc + 4 * c4 + 2],
                                              o[16 * hc + 4 * c4 + 3]);
                }
            }
            if (last && x < L.W) {
                const float* Wo = s_epi + 2 * kDecHidden;                 // [out_ch][32] then bo
                const float* bo = Wo + D.out_ch * kDecHidden;
                const int64_t plane = (int64_t)L.H * L.W;
                for (int oc = 0; oc < D.out_ch; ++oc) {
                    float sacc = bo[oc];
                    const float4* w = reinterpret_cast<const float4*>(Wo + oc * kDecHidden);
#pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) {
                        const float4 wv = w[c4];
                        sacc = fmaf(wv.x, o[4 * c4], sacc);
                        sacc = fmaf(wv.y, o[4 * c4 + 1], sacc);
                        sacc = fmaf(wv.z, o[4 * c4 + 2], sacc);
                        sacc = fmaf(wv.w, o[4 * c4 + 3], sacc);
                    }
                    D.out[oc * plane + p] = sacc;
                }
            }
        }
    }
#else
    } else {
        // ---- epilogue warps 2-9: TMEM lane quarter q = warp % 4 (tile rows 32 q ..), channel half
        // h (16 of the 32 hidden channels: f, g and bypass columns 16 h ..)
        const int q = warp & 3, h = (warp - 2) >> 2;
        const float* bf = s_epi + 16 * h;
        const float* bg = s_epi + kDecHidden + 16 * h;
        const bool last = l == 0;
        float* Yo = D.Y[l & 1];
        int it = 0;
        for (int tile = tile0; tile < tile1; tile += tstep, ++it) {
            const int acc = it % kDecAcc;
            const uint32_t aph = (uint32_t)(it / kDecAcc) & 1u;
            dec_mbar_wait(tfull + acc, aph);
            dec_tc_fence_after();
            const int y = tile_y(tile), x = tile_x0(tile) + 32 * q + lane;
            const int64_t p = (int64_t)y * L.W + x;
            const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * kDecN);
            if (!last) {
                // hidden layer: this warp's 16 channels of y_l
                uint32_t f[16], g[16], b[16];
                dec_tmem_ld16(ta + 16 * h, f);
                dec_tmem_ld16(ta + 32 + 16 * h, g);
                dec_tmem_ld16(ta + 64 + 16 * h, b);
                dec_tmem_wait();
                dec_tc_fence_before();
                __syncwarp();
                if (lane == 0) dec_mbar_arrive(tempty + acc);    // TMEM buffer may be refilled
                float o[16];
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    o[c] = dec_elu(__uint_as_float(f[c]) + bf[c]) * dec_sigmoid(__uint_as_float(g[c]) + bg[c]) +
                           __uint_as_float(b[c]);
                if (x < L.W) {
                    float4* dst = reinterpret_cast<float4*>(Yo + p * kDecHidden + 16 * h);
#pragma unroll
                    for (int c4 = 0; c4 < 4; ++c4) dst[c4] = make_float4(o[4 * c4], o[4 * c4 + 1], o[4 * c4 + 2], o[4 * c4 + 3]);
                }
            } else {
                // finest layer: the two warps of a lane quarter take alternate tiles whole (all 32
                // channels), so the output projection Wo y + bo needs no exchange between them
                const bool mine = (it & 1) == h;
                uint32_t f0[16], f1[16], g0[16], g1[16], b0[16], b1[16];
                if (mine) {
                    dec_tmem_ld16(ta, f0);
                    dec_tmem_ld16(ta + 16, f1);
                    dec_tmem_ld16(ta + 32, g0);
                    dec_tmem_ld16(ta + 48, g1);
                    dec_tmem_ld16(ta + 64, b0);
                    dec_tmem_ld16(ta + 80, b1);
                    dec_tmem_wait();
                }
                dec_tc_fence_before();
                __syncwarp();
                if (lane == 0) dec_mbar_arrive(tempty + acc);
                if (mine) {
                    const float* bf0 = bf - 16 * h;
                    const float* bg0 = bg - 16 * h;
                    float o[32];
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        o[c] = dec_elu(__uint_as_float(f0[c]) + bf0[c]) * dec_sigmoid(__uint_as_float(g0[c]) + bg0[c]) +
                               __uint_as_float(b0[c]);
                        o[16 + c] = dec_elu(__uint_as_float(f1[c]) + bf0[16 + c]) *
                                        dec_sigmoid(__uint_as_float(g1[c]) + bg0[16 + c]) + __uint_as_float(b1[c]);
                    }
                    const float* Wo = s_epi + 2 * kDecHidden;                 // [out_ch][32] then bo
                    const float* bo = Wo + D.out_ch * kDecHidden;
                    const int64_t plane = (int64_t)L.H * L.W;
                    if (x < L.W)
                        for (int oc = 0; oc < D.out_ch; ++oc) {
                            float sacc = bo[oc];
                            const float4* w = reinterpret_cast<const float4*>(Wo + oc * kDecHidden);
#pragma unroll
                            for (int c4 = 0; c4 < 8; ++c4) {
                                const float4 wv = w[c4];
                                sacc = fmaf(wv.x, o[4 * c4], sacc);
                                sacc = fmaf(wv.y, o[4 * c4 + 1], sacc);
                                sacc = fmaf(wv.z, o[4 * c4 + 2], sacc);
                                sacc = fmaf(wv.w, o[4 * c4 + 3], sacc);
                            }
                            D.out[oc * plane + p] = sacc;
                        }
                }
            }
        }
    }
#endif
    __syncthreads();
    if (warp == 1) {
        dec_tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(kDecTmemCols) : "memory");
    }
}

}  // namespace trips
