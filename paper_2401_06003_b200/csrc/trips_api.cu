// trips_api.cu -- host side of the C ABI declared in include/trips.h.
//
// Validation, plan/workspace layout, launch sequencing and optional per-stage CUDA-event
// timing.  No device allocation, no host synchronisation on the hot path.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/trips.h"
#include "kernels.cuh"
#include "knn.cuh"
#include "morton.cuh"
#include "microbench.cuh"
#include "decoder.cuh"
#ifndef TRIPS_TILE_PERM
#define TRIPS_TILE_PERM 0        // heaviest-first tile order: raster alone -15 us per view, but the two-stream
#endif                           // step measured slower (1432 vs 1445 frames/s, e2e 1367 vs 1387): off
#include <cudaTypedefs.h>

using namespace trips;

namespace {

std::atomic<long long> g_launches{0};
thread_local char g_msg[256];

constexpr int kStages = 5;   // 0 count (k_count), 1 emit (k_emit), 2 tscan (k_tscan), 3 raster (k_raster
                             // [+ k_coarse_blend]), 4 backward (k_backward_pairs | k_backward_coarse)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct EventPair {
    cudaEvent_t a, b;
};

}  // namespace

struct trips_plan {
    int32_t n_layers, F, FC, G, W, H, T;
    float t_min;
    int32_t coarse;         // coarse-layer inclusion depth, clamped to n_layers - 1
    int64_t max_points, P, pyr_floats;
    LayerGeom L[kMaxLayers];
    uint64_t kcap;
    // workspace layout (byte offsets)
    int32_t ctas;           // binning CTAs (persistent grid)
    bool gbin = false;      // global-counter binning (T > kMaxTilesSmem, or TRIPS_FORCE_GLOBAL_BINNING)
    size_t off_tperm = 0;   // [T] heaviest-first tile order (smem binning only)
    size_t off_gbsum = 0;   // [ceil(T / 1024)] segment totals of the global tile scan
    size_t off_geo, off_tau, off_z, off_hist, off_cvis, off_toff, off_tcnt, off_bkey, off_borig, off_pcnt, off_pmeta, off_kept, off_kgam,
        off_own, off_kpkey, off_kpinfo, off_kpcnt, off_stats, ws_bytes;
    // state
    const void* ws_bound = nullptr;
    int stage = 0;          // 0 none, 1 projected, 2 forward (saved), 3 forward (not saved)
    int64_t n = 0;
    Cam cam;
    const float* desc = nullptr;   // caller's descriptors of the last trips_project
    const float* last_gpyr = nullptr;  // grad_pyramid of the last backward (SCREEN_GRADS export)
    bool tau_direct = false;       // gathered in place (F % 4 == 0, 16-B aligned)
    // profiling
    bool prof = false;
    std::vector<EventPair> pending[kStages];
    std::vector<cudaEvent_t> pool;
    double ms[kStages] = {0, 0, 0, 0, 0};
    long long launches[kStages] = {0, 0, 0, 0, 0};
};

namespace {

cudaEvent_t get_event(trips_plan* p)
{
    if (!p->pool.empty()) {
        cudaEvent_t e = p->pool.back();
        p->pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct StageScope {
    trips_plan* p;
    int s;
    cudaStream_t st;
    EventPair ev{};
    StageScope(trips_plan* p_, int s_, cudaStream_t st_) : p(p_), s(s_), st(st_)
    {
        if (p->prof) {
            ev.a = get_event(p);
            ev.b = get_event(p);
            cudaEventRecord(ev.a, st);
        }
        p->launches[s]++;
    }
    ~StageScope()
    {
        if (p->prof) {
            cudaEventRecord(ev.b, st);
            p->pending[s].push_back(ev);
        }
    }
};

int cuda_status(cudaError_t e)
{
    if (e == cudaSuccess) return TRIPS_OK;
    snprintf(g_msg, sizeof(g_msg), "TRIPS_ERR_CUDA: %s", cudaGetErrorString(e));
    return TRIPS_ERR_CUDA;
}

// Per-device host caches (SM count, shared-memory opt-ins), guarded by one mutex: a process may
// drive several GPUs, and cudaFuncSetAttribute applies to the current device only.
constexpr int kMaxDevices = 64;
std::mutex g_dev_mu;

int current_device()
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
        cudaGetLastError();
        dev = 0;
    }
    return dev;
}

int num_sms()
{
    static int sms[kMaxDevices] = {};
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (!sms[dev]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = 148;                          // B200; plan creation must work without a GPU
        cudaGetLastError();
        sms[dev] = v;
    }
    return sms[dev];
}

template <int FC>
int set_emit_attr(size_t bytes)
{
    return (int)cudaFuncSetAttribute(k_count<FC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Opt the binning kernels into > 48 KB of dynamic shared memory (one counter per tile).
int set_smem_attrs(size_t bytes)
{
    static size_t done_dev[kMaxDevices] = {};
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_dev_mu);
    size_t& done = done_dev[dev];
    if (bytes <= done) return TRIPS_OK;
    cudaError_t e = cudaFuncSetAttribute(k_emit<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    int bad = (int)e;
    bad |= (int)cudaFuncSetAttribute(k_tscan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    bad |= set_emit_attr<4>(bytes) | set_emit_attr<8>(bytes) | set_emit_attr<12>(bytes) | set_emit_attr<16>(bytes) |
           set_emit_attr<20>(bytes) | set_emit_attr<24>(bytes) | set_emit_attr<28>(bytes) | set_emit_attr<32>(bytes);
    if (bad) return cuda_status(cudaGetLastError());
    done = bytes;
    return TRIPS_OK;
}

int check_launch()
{
    g_launches++;
    return cuda_status(cudaGetLastError());
}

Params make_params(const trips_plan* p, void* ws)
{
    Params P;
    memset(&P, 0, sizeof(P));
    P.n = (int32_t)p->n;
    P.F = p->F; P.FC = p->FC; P.G = 0;
    P.n_layers = p->n_layers; P.T = p->T;
    P.t_min = p->t_min;
    P.coarse = p->coarse;
    for (int l = 0; l < kMaxLayers; ++l) P.L[l] = p->L[l];
    P.cam = p->cam;
    char* b = static_cast<char*>(ws);
    P.geo = reinterpret_cast<float4*>(b + p->off_geo);
    P.tau_copy = reinterpret_cast<float*>(b + p->off_tau);
    P.tau_direct = p->tau_direct ? 1 : 0;
    P.tau = p->tau_direct ? p->desc : P.tau_copy;
    P.zbuf = reinterpret_cast<float*>(b + p->off_z);
    P.hist = reinterpret_cast<uint32_t*>(b + p->off_hist);
    P.cta_vis = reinterpret_cast<uint32_t*>(b + p->off_cvis);
    P.tile_off = reinterpret_cast<uint32_t*>(b + p->off_toff);
    P.tile_cnt = reinterpret_cast<uint32_t*>(b + p->off_tcnt);
    P.tile_perm = (TRIPS_TILE_PERM && !p->gbin && TRIPS_TILE_SCAN == 2) ? reinterpret_cast<uint32_t*>(b + p->off_tperm) : nullptr;
    P.bin_key = reinterpret_cast<uint64_t*>(b + p->off_bkey);
    P.bin_orig = reinterpret_cast<uint16_t*>(b + p->off_borig);
    P.pix_cnt = reinterpret_cast<uint32_t*>(b + p->off_pcnt);
    P.pix_meta = reinterpret_cast<uint32_t*>(b + p->off_pmeta);
    P.kept = p->coarse ? reinterpret_cast<uint64_t*>(b + p->off_kept) : nullptr;
    P.kp_key = p->coarse ? nullptr : reinterpret_cast<uint64_t*>(b + p->off_kpkey);
    P.kp_info = p->coarse ? nullptr : reinterpret_cast<uint32_t*>(b + p->off_kpinfo);
    P.kp_cnt = p->coarse ? nullptr : reinterpret_cast<uint32_t*>(b + p->off_kpcnt);
    P.kept_gamma = reinterpret_cast<float*>(b + p->off_kgam);
    P.own = p->coarse ? reinterpret_cast<uint64_t*>(b + p->off_own) : nullptr;
    P.stats = reinterpret_cast<unsigned long long*>(b + p->off_stats);
    return P;
}

bool aligned(const void* ptr, size_t a) { return (reinterpret_cast<uintptr_t>(ptr) & (a - 1)) == 0; }

template <typename WS>
int sort_scan(const WS& W, cudaStream_t st)
{
    const int nseg = (256 * W.nblk + 1023) / 1024;
    int rc;
    k_sort_scan_blocks<<<nseg, 1024, 0, st>>>(W);
    if ((rc = check_launch())) return rc;
    k_sort_scan_top<<<1, 1024, 0, st>>>(W);
    if ((rc = check_launch())) return rc;
    k_sort_scan_add<<<nseg, 1024, 0, st>>>(W);
    return check_launch();
}

#ifdef TRIPS_FC4_ONLY   // experiment builds (tools/ variants): F <= 4 only, ~6x faster to compile
#define TRIPS_FC_SWITCH(FC, CALL)                \
    switch (FC) {                                \
    case 4: { constexpr int kFC = 4; CALL; } break;   \
    default: return TRIPS_ERR_ARG;               \
    }
#else
#define TRIPS_FC_SWITCH(FC, CALL)                \
    switch (FC) {                                \
    case 4: { constexpr int kFC = 4; CALL; } break;   \
    case 8: { constexpr int kFC = 8; CALL; } break;   \
    case 12: { constexpr int kFC = 12; CALL; } break; \
    case 16: { constexpr int kFC = 16; CALL; } break; \
    case 20: { constexpr int kFC = 20; CALL; } break; \
    case 24: { constexpr int kFC = 24; CALL; } break; \
    case 28: { constexpr int kFC = 28; CALL; } break; \
    case 32: { constexpr int kFC = 32; CALL; } break; \
    default: return TRIPS_ERR_ARG;               \
    }
#endif

}  // namespace

extern "C" {

int trips_plan_create(const trips_config* cfg, int32_t width, int32_t height, int64_t max_points,
                      trips_plan** out)
{
    if (!cfg || !out) return TRIPS_ERR_ARG;
    *out = nullptr;
    const int n = cfg->num_layers, F = cfg->num_features;
    if (n < 1 || n > kMaxLayers || F < 1 || F > 32) return TRIPS_ERR_ARG;
    if (!(cfg->t_min >= 0.0f && cfg->t_min < 1.0f)) return TRIPS_ERR_ARG;
    if (cfg->coarse_layers < 0) return TRIPS_ERR_ARG;
    if (width < 1 || height < 1 || width > 32768 || height > 32768) return TRIPS_ERR_ARG;
    if (max_points < 0 || max_points >= (int64_t(1) << 28)) return TRIPS_ERR_ARG;
    trips_plan* p = new trips_plan();
    p->n_layers = n; p->F = F; p->FC = (F + 3) & ~3; p->G = 0;
    p->t_min = cfg->t_min;
    p->coarse = std::min(cfg->coarse_layers, n - 1);
    p->W = width; p->H = height; p->max_points = max_points;
    memset(p->L, 0, sizeof(p->L));
    int64_t pix = 0;
    int32_t tiles = 0;
    for (int l = 0; l < n; ++l) {
        LayerGeom& g = p->L[l];
        g.W = (width + (1 << l) - 1) >> l;
        g.H = (height + (1 << l) - 1) >> l;
        g.tiles_x = (g.W + kTile - 1) / kTile;
        g.tiles_y = (g.H + kTile - 1) / kTile;
        g.tile_base = tiles;
        g.pix_off = pix;
        g.float_off = pix * (F + 1);
        pix += (int64_t)g.W * g.H;
        tiles += g.tiles_x * g.tiles_y;
    }
    p->P = pix;
    p->T = tiles;
    p->pyr_floats = pix * (F + 1);
    p->kcap = (uint64_t)tiles * kTilePix * kCap;       // kept lists: 16 slots per tile pixel
    if (p->kcap >= (uint64_t(1) << 32)) { delete p; return TRIPS_ERR_ARG; }
    // more tiles than the per-CTA shared-memory counters hold (e.g. 8K frames): global counters
    const char* force = getenv("TRIPS_FORCE_GLOBAL_BINNING");     // tests: exercise that path at small sizes
    p->gbin = tiles > kMaxTilesSmem || (force && force[0] == '1');
    const size_t N = (size_t)(max_points > 0 ? max_points : 1);
    size_t o = 0;
    p->ctas = num_sms() * kBinCtasPerSm;
    p->off_geo = o;    o = align256(o + N * 16);
    p->off_tau = o;    o = align256(o + N * p->FC * sizeof(float));   // used only when desc is not gatherable in place
    p->off_z = o;      o = align256(o + N * sizeof(float));
    p->off_hist = o;   o = align256(o + (p->gbin ? 0 : (size_t)p->ctas * tiles * 4));
    p->off_gbsum = o;  o = align256(o + (size_t)(tiles + 1023) / 1024 * 4);
    p->off_cvis = o;   o = align256(o + (size_t)p->ctas * 4);
    p->off_toff = o;   o = align256(o + ((size_t)tiles + 1) * 4);
    p->off_tcnt = o;   o = align256(o + (size_t)(tiles + 1) * 4);   // [T] = k_count completion ticket
    p->off_tperm = o;  o = align256(o + (size_t)tiles * 4);
    p->off_bkey = o;   o = align256(o + 8 * N * 8);
    p->off_borig = o;  o = align256(o + 8 * N * 2);
    p->off_pcnt = o;  o = align256(o + (size_t)tiles * kTilePix * 4);
    p->off_pmeta = o; o = align256(o + (size_t)tiles * kTilePix * 4);
    // kept lists: coarse inclusion keeps per-pixel key lists; otherwise the raster stores the
    // tile's kept (point, tile) pairs (<= 4096 per tile) for the pair-wise backward
    p->off_kept = o;  o = align256(o + (p->coarse ? p->kcap * 8 : 0));
    p->off_kpkey = o; o = align256(o + (p->coarse ? 0 : p->kcap * 8));
    p->off_kpinfo = o; o = align256(o + (p->coarse ? 0 : p->kcap * 4));
    p->off_kpcnt = o; o = align256(o + (p->coarse ? 0 : (size_t)tiles * 4));
    p->off_kgam = o;  o = align256(o + (p->kcap ? p->kcap : 1) * 4);
    p->off_own = o;   o = align256(o + (p->coarse ? (size_t)tiles * kTilePix * kCap * 8 : 0));
    p->off_stats = o; o = align256(o + S_COUNT * 8);
    p->ws_bytes = o;
    *out = p;
    return TRIPS_OK;
}

void trips_plan_destroy(trips_plan* p)
{
    if (!p) return;
    for (int s = 0; s < kStages; ++s)
        for (auto& e : p->pending[s]) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
    for (auto e : p->pool) cudaEventDestroy(e);
    delete p;
}

size_t trips_workspace_bytes(const trips_plan* p) { return p ? p->ws_bytes : 0; }
int64_t trips_num_pixels(const trips_plan* p) { return p ? p->P : -1; }
int64_t trips_pyramid_floats(const trips_plan* p) { return p ? p->pyr_floats : -1; }

int trips_layer_dims(const trips_plan* p, int32_t l, int32_t* h, int32_t* w, int64_t* off)
{
    if (!p || l < 0 || l >= p->n_layers) return TRIPS_ERR_ARG;
    if (h) *h = p->L[l].H;
    if (w) *w = p->L[l].W;
    if (off) *off = p->L[l].float_off;
    return TRIPS_OK;
}

int trips_project(trips_plan* p, void* ws, const trips_camera* c, int64_t n, const float* pos,
                  const float* world_size, const float* opacity, const float* desc, int8_t* level_out,
                  float* proj_out, void* stream)
{
    if (!p || !ws || !c) return TRIPS_ERR_ARG;
    if (n < 0) return TRIPS_ERR_ARG;
    if (n > p->max_points) return TRIPS_ERR_CAPACITY;
    if (n > 0 && (!pos || !world_size || !opacity || !desc)) return TRIPS_ERR_ARG;
    if (c->width != p->W || c->height != p->H) return TRIPS_ERR_ARG;
    if (!(c->fx > 0) || !(c->fy > 0) || !(c->f > 0) || !(c->near_plane > 0)) return TRIPS_ERR_ARG;
    if (!aligned(ws, 256)) return TRIPS_ERR_ALIGN;
    if (!aligned(pos, 4) || !aligned(desc, 4) || !aligned(world_size, 4) || !aligned(opacity, 4) ||
        !aligned(proj_out, 16))
        return TRIPS_ERR_ALIGN;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    p->ws_bound = ws;
    p->stage = 0;
    p->n = n;
    p->last_gpyr = nullptr;
    // descriptors are gathered straight from the caller's rows when they are whole float4s;
    // otherwise k_count writes a padded copy into the workspace
    p->desc = desc;
    p->tau_direct = (p->F & 3) == 0 && aligned(desc, 16);
    Cam& cam = p->cam;
    cam.fx = c->fx; cam.fy = c->fy; cam.cx = c->cx; cam.cy = c->cy; cam.f = c->f;
    memcpy(cam.R, c->R, sizeof(cam.R));
    memcpy(cam.t, c->t, sizeof(cam.t));
    cam.near_plane = c->near_plane;
    Params P = make_params(p, ws);
    P.pos = pos; P.sw = world_size; P.alpha = opacity; P.desc = desc;
    int rc = cuda_status(cudaMemsetAsync(P.stats, 0, S_COUNT * 8, st));
    if (rc) return rc;
    rc = cuda_status(cudaMemsetAsync(P.tile_cnt, 0, (size_t)(p->T + 1) * 4, st));
    if (rc) return rc;
    if (p->gbin) {
        uint32_t* bsum = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + p->off_gbsum);
        const int nseg = (p->T + 1023) / 1024;
        {
            StageScope sc(p, 0, st);
            TRIPS_FC_SWITCH(p->FC, (k_count<kFC, true><<<p->ctas, kBinThreads, 0, st>>>(P, level_out, proj_out)));
            if ((rc = check_launch())) return rc;
        }
        {
            StageScope sc(p, 2, st);
            k_gscan_seg<<<nseg, 1024, 0, st>>>(P, bsum);
            if ((rc = check_launch())) return rc;
            k_gscan_top<<<1, 1024, 0, st>>>(P, bsum);
            if ((rc = check_launch())) return rc;
            k_gscan_add<<<nseg, 1024, 0, st>>>(P, bsum);
            if ((rc = check_launch())) return rc;
            if ((rc = cuda_status(cudaMemsetAsync(P.tile_cnt, 0, (size_t)p->T * 4, st)))) return rc;   // -> cursors
        }
        {
            StageScope sc(p, 1, st);
            k_emit<true><<<p->ctas, kBinThreads, 0, st>>>(P);
            if ((rc = check_launch())) return rc;
        }
        p->stage = 1;
        return TRIPS_OK;
    }
    const size_t hsm = (size_t)p->T * 4;
    if ((rc = set_smem_attrs(hsm))) return rc;
    {
        StageScope sc(p, 0, st);
        TRIPS_FC_SWITCH(p->FC, (k_count<kFC, false><<<p->ctas, kBinThreads, hsm, st>>>(P, level_out, proj_out)));
        if ((rc = check_launch())) return rc;
    }
#if TRIPS_TILE_SCAN == 0
    {
        StageScope sc(p, 2, st);
        k_tscan<<<1, 1024, hsm, st>>>(P);
        if ((rc = check_launch())) return rc;
    }
#endif
    {
        StageScope sc(p, 1, st);
        k_emit<false><<<p->ctas, kBinThreads, hsm, st>>>(P);
        if ((rc = check_launch())) return rc;
    }
    p->stage = 1;
    return TRIPS_OK;
}

int trips_splat_forward(trips_plan* p, void* ws, float* pyramid, uint32_t flags, void* stream)
{
    if (!p || !ws || !pyramid) return TRIPS_ERR_ARG;
    if (p->stage != 1 || ws != p->ws_bound) return TRIPS_ERR_STATE;
    if (!aligned(pyramid, 16)) return TRIPS_ERR_ALIGN;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Params P = make_params(p, ws);
    int rc;
    {
        StageScope sc(p, 3, st);
        const int save = (flags & TRIPS_FWD_SAVE_FOR_BACKWARD) ? 1 : 0;
        static bool rattr_dev[kMaxDevices][3][9] = {};
        const int mode = p->coarse ? kRasterOwn : (p->t_min > 0.f ? kRasterTmin : kRasterPlain);
        const size_t rsm = (size_t)raster_dyn_smem();
        const int dev = current_device();
        std::lock_guard<std::mutex> lk(g_dev_mu);
        bool (&rattr)[3][9] = rattr_dev[dev];
        if (!rattr[mode][p->FC / 4]) {
            const int a = (int)cudaFuncAttributeMaxDynamicSharedMemorySize;
            if (mode == kRasterOwn) {
                TRIPS_FC_SWITCH(p->FC, (cudaFuncSetAttribute(k_raster<kFC, kRasterOwn>, (cudaFuncAttribute)a, raster_dyn_smem())));
            } else if (mode == kRasterTmin) {
                TRIPS_FC_SWITCH(p->FC, (cudaFuncSetAttribute(k_raster<kFC, kRasterTmin>, (cudaFuncAttribute)a, raster_dyn_smem())));
            } else {
                TRIPS_FC_SWITCH(p->FC, (cudaFuncSetAttribute(k_raster<kFC, kRasterPlain>, (cudaFuncAttribute)a, raster_dyn_smem())));
            }
            rattr[mode][p->FC / 4] = true;
        }
        if (mode == kRasterOwn) {
            TRIPS_FC_SWITCH(p->FC, (k_raster<kFC, kRasterOwn><<<p->T, kTilePix, rsm, st>>>(P, pyramid, save)));
            if ((rc = check_launch())) return rc;
            TRIPS_FC_SWITCH(p->FC, (k_coarse_blend<kFC><<<p->T, kTilePix, 0, st>>>(P, pyramid, save)));
        } else if (mode == kRasterTmin) {
            TRIPS_FC_SWITCH(p->FC, (k_raster<kFC, kRasterTmin><<<p->T, kTilePix, rsm, st>>>(P, pyramid, save)));
        } else {
            TRIPS_FC_SWITCH(p->FC, (k_raster<kFC, kRasterPlain><<<p->T, kTilePix, rsm, st>>>(P, pyramid, save)));
        }
        if ((rc = check_launch())) return rc;
    }
    p->stage = (flags & TRIPS_FWD_SAVE_FOR_BACKWARD) ? 2 : 3;
    return TRIPS_OK;
}

namespace {

// Launches the backward of the last saved forward into the caller's buffers (go), or the
// screen-space gradients into go.screen (SCREEN, debug export).
int launch_backward(const trips_plan* p, const Params& P, const float* gpyr, const GradOut& go, float* gcam, bool screen,
                    cudaStream_t st)
{
#define TRIPS_BWD(KERNEL, CAM, SCR) TRIPS_FC_SWITCH(p->FC, (KERNEL<kFC, CAM, SCR><<<p->T, kTilePix, 0, st>>>(P, gpyr, go, gcam)))
    if (p->coarse) {
        if (screen) { TRIPS_BWD(k_backward_coarse, false, true); }
        else if (gcam) { TRIPS_BWD(k_backward_coarse, true, false); }
        else { TRIPS_BWD(k_backward_coarse, false, false); }
    } else {
        if (screen) { TRIPS_BWD(k_backward_pairs, false, true); }
        else if (gcam) { TRIPS_BWD(k_backward_pairs, true, false); }
        else { TRIPS_BWD(k_backward_pairs, false, false); }
    }
#undef TRIPS_BWD
    return check_launch();
}

}  // namespace

int trips_splat_backward(trips_plan* p, void* ws, const float* grad_pyramid, float* grad_pos_size, float* grad_opacity,
                         float* grad_desc, float* grad_camera, void* stream)
{
    if (!p || !ws || !grad_pyramid) return TRIPS_ERR_ARG;
    if (p->n > 0 && (!grad_pos_size || !grad_opacity || !grad_desc)) return TRIPS_ERR_ARG;
    if (p->stage != 2 || ws != p->ws_bound) return TRIPS_ERR_STATE;
    if (!aligned(grad_pyramid, 16) || !aligned(grad_pos_size, 16) || !aligned(grad_opacity, 4) ||
        !aligned(grad_desc, 4) || !aligned(grad_camera, 4))
        return TRIPS_ERR_ALIGN;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Params P = make_params(p, ws);
    GradOut go;
    go.pos_size = grad_pos_size;
    go.opacity = grad_opacity;
    go.desc = grad_desc;
    go.screen = nullptr;
    go.desc_vec = (p->F % 4 == 0 && aligned(grad_desc, 16)) ? 4 : ((p->F % 2 == 0 && aligned(grad_desc, 8)) ? 2 : 1);
    p->last_gpyr = grad_pyramid;
    StageScope sc(p, 4, st);
    return launch_backward(p, P, grad_pyramid, go, grad_camera, false, st);
}

int trips_read_stats(const trips_plan* p, const void* ws, trips_stats* out, void* stream)
{
    if (!p || !ws || !out) return TRIPS_ERR_ARG;
    if (p->stage == 0 || ws != p->ws_bound) return TRIPS_ERR_STATE;
    unsigned long long h[S_COUNT];
    uint32_t npairs = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Params P = make_params(p, const_cast<void*>(ws));
    int rc = cuda_status(cudaMemsetAsync(P.stats, 0, S_COUNT * 8, st));
    if (rc) return rc;
    const int npix = p->stage >= 2 ? p->T * kTilePix : 0;
    k_stats<<<std::max(1, std::min(148 * 4, (npix + 255) / 256)), 256, 0, st>>>(P, p->ctas, npix,
                                                                              (p->stage == 2 && !p->coarse) ? p->T : 0);
    if ((rc = check_launch())) return rc;
    rc = cuda_status(cudaMemcpyAsync(h, P.stats, sizeof(h), cudaMemcpyDeviceToHost, st));
    if (rc) return rc;
    rc = cuda_status(cudaMemcpyAsync(&npairs, P.tile_off + p->T, 4, cudaMemcpyDeviceToHost, st));
    if (rc) return rc;
    if ((rc = cuda_status(cudaStreamSynchronize(st)))) return rc;
    out->n_visible = (int64_t)h[S_VISIBLE];
    out->n_culled = p->n - out->n_visible;
    out->n_pairs = (int64_t)npairs;
    out->n_frag = (int64_t)h[S_FRAG];
    out->n_kept = (int64_t)h[S_KEPT];
    out->n_kept_pairs = (int64_t)h[S_KPAIRS];
    out->n_trunc_pixels = (int64_t)h[S_TRUNC];
    out->max_list = (int64_t)h[S_MAXLIST];
    return TRIPS_OK;
}

int trips_debug_export(const trips_plan* p, const void* ws, int32_t what, void* dst, void* stream)
{
    if (!p || !ws || !dst) return TRIPS_ERR_ARG;
    if (what != TRIPS_EXPORT_COUNTS && what != TRIPS_EXPORT_KEPT && what != TRIPS_EXPORT_KEPT_LAYER &&
        what != TRIPS_EXPORT_SCREEN_GRADS)
        return TRIPS_ERR_ARG;
    if (ws != p->ws_bound || p->stage < 2) return TRIPS_ERR_STATE;
    if (what != TRIPS_EXPORT_COUNTS && p->stage != 2) return TRIPS_ERR_STATE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Params P = make_params(p, const_cast<void*>(ws));
    int rc;
    if (what == TRIPS_EXPORT_SCREEN_GRADS) {
        if (!p->last_gpyr) return TRIPS_ERR_STATE;
        if (!aligned(dst, 4)) return TRIPS_ERR_ALIGN;
        if ((rc = cuda_status(cudaMemsetAsync(dst, 0, (size_t)p->n * (4 + p->F) * sizeof(float), st)))) return rc;
        GradOut go;
        memset(&go, 0, sizeof(go));
        go.screen = static_cast<float*>(dst);
        if ((rc = launch_backward(p, P, p->last_gpyr, go, nullptr, true, st))) return rc;
    } else {
        k_export<<<p->T, kTilePix, 0, st>>>(P, what, dst);
        if ((rc = check_launch())) return rc;
    }
    return cuda_status(cudaStreamSynchronize(st));
}

int trips_set_profiling(trips_plan* p, int32_t enable)
{
    if (!p) return TRIPS_ERR_ARG;
    p->prof = enable != 0;
    return TRIPS_OK;
}

int trips_read_stage_ms(trips_plan* p, double* ms, int64_t* launches, int32_t max_stages, int32_t reset)
{
    if (!p) return TRIPS_ERR_ARG;
    for (int s = 0; s < kStages; ++s) {
        for (auto& e : p->pending[s]) {
            float t = 0.f;
            if (cudaEventSynchronize(e.b) == cudaSuccess && cudaEventElapsedTime(&t, e.a, e.b) == cudaSuccess)
                p->ms[s] += t;
            p->pool.push_back(e.a);
            p->pool.push_back(e.b);
        }
        p->pending[s].clear();
    }
    const int m = max_stages < kStages ? max_stages : kStages;
    for (int s = 0; s < m; ++s) {
        if (ms) ms[s] = p->ms[s];
        if (launches) launches[s] = p->launches[s];
    }
    if (reset)
        for (int s = 0; s < kStages; ++s) { p->ms[s] = 0; p->launches[s] = 0; }
    return m;
}

int64_t trips_launch_count(void) { return (int64_t)g_launches.load(); }

size_t trips_knn_workspace_bytes(int64_t n)
{
    if (n < 0) return 0;
    const size_t N = (size_t)(n > 0 ? n : 1);
    const size_t nblk = (N + kSortBlock - 1) / kSortBlock;
    return 2 * align256(N * 8) + 2 * align256(N * 4) + align256(256 * nblk * 4) + align256((256 * nblk + 1023) / 1024 * 4) +
           align256(6 * 4) + align256(4) + align256(N * 16);
}

int trips_knn_sizes(void* ws, int64_t n, const float* pos, float* size_out, int32_t* nbr_out, void* stream)
{
    if (!ws || n < 0 || (n > 0 && (!pos || !size_out))) return TRIPS_ERR_ARG;
    if (n >= (int64_t(1) << 30)) return TRIPS_ERR_CAPACITY;
    if (!aligned(ws, 256) || !aligned(pos, 4) || !aligned(size_out, 4) || !aligned(nbr_out, 4)) return TRIPS_ERR_ALIGN;
    if (n == 0) return TRIPS_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t N = (size_t)n;
    KnnWs W;
    W.n = (int)n;
    W.nblk = (int)((N + kSortBlock - 1) / kSortBlock);
    W.last_pass = kKnnPasses - 1;
    char* b = static_cast<char*>(ws);
    size_t o = 0;
    W.keys[0] = reinterpret_cast<uint64_t*>(b + o); o += align256(N * 8);
    W.keys[1] = reinterpret_cast<uint64_t*>(b + o); o += align256(N * 8);
    W.vals[0] = reinterpret_cast<uint32_t*>(b + o); o += align256(N * 4);
    W.vals[1] = reinterpret_cast<uint32_t*>(b + o); o += align256(N * 4);
    W.hist = reinterpret_cast<uint32_t*>(b + o);    o += align256(256 * (size_t)W.nblk * 4);
    W.bsum = reinterpret_cast<uint32_t*>(b + o);    o += align256((256 * (size_t)W.nblk + 1023) / 1024 * 4);
    W.bbox = reinterpret_cast<uint32_t*>(b + o);    o += align256(6 * 4);
    W.nfin = reinterpret_cast<uint32_t*>(b + o);    o += align256(4);
    W.pts = reinterpret_cast<float4*>(b + o);
    int rc = cuda_status(cudaMemsetAsync(W.bbox, 0xff, 3 * 4, st));
    if (rc) return rc;
    if ((rc = cuda_status(cudaMemsetAsync(W.bbox + 3, 0, 3 * 4, st)))) return rc;
    if ((rc = cuda_status(cudaMemsetAsync(W.nfin, 0, 4, st)))) return rc;
    const int pb = (W.n + 255) / 256;
    k_bbox<<<std::min(pb, 148 * 8), 256, 0, st>>>(W, pos);
    if ((rc = check_launch())) return rc;
    k_knn_codes<<<pb, 256, 0, st>>>(W, pos);
    if ((rc = check_launch())) return rc;
    for (int pass = 0; pass < kKnnPasses; ++pass) {       // even count: sorted codes/indices in [0]
        k_sort_hist<<<W.nblk, 256, 0, st>>>(W, pass);
        if ((rc = check_launch())) return rc;
        if ((rc = sort_scan(W, st))) return rc;
        k_sort_scatter<<<W.nblk, 256, 0, st>>>(W, pass, nullptr);
        if ((rc = check_launch())) return rc;
    }
    k_knn_gather<<<pb, 256, 0, st>>>(W, pos);
    if ((rc = check_launch())) return rc;
    k_knn_query<<<pb, 256, 0, st>>>(W, size_out, nbr_out);
    return check_launch();
}

// ----------------------------------------------------------------------------- decoder

namespace {

constexpr int kDecHiddenH = 32;

int64_t dec_layer_params(int C) { return 2 * ((int64_t)kDecHiddenH * C * 9 + kDecHiddenH) + (int64_t)kDecHiddenH * C; }
int dec_in_channels(const trips_plan* p, int l) { return l == p->n_layers - 1 ? p->F + 1 : kDecHiddenH + p->F + 1; }

struct DecWsLayout {
    size_t wpack, X, Y0, Y1, bytes;
};

DecWsLayout dec_ws_layout(const trips_plan* p)
{
    DecWsLayout o;
    size_t b = 0;
    o.wpack = b; b = align256(b + (size_t)p->n_layers * kDecTaps * kDecN * kDecXC * 2);
    o.X = b;     b = align256(b + (size_t)p->L[0].H * p->L[0].W * kDecXC * 2);
    const size_t ysz = p->n_layers > 1 ? (size_t)p->L[1].H * p->L[1].W * kDecHidden * 4 : 256;
    o.Y0 = b;    b = align256(b + ysz);
    o.Y1 = b;    b = align256(b + ysz);
    o.bytes = b;
    return o;
}

PFN_cuTensorMapEncodeTiled_v12000 dec_encoder()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        cudaGetLastError();
    });
    return fn;
}

}  // namespace

int64_t trips_decoder_param_count(const trips_plan* p, int32_t out_channels)
{
    if (!p || out_channels < 1 || out_channels > kDecMaxOut) return -1;
    int64_t n = 0;
    for (int l = 0; l < p->n_layers; ++l) n += dec_layer_params(dec_in_channels(p, l));
    return n + (int64_t)out_channels * kDecHiddenH + out_channels;
}

size_t trips_decoder_workspace_bytes(const trips_plan* p)
{
    return p ? dec_ws_layout(p).bytes : 0;
}

int trips_decode(const trips_plan* p, void* dws, const float* params, int32_t out_channels, const float* pyramid,
                 float* out, void* stream)
{
    if (!p || !dws || !params || !pyramid || !out || out_channels < 1 || out_channels > kDecMaxOut) return TRIPS_ERR_ARG;
    if (p->F + 1 > kDecXC - kDecHidden) return TRIPS_ERR_ARG;            // pyramid channels must fit X
    if ((int64_t)p->L[0].H * p->L[0].W * (kDecXC / 8) >= (int64_t(1) << 31)) return TRIPS_ERR_ARG;
    if (!aligned(dws, 256) || !aligned(params, 4) || !aligned(pyramid, 4) || !aligned(out, 4)) return TRIPS_ERR_ALIGN;
    PFN_cuTensorMapEncodeTiled_v12000 encode = dec_encoder();
    if (!encode) {
        snprintf(g_msg, sizeof(g_msg), "TRIPS_ERR_CUDA: cuTensorMapEncodeTiled unavailable");
        return TRIPS_ERR_CUDA;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const DecWsLayout wl = dec_ws_layout(p);
    char* b = static_cast<char*>(dws);
    DecParams D;
    memset(&D, 0, sizeof(D));
    D.n_layers = p->n_layers;
    D.F = p->F;
    D.out_ch = out_channels;
    D.xc = (p->F + 1 <= 16) ? 48 : kDecXC;
    int64_t o = 0;
    for (int l = 0; l < p->n_layers; ++l) {
        DecLayer& L = D.L[l];
        L.H = p->L[l].H;
        L.W = p->L[l].W;
        L.Hc = l + 1 < p->n_layers ? p->L[l + 1].H : 0;
        L.Wc = l + 1 < p->n_layers ? p->L[l + 1].W : 0;
        L.pyr_off = p->L[l].float_off;
        L.prm_off = o;
        L.C = dec_in_channels(p, l);
        L.coarsest = l == p->n_layers - 1;
        o += dec_layer_params(L.C);
    }
    D.prm_out = o;
    D.prm = params;
    D.pyramid = pyramid;
    D.wpack = reinterpret_cast<__half*>(b + wl.wpack);
    D.X = reinterpret_cast<__half*>(b + wl.X);
    D.Y[0] = reinterpret_cast<float*>(b + wl.Y0);
    D.Y[1] = reinterpret_cast<float*>(b + wl.Y1);
    D.out = out;

    CUtensorMap tmB;
    {
        const cuuint64_t dims[2] = {(cuuint64_t)kDecXC, (cuuint64_t)p->n_layers * kDecTaps * kDecN};
        const cuuint64_t strides[1] = {(cuuint64_t)kDecXC * 2};
        const cuuint32_t box[2] = {(cuuint32_t)kDecXC, (cuuint32_t)kDecN};
        const cuuint32_t estr[2] = {1, 1};
        if (encode(&tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, D.wpack, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            snprintf(g_msg, sizeof(g_msg), "TRIPS_ERR_CUDA: weight tensor map");
            return TRIPS_ERR_CUDA;
        }
    }
    static bool attr_dev[kMaxDevices] = {};
    {
        const int dev = current_device();
        std::lock_guard<std::mutex> lk(g_dev_mu);
        if (!attr_dev[dev]) {
            int rc = cuda_status(cudaFuncSetAttribute(k_dec_conv, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmem));
            if (rc) return rc;
            attr_dev[dev] = true;
        }
    }
    int rc;
    {
        const int64_t tot = (int64_t)p->n_layers * kDecTaps * kDecN * kDecXC;
        k_dec_pack<<<(int)std::min<int64_t>((tot + 255) / 256, 148 * 16), 256, 0, st>>>(D);
        if ((rc = check_launch())) return rc;
    }
    const int sms = num_sms();
    for (int l = p->n_layers - 1; l >= 0; --l) {
        const DecLayer& L = D.L[l];
        const dim3 pg((L.W + kPrepW - 1) / kPrepW, (L.H + kPrepH - 1) / kPrepH);
        if (D.xc == 48) k_dec_prep<6><<<pg, 256, 0, st>>>(D, l);
        else k_dec_prep<8><<<pg, 256, 0, st>>>(D, l);
        if ((rc = check_launch())) return rc;
        CUtensorMap tmX;
        const cuuint64_t dims[3] = {(cuuint64_t)D.xc, (cuuint64_t)L.W, (cuuint64_t)L.H};
        const cuuint64_t strides[2] = {(cuuint64_t)D.xc * 2, (cuuint64_t)L.W * D.xc * 2};
        const cuuint32_t box[3] = {(cuuint32_t)kDecXC, (cuuint32_t)(TRIPS_DEC_ROWS ? kDecRowPix : kDecM), 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        if (encode(&tmX, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, D.X, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            snprintf(g_msg, sizeof(g_msg), "TRIPS_ERR_CUDA: activation tensor map");
            return TRIPS_ERR_CUDA;
        }
        const int ntiles = L.H * ((L.W + kDecM - 1) / kDecM);
        k_dec_conv<<<std::min(ntiles, sms), kDecThreads, kDecSmem, st>>>(tmX, tmB, D, l);
        if ((rc = check_launch())) return rc;
    }
    return TRIPS_OK;
}

#ifdef TRIPS_KNN_STATS
// experiment builds only: kNN query counters (see knn.cuh)
int trips_debug_knn_stats(unsigned long long* host4, int reset)
{
    if (cudaMemcpyFromSymbol(host4, g_knn_stats, 4 * sizeof(unsigned long long)) != cudaSuccess) return TRIPS_ERR_CUDA;
    if (reset) {
        unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(g_knn_stats, z, sizeof(z));
    }
    return TRIPS_OK;
}
#endif

#ifdef TRIPS_PHASE_CLOCK
// experiment builds only: k_raster per-phase clocks (see kernels.cuh)
int trips_debug_phase_clocks(unsigned long long* host8, int reset)
{
    if (cudaMemcpyFromSymbol(host8, g_pclk, 8 * sizeof(unsigned long long)) != cudaSuccess) return TRIPS_ERR_CUDA;
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_pclk, z, sizeof(z));
    }
    return TRIPS_OK;
}
#endif

size_t trips_morton_workspace_bytes(int64_t n)
{
    if (n < 0) return 0;
    const size_t N = (size_t)(n > 0 ? n : 1);
    const size_t nblk = (N + kSortBlock - 1) / kSortBlock;
    return 4 * align256(N * 4) + align256(256 * nblk * 4) + align256((256 * nblk + 1023) / 1024 * 4) + align256(6 * 4);
}

int trips_morton_order(void* ws, int64_t n, const float* pos, int32_t* perm_out, void* stream)
{
    if (!ws || n < 0 || (n > 0 && (!pos || !perm_out))) return TRIPS_ERR_ARG;
    if (n >= (int64_t(1) << 31)) return TRIPS_ERR_CAPACITY;
    if (!aligned(ws, 256) || !aligned(pos, 4) || !aligned(perm_out, 4)) return TRIPS_ERR_ALIGN;
    if (n == 0) return TRIPS_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t N = (size_t)n;
    MortonWs W;
    W.n = (int)n;
    W.nblk = (int)((N + kSortBlock - 1) / kSortBlock);
    W.last_pass = 3;
    char* b = static_cast<char*>(ws);
    size_t o = 0;
    W.keys[0] = reinterpret_cast<uint32_t*>(b + o); o += align256(N * 4);
    W.keys[1] = reinterpret_cast<uint32_t*>(b + o); o += align256(N * 4);
    W.vals[0] = reinterpret_cast<uint32_t*>(b + o); o += align256(N * 4);
    W.vals[1] = reinterpret_cast<uint32_t*>(b + o); o += align256(N * 4);
    W.hist = reinterpret_cast<uint32_t*>(b + o); o += align256(256 * (size_t)W.nblk * 4);
    W.bsum = reinterpret_cast<uint32_t*>(b + o); o += align256((256 * (size_t)W.nblk + 1023) / 1024 * 4);
    W.bbox = reinterpret_cast<uint32_t*>(b + o);
    int rc = cuda_status(cudaMemsetAsync(W.bbox, 0xff, 3 * 4, st));
    if (rc) return rc;
    if ((rc = cuda_status(cudaMemsetAsync(W.bbox + 3, 0, 3 * 4, st)))) return rc;
    k_bbox<<<std::min(W.nblk * 16, 148 * 8), 256, 0, st>>>(W, pos);
    if ((rc = check_launch())) return rc;
    k_codes<<<(W.n + 255) / 256, 256, 0, st>>>(W, pos);
    if ((rc = check_launch())) return rc;
    for (int pass = 0; pass < 4; ++pass) {
        k_sort_hist<<<W.nblk, 256, 0, st>>>(W, pass);
        if ((rc = check_launch())) return rc;
        if ((rc = sort_scan(W, st))) return rc;
        k_sort_scatter<<<W.nblk, 256, 0, st>>>(W, pass, reinterpret_cast<uint32_t*>(perm_out));
        if ((rc = check_launch())) return rc;
    }
    return TRIPS_OK;
}

int trips_microbench(int32_t op, int32_t pattern, void* buf, int64_t bytes, int32_t row_bytes, int64_t ops, void* stream,
                     double* ms_out, int64_t* ops_done)
{
    if (op < kMbRedV4 || op > kMbLdV4 || (pattern != 0 && pattern != 1) || !buf || !ms_out || ops <= 0)
        return TRIPS_ERR_ARG;
    if (row_bytes < 16 || row_bytes % 16 || bytes < (int64_t)row_bytes * 64) return TRIPS_ERR_ARG;
    if (!aligned(buf, 16)) return TRIPS_ERR_ALIGN;
    uint64_t rows = 1;
    while (rows * 2 * (uint64_t)row_bytes <= (uint64_t)bytes) rows *= 2;
    const int blocks = num_sms() * 8, threads = 256;
    const int64_t tot = (int64_t)blocks * threads;
    const uint32_t iters = (uint32_t)std::max<int64_t>(1, (ops + tot - 1) / tot);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint32_t* sink = reinterpret_cast<uint32_t*>(buf);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    switch (op) {
    case kMbRedV4: k_microbench<kMbRedV4><<<blocks, threads, 0, st>>>((char*)buf, rows - 1, row_bytes, pattern, iters, 1u, sink); break;
    case kMbRedF32: k_microbench<kMbRedF32><<<blocks, threads, 0, st>>>((char*)buf, rows - 1, row_bytes, pattern, iters, 2u, sink); break;
    case kMbAtomU32: k_microbench<kMbAtomU32><<<blocks, threads, 0, st>>>((char*)buf, rows - 1, row_bytes, pattern, iters, 3u, sink); break;
    case kMbStV4: k_microbench<kMbStV4><<<blocks, threads, 0, st>>>((char*)buf, rows - 1, row_bytes, pattern, iters, 4u, sink); break;
    default: k_microbench<kMbLdV4><<<blocks, threads, 0, st>>>((char*)buf, rows - 1, row_bytes, pattern, iters, 5u, sink); break;
    }
    int rc = check_launch();
    cudaEventRecord(b, st);
    float ms = 0.f;
    if (!rc) rc = cuda_status(cudaEventSynchronize(b));
    if (!rc) rc = cuda_status(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ms_out = ms;
    if (ops_done) *ops_done = (int64_t)iters * tot;
    return rc;
}

const char* trips_status_string(int status)
{
    switch (status) {
    case TRIPS_OK: return "TRIPS_OK";
    case TRIPS_ERR_ARG: return "TRIPS_ERR_ARG: invalid argument";
    case TRIPS_ERR_ALIGN: return "TRIPS_ERR_ALIGN: misaligned pointer";
    case TRIPS_ERR_CAPACITY: return "TRIPS_ERR_CAPACITY: n exceeds the plan's max_points";
    case TRIPS_ERR_STATE: return "TRIPS_ERR_STATE: call order violated or workspace mismatch";
    case TRIPS_ERR_CUDA: return g_msg[0] ? g_msg : "TRIPS_ERR_CUDA";
    default: return "unknown status";
    }
}

}  // extern "C"
