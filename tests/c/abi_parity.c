/*
 * Pure C user of the C ABI (include/trips.h): no Python, no torch.  Test infrastructure
 * (tests/test_c_abi.py builds and runs it).  It allocates device memory with the CUDA
 * runtime, runs project -> forward (saved) -> backward through libtrips.so on a seeded
 * random scene, and compares against the CPU oracle (oracle/liboracle_f32.so, called
 * through its own C entry points, declared here -- the two libraries share no header):
 *   - per-pixel fragment counts and kept lists bit-exact (SURVEY.md 8(c) parity bar),
 *   - features |C_gpu - C_ora| <= 1e-5 * M_C (per channel magnitude from the oracle),
 *   - gradients |g_gpu - g_ora| <= 1e-3 * M_g per element.
 * Also exercises the documented error paths (TRIPS_ERR_STATE for backward before forward).
 * Exit status 0 = pass.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "trips.h"

/* ---- oracle entry points (oracle/trips_oracle.c) ---- */
typedef struct {
    float fx, fy, cx, cy, f;
    float R[9], t[3];
    int32_t width, height;
    float near_plane;
} ora_camera;
typedef struct {
    int64_t n_culled, n_visible, n_frag, n_kept, n_trunc_pixels, max_list;
} ora_stats;
int oracle_forward(const ora_camera* cam, int n_layers, int F, int64_t n, const float* pos, const float* sw,
                   const float* alpha, const float* desc, double* pyramid, double* pyramid_mag, uint32_t* counts,
                   int32_t* kept, const uint8_t* mask, ora_stats* stats);
int oracle_backward(const ora_camera* cam, int n_layers, int F, int64_t n, const float* pos, const float* sw,
                    const float* alpha, const float* desc, const float* grad_pyramid, double* grad,
                    double* grad_mag, const uint8_t* mask, double* grad_cam, double* grad_cam_mag);

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 2;                                                                          \
        }                                                                                      \
    } while (0)
#define TK(x)                                                                                  \
    do {                                                                                       \
        int r_ = (x);                                                                          \
        if (r_ != TRIPS_OK) {                                                                  \
            fprintf(stderr, "trips error %d (%s) at %s:%d\n", r_, trips_status_string(r_), __FILE__, __LINE__); \
            return 3;                                                                          \
        }                                                                                      \
    } while (0)

/* splitmix64 -> uniform [0, 1) (input generation only; no method arithmetic) */
static uint64_t g_state = 0x5eed;
static double urand(void)
{
    uint64_t z = (g_state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

int main(void)
{
    const int W = 72, H = 53, NL = 4, F = 4;
    const int64_t n = 1500;
    /* scene: points in front of an identity camera, pixel targets over (and beyond) the
     * image, sizes spanning the eps branch, two-layer and clamp cases */
    float* pos = malloc(sizeof(float) * 3 * n);
    float* sw = malloc(sizeof(float) * n);
    float* al = malloc(sizeof(float) * n);
    float* de = malloc(sizeof(float) * n * F);
    const float fx = 70.f;
    for (int64_t i = 0; i < n; ++i) {
        const double z = 1.0 + 3.0 * urand();
        const double u = -6.0 + (W + 12) * urand(), v = -6.0 + (H + 12) * urand();
        const double s = exp2(-3.0 + 7.5 * urand());
        pos[3 * i + 0] = (float)((u - (W - 1) / 2.0) * z / fx);
        pos[3 * i + 1] = (float)((v - (H - 1) / 2.0) * z / fx);
        pos[3 * i + 2] = (float)z;
        sw[i] = (float)(s * z / fx);
        al[i] = (float)(0.05 + 0.9 * urand());
        for (int c = 0; c < F; ++c) de[i * F + c] = (float)(2.0 * urand() - 1.0);
    }
    trips_camera cam;
    memset(&cam, 0, sizeof(cam));
    cam.fx = fx; cam.fy = fx; cam.cx = (W - 1) / 2.f; cam.cy = (H - 1) / 2.f; cam.f = fx;
    cam.R[0] = cam.R[4] = cam.R[8] = 1.f;
    cam.width = W; cam.height = H; cam.near_plane = 0.01f;

    trips_config cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.num_layers = NL; cfg.num_features = F;
    trips_plan* plan = NULL;
    TK(trips_plan_create(&cfg, W, H, n, &plan));
    const int64_t P = trips_num_pixels(plan), PF = trips_pyramid_floats(plan);
    const int G = 5 + F;       /* flat gradient buffer [pos_size n x 4 | desc n x F | opacity n] */

    float *d_pos, *d_sw, *d_al, *d_de, *d_pyr, *d_gpyr, *d_grad;
    void *d_ws, *d_exp;
    CK(cudaMalloc((void**)&d_pos, sizeof(float) * 3 * n));
    CK(cudaMalloc((void**)&d_sw, sizeof(float) * n));
    CK(cudaMalloc((void**)&d_al, sizeof(float) * n));
    CK(cudaMalloc((void**)&d_de, sizeof(float) * n * F));
    CK(cudaMalloc((void**)&d_pyr, sizeof(float) * PF));
    CK(cudaMalloc((void**)&d_gpyr, sizeof(float) * PF));
    CK(cudaMalloc((void**)&d_grad, sizeof(float) * n * G));
    CK(cudaMalloc(&d_ws, trips_workspace_bytes(plan)));
    CK(cudaMalloc(&d_exp, sizeof(int32_t) * P * 16));
    CK(cudaMemcpy(d_pos, pos, sizeof(float) * 3 * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_sw, sw, sizeof(float) * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_al, al, sizeof(float) * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_de, de, sizeof(float) * n * F, cudaMemcpyHostToDevice));
    float* gpyr = malloc(sizeof(float) * PF);
    for (int64_t k = 0; k < PF; ++k) gpyr[k] = (float)(2.0 * urand() - 1.0);
    CK(cudaMemcpy(d_gpyr, gpyr, sizeof(float) * PF, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_grad, 0, sizeof(float) * n * G));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));

    int fails = 0;
    /* documented call-order error: backward before any forward */
    TK(trips_project(plan, d_ws, &cam, n, d_pos, d_sw, d_al, d_de, NULL, NULL, st));
    float *d_gps = d_grad, *d_gde = d_grad + 4 * n, *d_gop = d_grad + (4 + F) * n;
    if (trips_splat_backward(plan, d_ws, d_gpyr, d_gps, d_gop, d_gde, NULL, st) != TRIPS_ERR_STATE) {
        fprintf(stderr, "backward before forward was not rejected\n");
        ++fails;
    }
    TK(trips_splat_forward(plan, d_ws, d_pyr, TRIPS_FWD_SAVE_FOR_BACKWARD, st));
    TK(trips_splat_backward(plan, d_ws, d_gpyr, d_gps, d_gop, d_gde, NULL, st));
    CK(cudaStreamSynchronize(st));

    float* pyr = malloc(sizeof(float) * PF);
    float* grad = malloc(sizeof(float) * n * G);
    uint32_t* cnt = malloc(sizeof(uint32_t) * P);
    int32_t* kept = malloc(sizeof(int32_t) * P * 16);
    CK(cudaMemcpy(pyr, d_pyr, sizeof(float) * PF, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(grad, d_grad, sizeof(float) * n * G, cudaMemcpyDeviceToHost));
    TK(trips_debug_export(plan, d_ws, TRIPS_EXPORT_COUNTS, d_exp, st));
    CK(cudaMemcpy(cnt, d_exp, sizeof(uint32_t) * P, cudaMemcpyDeviceToHost));
    TK(trips_debug_export(plan, d_ws, TRIPS_EXPORT_KEPT, d_exp, st));
    CK(cudaMemcpy(kept, d_exp, sizeof(int32_t) * P * 16, cudaMemcpyDeviceToHost));
    trips_stats gst;
    TK(trips_read_stats(plan, d_ws, &gst, st));

    /* oracle */
    ora_camera oc;
    memset(&oc, 0, sizeof(oc));
    oc.fx = cam.fx; oc.fy = cam.fy; oc.cx = cam.cx; oc.cy = cam.cy; oc.f = cam.f;
    memcpy(oc.R, cam.R, sizeof(oc.R));
    memcpy(oc.t, cam.t, sizeof(oc.t));
    oc.width = W; oc.height = H; oc.near_plane = cam.near_plane;
    double* opyr = calloc(PF, sizeof(double));
    double* omag = calloc(PF, sizeof(double));
    uint32_t* ocnt = calloc(P, sizeof(uint32_t));
    int32_t* okept = calloc(P * 16, sizeof(int32_t));
    double* og = calloc(n * (5 + F), sizeof(double));
    double* ogm = calloc(n * (5 + F), sizeof(double));
    ora_stats ost;
    if (oracle_forward(&oc, NL, F, n, pos, sw, al, de, opyr, omag, ocnt, okept, NULL, &ost) != 0 ||
        oracle_backward(&oc, NL, F, n, pos, sw, al, de, gpyr, og, ogm, NULL, NULL, NULL) != 0) {
        fprintf(stderr, "oracle failed\n");
        return 4;
    }

    int64_t bad_cnt = 0, bad_kept = 0, bad_feat = 0, bad_grad = 0;
    for (int64_t p = 0; p < P; ++p) bad_cnt += cnt[p] != ocnt[p];
    for (int64_t k = 0; k < P * 16; ++k) bad_kept += kept[k] != okept[k];
    for (int64_t k = 0; k < PF; ++k) bad_feat += fabs((double)pyr[k] - opyr[k]) > 1e-5 * omag[k] + 1e-30;
    for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < 5 + F; ++c) {
            /* oracle row order (d pos, d s_w, d alpha, d tau) from the flat buffer */
            const double g = c < 4 ? grad[4 * i + c] : (c == 4 ? grad[(4 + F) * n + i] : grad[4 * n + i * F + (c - 5)]);
            const double o = og[i * (5 + F) + c], m = ogm[i * (5 + F) + c];
            bad_grad += fabs(g - o) > 1e-3 * m + 1e-30;
        }
    if (gst.n_frag != ost.n_frag || gst.n_kept != ost.n_kept || gst.max_list != ost.max_list) {
        fprintf(stderr, "stats differ: frag %lld/%lld kept %lld/%lld\n", (long long)gst.n_frag,
                (long long)ost.n_frag, (long long)gst.n_kept, (long long)ost.n_kept);
        ++fails;
    }
    printf("C ABI parity: P=%lld frag=%lld kept=%lld | bad counts %lld, kept %lld, features %lld, grads %lld\n",
           (long long)P, (long long)gst.n_frag, (long long)gst.n_kept, (long long)bad_cnt, (long long)bad_kept,
           (long long)bad_feat, (long long)bad_grad);
    fails += (bad_cnt != 0) + (bad_kept != 0) + (bad_feat != 0) + (bad_grad != 0);
    if (gst.n_frag == 0) ++fails;                     /* the scene must exercise the path */

    trips_plan_destroy(plan);
    cudaFree(d_pos); cudaFree(d_sw); cudaFree(d_al); cudaFree(d_de); cudaFree(d_pyr); cudaFree(d_gpyr);
    cudaFree(d_grad); cudaFree(d_ws); cudaFree(d_exp);
    cudaStreamDestroy(st);
    return fails ? 1 : 0;
}
