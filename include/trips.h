/*
 * trips.h -- C ABI of the B200-native TRIPS trilinear point-splatting rasterizer.
 *
 * The operation is the render function Phi of arXiv 2401.06003, Eq. (1)
 * restricted to the rasterizer (no environment map, no decoder network):
 *   camera intrinsics C and pose (R, t), point positions x, world sizes s_w,
 *   descriptors tau, opacities alpha  ->  an n-layer feature pyramid,
 * computed in the paper's three stages (Sec. 3.6):
 *   trips_project        "collecting": project every point, its screen size s = f s_w / z
 *                        (Eq. 2) and its two pyramid layers
 *                        (Eq. 4), count the work per pyramid tile;
 *   trips_splat_forward  "splatting" + "accumulation": bin points into per-tile lists,
 *                        build per-pixel fragment lists, keep the 16 nearest by
 *                        (depth, point index) (Sec. 3.2) and
 *                        alpha-blend them front to back (Eqs. 5-6);
 *                        the sorted lists are stored for the backward;
 *   trips_splat_backward gradients w.r.t. positions, world sizes, opacities and
 *                        descriptors (chain rule of Eqs. 2-6).
 * Readings of the paper where it is silent are listed in DESIGN.md ("Readings", Q1-Q24).
 *
 * CONVENTIONS
 *  - All array pointers are CUDA DEVICE pointers owned by the caller, except `trips_camera*`,
 *    `trips_config*`, `trips_stats*` and output scalars, which are host pointers.
 *  - The library never allocates device memory.  The caller allocates one workspace of
 *    trips_workspace_bytes() bytes (256-byte aligned, contents need not be initialised) per
 *    plan; a workspace belongs to one plan.
 *  - All work is enqueued asynchronously on `stream` (a cudaStream_t, passed as void*; NULL =
 *    legacy default stream).  Nothing synchronises except trips_read_stats,
 *    trips_debug_export and trips_read_stage_ms.  Kernel faults surface at the caller's next
 *    synchronisation.
 *  - On error a negative trips_status is returned and NOTHING is enqueued.
 *  - Points that are behind the near plane, non-finite, or have negative size are CULLED
 *    (counted in the stats), not errors.  alpha outside [0,1] is caller error: results are
 *    defined arithmetically but meaningless.
 *  - A plan is not thread-safe; distinct plans/workspaces are independent.
 */
#ifndef TRIPS_H_
#define TRIPS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Pinhole camera (Sec. 3.1).  Pixel (i, j) of layer 0 has its centre at
 * (i, j); layer l is addressed with x_l = x * 2^-l (reading Q7).  OpenCV axes: x right,
 * y down, z forward; world -> view p = R x + t (reading Q24). */
typedef struct {
    float fx, fy, cx, cy;      /* pixels */
    float f;                   /* focal length of Eq. (2); callers use sqrt(fx*fy) (Q6) */
    float R[9];                /* row-major world -> view rotation */
    float t[3];
    int32_t width, height;     /* layer-0 size; must equal the plan's */
    float near_plane;          /* points with !(z > near_plane) are culled (Q14); > 0 */
} trips_camera;

typedef struct {
    int32_t num_layers;        /* n in [1, 16]  (paper studies 3..8) */
    int32_t num_features;      /* F in [1, 32]  (paper uses 4..8) */
    float t_min;               /* 0 = the exact definition.  In [0, 1): variant with early
                                  termination -- a pixel's kept list ends with the fragment
                                  after which the fp32 transmittance T = prod (1 - gamma) drops
                                  below t_min (reading Q17) */
    int32_t coarse_layers;     /* 0 = the exact definition.  c > 0: coarse-layer inclusion
                                  ("we include points from coarser layers
                                  during blending (in the usual way)", reading Q22): the list
                                  blended at pyramid pixel (l, x, y) is the 16 front-most of
                                  the union of the fragment lists of (l + d, x >> d, y >> d),
                                  d = 0 .. min(c, n - 1 - l), ordered by (z, i, d); each
                                  fragment keeps its own gamma (Eq. 3 in its own layer).
                                  Per-pixel counts and stats stay the pixel's own list.  Costs
                                  an extra 16 keys per pyramid pixel of workspace (each pixel's
                                  own sorted list).  c > n - 1 behaves as n - 1; c < 0 is an
                                  error. */
} trips_config;

typedef struct trips_plan trips_plan;   /* opaque, host memory, owned by the library */

typedef struct {
    int64_t n_culled;          /* points culled in the last trips_project */
    int64_t n_visible;
    int64_t n_pairs;           /* (point, pyramid tile) work items */
    int64_t n_frag;            /* fragments = sum of per-pixel list lengths */
    int64_t n_kept;            /* sum over pixels of min(16, list length) */
    int64_t n_trunc_pixels;    /* pixels whose list was longer than 16 */
    int64_t max_list;          /* longest per-pixel list */
    int64_t n_kept_pairs;      /* (point, tile) pairs with >= 1 kept fragment (the backward's
                                  reduction units; 0 with coarse_layers > 0) */
} trips_stats;

typedef enum {
    TRIPS_OK = 0,
    TRIPS_ERR_ARG = -1,        /* null required pointer, n < 0, bad config/camera */
    TRIPS_ERR_ALIGN = -2,      /* a device pointer violates the alignment stated below */
    TRIPS_ERR_CAPACITY = -3,   /* n > max_points of the plan */
    TRIPS_ERR_STATE = -4,      /* call order violated (see each call) or different workspace */
    TRIPS_ERR_CUDA = -5        /* a launch failed; see trips_status_string */
} trips_status;

/* Flags of trips_splat_forward. */
#define TRIPS_FWD_SAVE_FOR_BACKWARD 1u

/* What trips_debug_export copies (into a caller DEVICE buffer). */
typedef enum {
    TRIPS_EXPORT_COUNTS = 1,   /* uint32[P]: per-pixel list length, pyramid pixel order     */
    TRIPS_EXPORT_KEPT = 2,     /* int32[P*16]: kept point indices in blend order, -1 padded */
    TRIPS_EXPORT_KEPT_LAYER = 3, /* int32[P*16]: layer offset d of each kept entry (0 unless
                                  coarse_layers > 0), -1 padded */
    TRIPS_EXPORT_SCREEN_GRADS = 4 /* float[n][4+F]: screen-space gradients of the last
                                  trips_splat_backward's grad_pyramid:
                                  (dL/dx, dL/dy, dL/ds in layer-0 pixels, dL/dalpha, dL/dtau[F])
                                  of this view, before the projection chain.  The caller keeps
                                  that grad_pyramid unchanged until the export. */
} trips_export;

/* ---- plan ------------------------------------------------------------------------- */

/* Creates a plan for images of width x height and up to max_points points.  Plans whose pyramid
 * has more 16 x 16 tiles than the binning kernels' shared-memory counters hold (49 152, e.g. 8K
 * frames) bin with global-memory counters instead (same results; slower binning); setting the
 * environment variable TRIPS_FORCE_GLOBAL_BINNING=1 before creating a plan selects that path
 * at any size (tests).
 * Errors: TRIPS_ERR_ARG (null, bad config, width/height < 1 or > 32768, max_points < 0 or
 * >= 2^28, more than 2^20 tiles). */
int trips_plan_create(const trips_config* cfg, int32_t width, int32_t height, int64_t max_points,
                      trips_plan** out);
void trips_plan_destroy(trips_plan* plan);

/* Workspace size in bytes for this plan (caller allocates, 256-B aligned). */
size_t trips_workspace_bytes(const trips_plan* plan);

/* P = number of pyramid pixels = sum_l ceil(H/2^l) * ceil(W/2^l) (reading Q8). */
int64_t trips_num_pixels(const trips_plan* plan);

/* Pyramid floats = (F+1) * P.  Layout: layer-major; layer l is planar [(F+1), H_l, W_l];
 * channel F is the accumulated opacity A = sum_m T_m gamma_m (reading Q16). */
int64_t trips_pyramid_floats(const trips_plan* plan);

/* Layer l geometry: *h = H_l, *w = W_l, *offset_floats = float offset of layer l in the
 * pyramid.  Any output pointer may be NULL.  Errors: TRIPS_ERR_ARG (l out of range). */
int trips_layer_dims(const trips_plan* plan, int32_t l, int32_t* h, int32_t* w,
                     int64_t* offset_floats);

/* ---- the three stages -------------------------------------------------------------- */

/* Stage 1, "collecting".  Projects the n points (Eq. 2), selects their
 * layers (Eq. 4) and counts the (point, tile) work per pyramid tile.  Stores per-point
 * screen records in the workspace.  Starts a new frame on this plan (any saved forward
 * state is invalidated).
 *   pos        float[n][3] world positions, 4-byte aligned
 *   world_size float[n]    s_w
 *   opacity    float[n]    alpha
 *   desc       float[n][F] descriptors tau, row-major, 4-byte aligned.  When F % 4 == 0 and
 *              desc is 16-B aligned, trips_splat_forward/backward of this frame gather the
 *              descriptors from these rows directly (no per-view copy): the caller keeps
 *              desc allocated and unmodified until the frame's last forward/backward.
 *              Otherwise a padded copy is taken here.
 *   level_out  int8[n]  nullable: -1 culled, else bits 0-3 lowest layer, 0x10 two layers,
 *                       0x20 eps branch (s < 1), 0x40 clamped (s >= 2^(n-1))
 *   proj_out   float[n][4] nullable: (x, y, z, s), NaN rows for culled points
 * Errors: TRIPS_ERR_ARG, TRIPS_ERR_CAPACITY (n > max_points), TRIPS_ERR_ALIGN (ws not 256-B
 * aligned), TRIPS_ERR_CUDA. */
int trips_project(trips_plan* plan, void* ws, const trips_camera* cam, int64_t n,
                  const float* pos, const float* world_size, const float* opacity,
                  const float* desc, int8_t* level_out, float* proj_out, void* stream);

/* Stages 2-3.  Writes the whole pyramid (trips_pyramid_floats floats,
 * 16-B aligned).  With TRIPS_FWD_SAVE_FOR_BACKWARD the sorted kept lists stay in the
 * workspace for trips_splat_backward.  Errors: TRIPS_ERR_STATE (no trips_project since
 * the plan was created or since the last forward, or ws differs), TRIPS_ERR_ARG,
 * TRIPS_ERR_ALIGN, TRIPS_ERR_CUDA. */
int trips_splat_forward(trips_plan* plan, void* ws, float* pyramid, uint32_t flags, void* stream);

/* Backward of the last saved forward: gradients w.r.t. positions, world sizes, opacities and
 * descriptors (chain rule of Eqs. 2-6, sorted lists reused).
 * grad_pyramid has the pyramid layout (16-B aligned).  Gradients are ACCUMULATED (+=) so that
 * several views sum into one set of buffers (reading Q21); the caller zeroes them once per batch:
 *   grad_pos_size  float[n][4]  (dL/dx, dL/dy, dL/dz, dL/ds_w) per point, 16-B aligned.  Position
 *                               and world size share one 16-byte row so that one vector reduction
 *                               carries both (SURVEY.md 8(b) lists them as two arrays; DESIGN.md
 *                               "Boundary" records this and the other deviations)
 *   grad_opacity   float[n]     dL/dalpha, 4-B aligned
 *   grad_desc      float[n][F]  dL/dtau, row-major, 4-B aligned (16-B aligned rows with F % 4 == 0
 *                               use 16-byte vector reductions)
 * Laid out contiguously ([4n | F n | n] floats) the three form one (5+F) n-float buffer -- 36 B
 * per point at F = 4 -- that a multi-GPU caller all-reduces once per batch.
 * grad_camera (nullable, device float[17], 4-B aligned) receives += the gradient w.r.t. the
 * camera of the last trips_project (the paper optimises camera parameters):
 * (dR00..dR22 row-major, dt0..dt2, dfx, dfy, dcx, dcy, df) for p = R x + t, x = fx p_x/z + cx,
 * y = fy p_y/z + cy, s = f s_w/z.  Passing NULL costs nothing.
 * Summation order: fragments of different pixels reduce into a point's row with float atomics
 * (red.global.add), so the low bits of the gradients vary from run to run (the forward is
 * deterministic).  May be called more than once per forward.  Errors: TRIPS_ERR_STATE (last
 * forward not saved, or ws differs), TRIPS_ERR_ARG (null buffer with n > 0), TRIPS_ERR_ALIGN,
 * TRIPS_ERR_CUDA. */
int trips_splat_backward(trips_plan* plan, void* ws, const float* grad_pyramid, float* grad_pos_size,
                         float* grad_opacity, float* grad_desc, float* grad_camera, void* stream);

/* ---- introspection ----------------------------------------------------------------- */

/* Synchronises `stream` and reads the statistics of the last project/forward. */
int trips_read_stats(const trips_plan* plan, const void* ws, trips_stats* out, void* stream);

/* Synchronises `stream` and copies debug state of the last forward into the device buffer
 * dst (sizes in trips_export).  Errors: TRIPS_ERR_STATE (no saved forward; SCREEN_GRADS: no
 * backward since the last trips_project), TRIPS_ERR_ARG, TRIPS_ERR_ALIGN. */
int trips_debug_export(const trips_plan* plan, const void* ws, int32_t what, void* dst, void* stream);

/* Per-stage device timing.  When enabled, CUDA events bracket every kernel stage
 * (0 count = k_count, 1 emit = k_emit, 2 tscan = k_tscan, 3 raster = k_raster [+ k_coarse_blend],
 * 4 backward = k_backward_pairs | k_backward_coarse); trips_read_stage_ms synchronises
 * the events and returns the accumulated milliseconds and launch counts since the last
 * reset.  Returns the number of stages written. */
int trips_set_profiling(trips_plan* plan, int32_t enable);
int trips_read_stage_ms(trips_plan* plan, double* ms, int64_t* launches, int32_t max_stages,
                        int32_t reset);

/* ---- data layout utility ------------------------------------------------------------ */

/* One-time spatial ordering of a point cloud (not part of the per-view path).  Writes a
 * permutation perm[n] (int32, device) such that pos[perm[0]], pos[perm[1]], ... follow a 3-D
 * Morton (Z-order) curve over the cloud's bounding box, 10 bits per axis; ties keep index
 * order; non-finite points go last.  Applying it once to all per-point arrays makes every
 * per-view gather and gradient reduction spatially coherent (cache lines and tiles shared by
 * neighbouring indices), as in the spatially sorted batches of the software point rasterizer
 * the paper builds on (PAPER.md:160 cites it as [schutz2022software]).  Results of the
 * rasterizer are unchanged up to the point-index tie-break of equal depths (reading Q12).
 *   ws   device scratch of trips_morton_workspace_bytes(n) bytes, 256-B aligned
 *   pos  float[n][3] device, 4-B aligned
 * Errors: TRIPS_ERR_ARG, TRIPS_ERR_ALIGN, TRIPS_ERR_CAPACITY (n >= 2^31), TRIPS_ERR_CUDA. */
size_t trips_morton_workspace_bytes(int64_t n);
int trips_morton_order(void* ws, int64_t n, const float* pos, int32_t* perm_out, void* stream);

/* Point-size initialisation ("Point sizes are initialized with the average
 * distance to the four nearest neighbor"; reading Q25): size_out[i] = mean Euclidean distance
 * from point i to its K = min(4, #finite points - 1) nearest other finite points, neighbours
 * ordered by (squared distance, index) with d^2 = ((dx^2 + dy^2) + dz^2) in fp32 and the mean
 * (((d1 + d2) + d3) + d4) / K in fp32 (bit-identical to a brute-force evaluation); 0 for
 * non-finite points.  One-time initialisation, not part of the per-view path.
 *   ws       device scratch of trips_knn_workspace_bytes(n) bytes, 256-B aligned
 *   pos      float[n][3] device;  size_out float[n] device;  nbr_out nullable int32[n][4]
 *            (neighbour indices in order, -1 padded)
 * Errors: TRIPS_ERR_ARG, TRIPS_ERR_ALIGN, TRIPS_ERR_CAPACITY (n >= 2^30), TRIPS_ERR_CUDA. */
size_t trips_knn_workspace_bytes(int64_t n);
int trips_knn_sizes(void* ws, int64_t n, const float* pos, float* size_out, int32_t* nbr_out, void* stream);

/* ---- decoder ---------------------------------------------------------------------- */

/* The gated-convolution decoder over the pyramid (Sec.
 * 3.3 and Fig. fig:conv: "a single gated convolution in each layer with a self-bypass connection
 * and a feature size of 32 ... a bilinear upsampling operation for all layers except the final
 * one, merging the output with the subsequent level"; readings D1-D8 in DESIGN.md):
 *   for l = n-1 .. 0:  x_l = [U(y_{l+1}) cropped to the layer (32 ch, absent at l = n-1),
 *                             pyramid layer l (F features + opacity)]
 *                      y_l = ELU(conv3x3(x_l; Wf_l) + bf_l) * sigmoid(conv3x3(x_l; Wg_l) + bg_l)
 *                            + Wb_l x_l                         (zero-padded 3x3 convolutions)
 *   out = Wo y_0 + bo                                           (1x1, out_channels = 3 or 27)
 * U = bilinear 2x upsampling with half-pixel centres, edge-clamped.  The 3x3 convolutions and
 * the bypass run on the tcgen05 tensor cores with fp16 operands (x_l and the weights rounded to
 * half) and fp32 accumulation; biases, activations and the output projection in fp32.
 *   params  float[trips_decoder_param_count(plan, out_channels)] device, layer by layer
 *           (l = 0 .. n-1): Wf [32][C_l][3][3], bf [32], Wg [32][C_l][3][3], bg [32], Wb [32][C_l]
 *           with C_l = F + 1 for the coarsest layer, 32 + F + 1 otherwise (input channel order:
 *           the 32 upsampled channels, then the pyramid's F features and its opacity); then
 *           Wo [out_channels][32], bo [out_channels].  4-B aligned.
 *   pyramid float[trips_pyramid_floats(plan)] device, the layout trips_splat_forward writes
 *   out     float[out_channels][H][W] device (full resolution, planar)
 *   dws     device scratch of trips_decoder_workspace_bytes(plan) bytes, 256-B aligned; holds
 *           the packed fp16 weights and the per-layer activations (independent of the
 *           rasterizer's workspace; the plan only supplies the pyramid geometry).
 * Errors: TRIPS_ERR_ARG (null pointer, out_channels outside [1, 32], F + 1 > 32),
 * TRIPS_ERR_ALIGN, TRIPS_ERR_CUDA (launch failure, no tensor-map encoder). */
int64_t trips_decoder_param_count(const trips_plan* plan, int32_t out_channels);
size_t trips_decoder_workspace_bytes(const trips_plan* plan);
int trips_decode(const trips_plan* plan, void* dws, const float* params, int32_t out_channels,
                 const float* pyramid, float* out, void* stream);

/* ---- measurement ------------------------------------------------------------------ */

/* Memory-operation microbenchmark giving the measured ceilings the backward's gradient
 * reductions are reported against ("random-address red.add.f32 and atomicAdd
 * u32 on L2-resident and DRAM-sized arrays").  Not part of the rasterizer path.
 *   op        0 red.global.add.v4.f32, 1 red.global.add.f32, 2 atomicAdd u32 (result used),
 *             3 st.global.v4 (scatter store), 4 ld.global.cg.v4 (gather load)
 *   pattern   0: every lane an independent random row; 1: the 32 lanes of a warp hit 32
 *             consecutive rows from a random base (spatially coherent, like a Morton cloud)
 *   buf       device buffer of `bytes` bytes, 16-B aligned (contents are modified); the rows
 *             used are the largest power of two of `row_bytes`-byte rows that fit in it
 *   ops       requested operations (rounded up to whole iterations of 8 CTAs x 256 threads
 *             per SM); *ops_done (nullable) receives the count issued
 *   ms_out    device time of the one launch (CUDA events on `stream`); SYNCHRONISES `stream`.
 * Errors: TRIPS_ERR_ARG (bad op/pattern, row_bytes not a multiple of 16, bytes < 64 rows),
 * TRIPS_ERR_ALIGN, TRIPS_ERR_CUDA. */
int trips_microbench(int32_t op, int32_t pattern, void* buf, int64_t bytes, int32_t row_bytes, int64_t ops,
                     void* stream, double* ms_out, int64_t* ops_done);

/* Total kernel launches issued by this library in this process. */
int64_t trips_launch_count(void);

/* Human-readable text for a status code (includes the last CUDA error for TRIPS_ERR_CUDA). */
const char* trips_status_string(int status);

#ifdef __cplusplus
}
#endif
#endif /* TRIPS_H_ */
