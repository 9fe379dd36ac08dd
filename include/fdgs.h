/*
 * fdgs.h -- C ABI of libfdgs.so, the B200 (sm_100a) render hot path of
 * 4DGS-1K (arXiv 2503.16422).
 *
 * Citations: P:n = PAPER.md line n (the paper's LaTeX source), with its
 * section / equation.  DESIGN.md lists every reading taken where the paper is
 * silent (R1..R20) and the pinned decision path.
 *
 * Conventions for every entry point
 *   - All pointers named d_* / documented "device" are CUDA device pointers;
 *     "host" pointers are ordinary host memory.  The caller owns every buffer.
 *     The library never allocates or frees device memory; scratch lives in a
 *     caller-provided workspace whose size the *_workspace_bytes functions
 *     return (256-byte aligned base required).  The two handle types
 *     (fdgs_render_graph, fdgs_pipeline) own host objects, CUDA graphs and
 *     events, released by their destroy calls.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     All work is stream-ordered; functions documented "async" never
 *     synchronise the host.
 *   - Every function returns fdgs_status.  No C++ exception crosses the ABI;
 *     nothing aborts.  fdgs_last_error() returns a thread-local message for the
 *     last non-OK status of the calling thread.
 *   - Layouts are PyTorch-contiguous float32 / uint32 arrays.
 *   - Re-entrant: there is no global mutable state besides the thread-local
 *     error string and two process-wide, initialise-once values (the device's
 *     SM count and the kernels' shared-memory attributes, both set under
 *     std::call_once / static initialisation); concurrent calls on different
 *     workspaces are safe.  The library reads no environment variables: every
 *     tuning choice (grid shapes, unroll factors) is a compile-time constant.
 */
#ifndef FDGS_H
#define FDGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDGS_ABI_VERSION 2  /* 2: fdgs_scene.d_n, fdgs_pipeline_slot.graph, the pipeline and timed-graph entries */
#define FDGS_TILE 16            /* 16x16-pixel tiles (reading R7) */
#define FDGS_MAX_TILES 16384    /* tile-grid limit of the binning kernel    */

typedef enum {
    FDGS_OK = 0,
    FDGS_ERR_INVALID_ARG = 1,       /* bad pointer / size / camera              */
    FDGS_ERR_INVALID_SCENE = 2,     /* scene violates the invariants below      */
    FDGS_ERR_WORKSPACE_TOO_SMALL = 3,
    FDGS_ERR_OVERFLOW = 4,          /* tile entries exceeded max_entries        */
    FDGS_ERR_CUDA = 5,              /* a CUDA runtime call failed               */
    FDGS_ERR_UNSUPPORTED = 6        /* valid request this build does not serve  */
} fdgs_status;

/* A set of N 4D Gaussians (Sec. 3): mean mu=(x,y,z,t), scales
 * S_4D, rotation R_4D = L(q_l) R(q_r) from a left and a right quaternion,
 * opacity sigma, degree-3 SH colour c_i(d).  All DEVICE pointers,
 * 16-byte aligned, SoA:
 *   mean, scale, rot_l, rot_r : float[n][4]  (rot in (w,x,y,z) order; scales
 *                               are linear standard deviations > 0, R12)
 *   opacity                   : float[n], sigma in (0,1]
 *   log255_opacity            : float[n], L_i = fp32(ln(255 sigma_i)) computed
 *                               in binary64 (fdgs_log255_opacity fills it)
 *   sh                        : float[n][16][3], coefficient k*3+channel
 *   param_stride              : float4 elements between consecutive Gaussians
 *                               in mean/scale/rot_l/rot_r: 0 or 1 = four SoA
 *                               planes; 4 = one interleaved 64-byte record per
 *                               Gaussian {mean, scale, rot_l, rot_r} (what the
 *                               Python Scene allocates: a sparse, mask-driven
 *                               gather then touches one 64-byte DRAM burst per
 *                               Gaussian instead of four)
 *   gid                       : DEVICE uint32[n] or NULL: the ORIGINAL index of
 *                               Gaussian i when this scene is a compacted
 *                               working set (fdgs_scene_compact, ascending
 *                               order kept); records report gid[i].  NULL = i
 *   sh_index, sh_codebook_size: vector-quantised SH (the "Ours-PP" storage of
 *                               P:483, SH "vector quantization" after CompGS):
 *                               when sh_index != NULL, `sh` points to a
 *                               CODEBOOK float[sh_codebook_size][16][3] and
 *                               Gaussian i's coefficients are codebook entry
 *                               sh_index[i] (DEVICE uint16[n]); NULL = dense SH
 * Invariants (checked by fdgs_scene_validate): |‖q‖-1| <= 1e-6, scales > 0,
 * sigma in (0,1], Sigma_44 > 1e-12, sh_index[i] < sh_codebook_size. */
typedef struct {
    int32_t n;
    const float *mean;
    const float *scale;
    const float *rot_l;
    const float *rot_r;
    const float *opacity;
    const float *log255_opacity;
    const float *sh;
    const uint16_t *sh_index;     /* nullable: dense SH                        */
    int32_t sh_codebook_size;     /* entries of the codebook when sh_index set */
    int32_t param_stride;         /* 0/1 SoA planes, 4 interleaved (see above) */
    const uint32_t *gid;          /* nullable: original indices (compacted set) */
    int32_t n_capacity;           /* 0, or >= n: render workspaces are laid out
                                     for max(n, n_capacity) Gaussians, so a full
                                     scene and its working sets share one
                                     workspace layout (no re-zeroing)           */
    const uint32_t *d_n;          /* nullable DEVICE count: the render uses the
                                     first min(*d_n, n) Gaussians (n then is the
                                     arrays' capacity).  Lets a working set whose
                                     size fdgs_scene_compact wrote on the device
                                     be rendered with no host synchronisation   */
} fdgs_scene;

/* Pinhole view "I" of P:126 (HOST struct).  world->camera rotation R
 * (row-major) and translation T, OpenCV axes (x right, y down, z forward),
 * pixel (i,j) has centre (i+0.5, j+0.5), u = fx*x/z + cx (reading R13).
 * Valid iff 1 <= width,height <= 8192, fx,fy > 0, z_near > 0 and
 * ‖R R^T - I‖_inf <= 1e-5.  bg is the background of the composite (R14). */
typedef struct {
    int32_t width, height;
    float fx, fy, cx, cy;
    float R[9];
    float T[3];
    float z_near;
    float bg[3];
} fdgs_camera;

/* Per-frame counters written on the DEVICE by fdgs_render (after the blend). */
typedef struct {
    uint32_t n_act;        /* Gaussians in the active set A = M_l | M_r           */
    uint32_t n_vis;        /* active Gaussians surviving all culls                */
    uint32_t n_entries;    /* (tile, Gaussian) entries E                          */
    uint32_t status;       /* fdgs_status of the frame (OVERFLOW when E > cap)    */
    uint64_t n_evaluated;  /* (pixel, Gaussian) pairs inside the pixel AABB tested
                              before the pixel terminated (Eq. 2 work)            */
    uint64_t n_blended;    /* pairs composited (alpha >= 1/255, not terminated)   */
} fdgs_frame_stats;

const char *fdgs_status_string(fdgs_status s);
const char *fdgs_last_error(void);
int32_t fdgs_abi_version(void);

/* Scene checks of SPEC invariants (degenerate Sigma_t guard).
 * Synchronises `stream`.  *first_bad (host, nullable) receives the lowest
 * offending index or -1.  Returns FDGS_ERR_INVALID_SCENE if any. */
fdgs_status fdgs_scene_validate(const fdgs_scene *scene, int64_t *first_bad, void *d_ws, size_t ws_bytes,
                                void *stream);
size_t fdgs_scene_validate_workspace_bytes(void);

/* L_i = fp32(ln(255 * sigma_i)) evaluated in binary64 (async). d_out: float[n]. */
fdgs_status fdgs_log255_opacity(const float *d_opacity, int32_t n, float *d_out, void *stream);

/* Workspace bytes of fdgs_render for n Gaussians, a width x height image and
 * room for max_entries (tile, Gaussian) entries.  A render workspace must be
 * zero-filled (cudaMemset 0) before its first fdgs_render and again whenever
 * it is reused for a different (n, width, height, max_entries); between those
 * it serves any number of frames on one stream (its look-back tables are
 * epoch-tagged). */
size_t fdgs_render_workspace_bytes(int32_t n, int32_t width, int32_t height, int64_t max_entries);

/* Render one frame at timestamp t (Eq. 1-3) under the key-frame
 * temporal filter (Sec. 4.2.2).  ASYNC, no host synchronisation.
 *   d_mask_l, d_mask_r : DEVICE uint32[ceil(n/32)] masks M(t_l), M(t_r) of the
 *                        two bracketing key-frames, bit i of word i/32 is
 *                        Gaussian i (LSB-first).  The active set is their OR;
 *                        pass the same pointer twice (or d_mask_r = NULL) at a
 *                        key-frame; both NULL = every Gaussian active.
 *   cam                : HOST camera.
 *   t                  : timestamp (may lie outside [0,1]).
 *   d_out_rgb          : DEVICE float[3][height][width] (CHW), C + T*bg.
 *   d_out_T            : DEVICE float[height][width] final transmittance, nullable.
 *   d_stats            : DEVICE fdgs_frame_stats, nullable.
 * Steps: mask OR + cull-first slice (Eq. 1/3) + EWA
 * projection + SH3 colour + order-preserving compaction; stable radix sort of
 * depth keys; stable tile binning; per-tile front-to-back blend (Eq. 2).
 * Device-detected errors (E > max_entries) set d_stats->status; the frame is
 * then undefined and must be re-rendered with a larger workspace.
 * Errors returned: INVALID_ARG (null scene/output, bad camera, n < 0),
 * WORKSPACE_TOO_SMALL, UNSUPPORTED (tile grid > FDGS_MAX_TILES), CUDA. */
fdgs_status fdgs_render(const fdgs_scene *scene, const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                        const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T, void *d_ws,
                        size_t ws_bytes, int64_t max_entries, fdgs_frame_stats *d_stats, void *stream);

/* fdgs_render that also records 5 caller-created CUDA events (host array of
 * cudaEvent_t, passed as void*) on `stream` at the stage boundaries:
 * [0] start, [1] after preprocess (rows 1-4), [2] after the depth sort
 * (row 5a), [3] after tile binning (row 5b), [4] after the blend (row 6).
 * ASYNC; for live per-stage timing (bench.py). */
fdgs_status fdgs_render_timed(const fdgs_scene *scene, const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                              const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T, void *d_ws,
                              size_t ws_bytes, int64_t max_entries, fdgs_frame_stats *d_stats, void *stream,
                              void *const *stage_events);

/* fdgs_render with the blend (row 6) on a second stream: the front end
 * (rows 1-5) runs on `stream`, then `split_event` (a caller-created
 * cudaEvent_t, passed as void*) is recorded on it and `blend_stream` waits for
 * it before the blend.  Lets a caller give the latency-bound front end a
 * higher stream priority than the ALU-bound blend so that consecutive frames
 * interleave.  The workspace is in use until the blend completes on
 * `blend_stream`: the caller must order the workspace's next frame after it.
 * stage_events (nullable) as in fdgs_render_timed ([3], [4] on blend_stream).
 * ASYNC. */
fdgs_status fdgs_render_split(const fdgs_scene *scene, const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                              const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T, void *d_ws,
                              size_t ws_bytes, int64_t max_entries, fdgs_frame_stats *d_stats, void *stream,
                              void *blend_stream, void *split_event, void *const *stage_events);

/* Same as fdgs_render, then synchronises `stream` and returns the frame status
 * (FDGS_ERR_OVERFLOW if E > max_entries).  host_stats (nullable) receives the
 * counters.  For tests and the end-to-end path. */
fdgs_status fdgs_render_checked(const fdgs_scene *scene, const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                                const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T, void *d_ws,
                                size_t ws_bytes, int64_t max_entries, fdgs_frame_stats *host_stats,
                                void *stream);

/* CUDA-graph form of fdgs_render (the same kernels and results): the frame's
 * 21 front-end launches are captured once per (workspace, layout) and
 * replayed with one graph launch per frame; only the arguments that change
 * between frames are updated (scene, masks, t, camera, stage events).
 * Front-end nodes carry the device's greatest stream priority (cf. P:478:
 * the FPS of the whole render call).  The blend (the timed
 * k_blend_wi, no work counters) is launched directly after the graph, on the
 * same stream or (fdgs_render_graph_launch_split) on a blend stream.
 *   create: `scene` fixes the layout (max(n, n_capacity)); d_ws / ws_bytes /
 *           max_entries / width / height as for fdgs_render; *out (HOST)
 *           receives an opaque handle.  Synchronous (captures, instantiates).
 *   launch: a scene of the same layout n, camera of the same size; otherwise
 *           as fdgs_render (ASYNC on `stream`; frame status in the workspace
 *           counters).  The handle may not be launched concurrently from two
 *           host threads.
 *   destroy: frees the handle (NULL is a no-op).
 * Errors: INVALID_ARG (NULL, layout / size mismatch, bad camera),
 * WORKSPACE_TOO_SMALL, UNSUPPORTED, CUDA. */
typedef struct fdgs_render_graph fdgs_render_graph;
fdgs_status fdgs_render_graph_create(const fdgs_scene *scene, int32_t width, int32_t height, void *d_ws,
                                     size_t ws_bytes, int64_t max_entries, fdgs_render_graph **out);
fdgs_status fdgs_render_graph_launch(fdgs_render_graph *graph, const fdgs_scene *scene, const uint32_t *d_mask_l,
                                     const uint32_t *d_mask_r, const fdgs_camera *cam, float t, float *d_out_rgb,
                                     float *d_out_T, void *stream);
/* As fdgs_render_graph_launch, with the blend on `blend_stream` ordered after
 * the front end by `split_event` (a HOST cudaEvent_t the caller owns), as
 * fdgs_render_split does: the front-end graph on `stream`, the blend launched
 * directly on the (lower-priority) blend stream.  ASYNC. */
fdgs_status fdgs_render_graph_launch_split(fdgs_render_graph *graph, const fdgs_scene *scene,
                                           const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                                           const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T,
                                           void *stream, void *blend_stream, void *split_event);
/* As fdgs_render_graph_launch_split (blend_stream / split_event both NULL =
 * the blend on `stream`), with optional stage events: stage_events NULL or 5
 * caller-created cudaEvent_t (HOST handles, timing enabled) recorded as in
 * fdgs_render_timed -- events 0-2 by event-record nodes inside the graph
 * (re-pointed at this frame's events), 3-4 around the blend.  ASYNC. */
fdgs_status fdgs_render_graph_launch_timed(fdgs_render_graph *graph, const fdgs_scene *scene,
                                           const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                                           const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T,
                                           void *stream, void *blend_stream, void *split_event,
                                           void *const *stage_events);
fdgs_status fdgs_render_graph_destroy(fdgs_render_graph *graph);

/* Batched submission of frames over a pipeline of render workspaces (the
 * host side of the render path).  A pipeline has
 * `depth` slots, each a render workspace (zero-filled once, as for
 * fdgs_render) with a front-end stream and a blend stream (cudaStream_t as
 * void*; blend_stream NULL = the blend on the front stream); streams should
 * have the front end at a higher priority than the blend.  Frame k of a batch
 * renders in slot k mod depth (fdgs_render_split); a slot's next frame is
 * ordered after its previous blend.  The handle owns n_threads host threads
 * that issue the batch's launches in parallel (one group of slots per
 * thread; 1 = the caller's thread, frames in order), plus its own CUDA
 * events.  Several threads cut the host time per frame but interleave the
 * frames' launches, which costs device throughput with 12 streams (measured;
 * DESIGN.md "Host submission"): 1 is the default of the Python binding.
 *   fdgs_frame_job: the frame (scene and camera BY VALUE, masks, t, outputs
 *   as for fdgs_render; d_stats nullable = the timed blend, else the counting
 *   blend); h_out_rgb (nullable, pinned HOST float[3][H][W]): copied D2H on
 *   copy stream k mod n_copy after the blend; d_status (nullable, DEVICE 16
 *   bytes): the frame's {n_act, n_vis, n_entries, status} after the blend;
 *   done_event (nullable cudaEvent_t): recorded once the frame is complete.
 *   fdgs_pipeline_slot.graph (nullable): a fdgs_render_graph created on the
 *   slot's workspace; the slot's timed frames (d_stats NULL) then launch the
 *   front end as that graph (fdgs_render_graph_launch_timed: one launch per
 *   frame instead of ~21), frames with d_stats as stream launches.  The
 *   caller keeps the graph alive while the pipeline uses it.
 *   fdgs_pipeline_render: ASYNC on `stream`: every slot and copy stream first
 *   waits for `stream`'s work, and `stream` waits for every frame and copy of
 *   the batch; stage_events (nullable): 5 caller-created events per job, as
 *   fdgs_render_timed.  Returns when every launch is issued.  One batch at a
 *   time per handle.
 * Errors: INVALID_ARG, those of fdgs_render_split / fdgs_render_graph_launch_timed, CUDA. */
typedef struct {
    void *d_ws;
    size_t ws_bytes;
    int64_t max_entries;
    void *front_stream, *blend_stream;
    fdgs_render_graph *graph;
} fdgs_pipeline_slot;
typedef struct {
    fdgs_scene scene;
    const uint32_t *d_mask_l, *d_mask_r;
    fdgs_camera cam;
    float t;
    float *d_out_rgb, *d_out_T;
    fdgs_frame_stats *d_stats;
    float *h_out_rgb;
    void *d_status;
    void *done_event;
} fdgs_frame_job;
typedef struct fdgs_pipeline fdgs_pipeline;
fdgs_status fdgs_pipeline_create(const fdgs_pipeline_slot *slots, int32_t depth, void *const *copy_streams,
                                 int32_t n_copy, int32_t n_threads, fdgs_pipeline **out);
fdgs_status fdgs_pipeline_render(fdgs_pipeline *pipeline, const fdgs_frame_job *jobs, int32_t n_jobs, void *stream,
                                 void *const *stage_events);
fdgs_status fdgs_pipeline_destroy(fdgs_pipeline *pipeline);

/* Device views into a render workspace after fdgs_render (tests/debug only).
 * Records are indexed by the SLOT of a Gaussian that passed the mask and the
 * temporal cull (survivor order = ascending Gaussian index); only the slots of
 * visible Gaussians hold data, and vis uint32[n_vis] lists them ascending:
 *   rec0 float4 {u, v, A', B'}, rec1 float4 {C', Q2, aabb_x, aabb_y}
 *   (aabb_x = px0 | px1 << 16 as int bits, aabb_y likewise with bit 31 set
 *   when the per-pixel AABB test is provably redundant for the record),
 *   rec2 float4 {r, g, b, gid bits},
 *   depth uint32 (fp32 bits of camera z), order uint32[n_vis] (slots in
 *   canonical (depth, index) order), tile_start uint32[n_tiles + 1],
 *   entries uint32[E] (slots, per tile in canonical order). */
typedef struct {
    const void *rec0, *rec1, *rec2;
    const uint32_t *depth;
    const uint32_t *vis;
    const uint32_t *order;
    const uint32_t *tile_start;
    const uint32_t *entries;
    const uint32_t *counters; /* [0]=n_act [1]=n_vis [2]=E [3]=status */
    int32_t n_tiles;
} fdgs_debug_views;
fdgs_status fdgs_render_debug_views(void *d_ws, size_t ws_bytes, int32_t n, int32_t width, int32_t height,
                                    int64_t max_entries, fdgs_debug_views *out);

/* Tests/debug: the timed blend's record-to-strip culling decisions for the
 * frame last rendered in the workspace (same layout arguments as
 * fdgs_render_debug_views): bit w of d_out[k] (DEVICE uint8[E]) is set iff
 * entry k's record is staged for warp strip w (pixel rows 4w..4w+3 of its
 * tile) -- the device function k_blend_wi uses, replayed.  ASYNC. */
fdgs_status fdgs_debug_strip_reach(void *d_ws, size_t ws_bytes, int32_t n, int32_t width, int32_t height,
                                   int64_t max_entries, uint8_t *d_out, void *stream);

/* Key-frame visibility mask (Sec. 4.2.2): bit i of d_out_mask is set
 * iff Gaussian i is visible at t_key from at least one of the n_cams HOST
 * cameras, "visible" = temporal & support & near & cover culls of the render
 * decision path (reading R3), so the stored mask is the union over views
 * {U_j m_{i,j}}.  ASYNC.  d_out_mask: DEVICE uint32[ceil(n/32)]. */
size_t fdgs_keyframe_workspace_bytes(int32_t n_cams);
fdgs_status fdgs_keyframe_mask(const fdgs_scene *scene, const fdgs_camera *cams, int32_t n_cams, float t_key,
                               uint32_t *d_out_mask, void *d_ws, size_t ws_bytes, void *stream);

/* Key-frame mask read literally: m_{i,j} = {i : the
 * blending weights alpha_i prod_{j<i}(1 - alpha_j) of Gaussian i over all
 * pixels of the UNMASKED view-j render at t_key (Eq. 2) sum to more than
 * `threshold`}; bit i of d_out_mask = OR over the n_cams views (
 * threshold 0 = any blended pixel).  Weights are summed in 2^-24 fixed point
 * (as fdgs_stv_score); the test is sum_fixed > floor(threshold * 2^24).
 * Every blended weight is >= (1/255) * 1e-4 > 2^-24, so at threshold 0 a bit
 * is set iff the Gaussian is blended at least once.  Unlike
 * fdgs_keyframe_mask (reading R3) an occluded Gaussian stays clear.
 * cams HOST views (any sizes); d_out_mask DEVICE uint32[ceil(n/32)];
 * workspace of fdgs_keyframe_mask_contrib_workspace_bytes (256-aligned);
 * max_entries: tile-entry capacity of each view's render; h_max_entries HOST
 * (nullable) receives the largest per-view entry count.  SYNCHRONOUS.
 * Errors: INVALID_ARG (NULL, bad camera, n_cams < 1, threshold < 0 or not
 * finite, non-finite t_key), WORKSPACE_TOO_SMALL, UNSUPPORTED, OVERFLOW
 * (retry with *h_max_entries; mask undefined), CUDA. */
size_t fdgs_keyframe_mask_contrib_workspace_bytes(int32_t n, const fdgs_camera *cams, int32_t n_cams,
                                                  int64_t max_entries);
fdgs_status fdgs_keyframe_mask_contrib(const fdgs_scene *scene, const fdgs_camera *cams, int32_t n_cams,
                                       float t_key, double threshold, int64_t max_entries, uint32_t *d_out_mask,
                                       void *d_ws, size_t ws_bytes, uint32_t *h_max_entries, void *stream);

/* Compacted working set of a key-frame window (Sec. 4.2.2: "perform
 * rasterization while only considering the Gaussians marked by mask"): the
 * Gaussians of d_mask_l | d_mask_r (d_mask_r nullable) in ascending index
 * order, copied into caller-owned DEVICE arrays of capacity scene->n:
 *   d_params float[n][16] (mean, scale, rot_l, rot_r interleaved: use
 *   param_stride 4), d_opacity float[n], d_L float[n], d_sh float[n][48]
 *   (dense SH; NULL for a VQ scene), d_sh_index uint16[n] (VQ scene; NULL
 *   otherwise; the codebook is shared), d_gid uint32[n] (original indices).
 * *d_count (DEVICE uint32) receives the count m; the caller builds an
 * fdgs_scene of n = m over these arrays with gid = d_gid and renders it with
 * NULL masks: frames are bit-identical to masked renders of the full scene
 * (same decisions, same canonical order), while the per-frame culls read a
 * dense 64-byte record per active Gaussian instead of a scattered one.
 * Workspace: fdgs_scene_compact_workspace_bytes(n).  ASYNC.  Errors:
 * INVALID_ARG (NULL outputs, d_mask_l NULL, scene already compacted),
 * WORKSPACE_TOO_SMALL, CUDA. */
size_t fdgs_scene_compact_workspace_bytes(int32_t n);
fdgs_status fdgs_scene_compact(const fdgs_scene *scene, const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                               float *d_params, float *d_opacity, float *d_L, float *d_sh, uint16_t *d_sh_index,
                               uint32_t *d_gid, uint32_t *d_count, void *d_ws, size_t ws_bytes, void *stream);

/* d_out = d_a | d_b over ceil(n/32) words (P:285 active set).  ASYNC. */
fdgs_status fdgs_mask_or(const uint32_t *d_a, const uint32_t *d_b, int32_t n, uint32_t *d_out, void *stream);

/* Active-set compaction: ascending indices of the set bits
 * of (d_a | d_b) (d_b nullable) into d_out_idx (DEVICE int32[n]) and their
 * count into *d_count (DEVICE uint32).  Warp ballot + block scan + decoupled
 * look-back.  ASYNC. */
size_t fdgs_mask_compact_workspace_bytes(int32_t n);
fdgs_status fdgs_mask_compact(const uint32_t *d_a, const uint32_t *d_b, int32_t n, int32_t *d_out_idx,
                              uint32_t *d_count, void *d_ws, size_t ws_bytes, void *stream);

/* Spatial-temporal variation score (Sec. 4.2.1), the global
 * pruning criterion:
 *   S^S_i(t)  = sum over the n_cams views and all their pixels of the blending
 *               weight alpha_i prod_{j<i}(1 - alpha_j) of Gaussian i in the
 *               UNMASKED render at t (the weights of fdgs_render's
 *               composite, summed in 2^-24 fixed point: deterministic, error
 *               <= 2^-25 per (pixel, Gaussian) beyond the fp32 weight itself)
 *   S^TV_i(t) = 1 / (0.5 tanh|p2_i(t)| + 0.5),
 *               p2_i(t) = ((t-mu_t)^2/Sigma_t^2 - 1/Sigma_t) p_i(t)
 *   gamma_i   = min(V_i / V_p, 1), V_i = s_x s_y s_z s_t (fp32, left to right),
 *               V_p = the nearest-rank volume_percentile of V over the scene,
 *               i.e. the element of rank ceil(p n) - 1 (0-based) of sorted V
 *               (LightGaussian normalisation; reading R20)
 *   combine_mode 0: S_i = sum_t S^TV_i(t) gamma_i S^S_i(t)  (time-aligned, R20)
 *   combine_mode 1: S_i = gamma_i (sum_t S^TV_i(t)) (sum_t S^S_i(t))  (the
 *               literal product of the two sums of P:264-272)
 *   variant (score ablations of P:636-669; the per-t factors T(t), S(t) that
 *   the combine folds): 0 full T = S^TV gamma, S = S^S; 1 S^S only T = 1;
 *   2 S^T only S = 1; 3 S^TV from p1_i(t) = -((t-mu_t)/Sigma_t) p_i(t);
 *   4 T = Sigma_t gamma
 * Arguments: cams HOST array of n_cams views (any sizes); ts HOST float[n_ts];
 *   d_out_score DEVICE float[n]; d_out_spatial DEVICE float[n_ts][n] S^S_i(t)
 *   (nullable); d_out_gamma DEVICE float[n] (nullable); d_ws DEVICE workspace
 *   of fdgs_stv_workspace_bytes (256-aligned, no zero-fill needed);
 *   h_max_entries HOST (nullable) receives the largest per-view tile-entry
 *   count E, so a caller can size opts->max_entries.
 * SYNCHRONOUS (one stream sync at the end).  Errors: INVALID_ARG (NULL
 * pointers, bad camera, n_ts < 0, n_cams < 1, non-finite t, percentile outside
 * (0, 1], unknown combine_mode or variant), WORKSPACE_TOO_SMALL, UNSUPPORTED (tile grid >
 * FDGS_MAX_TILES), OVERFLOW (some view needed more than opts->max_entries tile
 * entries: outputs undefined; retry with *h_max_entries), CUDA. */
typedef struct {
    double volume_percentile;  /* gamma clip percentile, nearest rank (0.9)  */
    int32_t combine_mode;      /* 0 time-aligned (default), 1 product of sums */
    int32_t variant;           /* 0 full (default) .. 4, see above            */
    int64_t max_entries;       /* tile-entry capacity of each per-view render  */
} fdgs_stv_opts;
size_t fdgs_stv_workspace_bytes(int32_t n, const fdgs_camera *cams, int32_t n_cams, int64_t max_entries);
fdgs_status fdgs_stv_score(const fdgs_scene *scene, const fdgs_camera *cams, int32_t n_cams, const float *ts,
                           int32_t n_ts, const fdgs_stv_opts *opts, float *d_out_score, float *d_out_spatial,
                           float *d_out_gamma, void *d_ws, size_t ws_bytes, uint32_t *h_max_entries, void *stream);

/* Pruning selection (Sec. 4.2.1 "Pruning": "All 4D Gaussians are
 * ranked based on their spatial-temporal variation score S_i, and Gaussians
 * with lower scores are pruned"; SURVEY NEXT-f1 top-k select): bit i of
 * d_out_mask (DEVICE uint32[ceil(n/32)], LSB-first, bits >= n zero) is set iff
 * Gaussian i is among the `keep` highest d_score values (DEVICE float[n]);
 * equal scores are ranked by ascending index (reading R23), -0 equals +0.
 * Scores must not be NaN (the ranking is then undefined).  keep >= n keeps all,
 * keep == 0 none.  Radix select (4 x 8-bit passes over the scores) + ordered
 * tie emission; d_ws DEVICE workspace of fdgs_prune_workspace_bytes(n), no
 * zero-fill needed.  The pruned scene is fdgs_scene_compact(scene, mask).
 * ASYNC on `stream`.  Errors: INVALID_ARG (n < 0, keep < 0, NULL pointers),
 * WORKSPACE_TOO_SMALL, CUDA. */
size_t fdgs_prune_workspace_bytes(int32_t n);
fdgs_status fdgs_prune_mask(const float *d_score, int32_t n, int64_t keep, uint32_t *d_out_mask, void *d_ws,
                            size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FDGS_H */
