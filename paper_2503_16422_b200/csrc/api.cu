// api.cu -- the extern "C" boundary of libfdgs.so (include/fdgs.h).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "fdgs_internal.h"

namespace fdgs {
cudaError_t render_set_smem_attrs();

static thread_local char g_err[512] = "";

static fdgs_status fail(fdgs_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return s;
}

fdgs_status set_error(fdgs_status s, const char *msg) { return fail(s, "%s", msg); }

static fdgs_status cuda_fail(cudaError_t e, const char *where) {
    return fail(FDGS_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static int sm_count() {
    // the SM count of the current device, queried once per process (thread-safe static init)
    static const int cached = [] {
        int dev = 0, c = 148;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && c > 0)
            return c;
        return 148;
    }();
    return cached;
}

RenderLayout render_layout(int32_t n, int32_t width, int32_t height, int64_t max_entries) {
    RenderLayout L{};
    L.n = n;
    L.width = width;
    L.height = height;
    L.tiles_x = (width + FDGS_TILE - 1) / FDGS_TILE;
    L.tiles_y = (height + FDGS_TILE - 1) / FDGS_TILE;
    L.n_tiles = L.tiles_x * L.tiles_y;
    L.n_parts = (n + 2 * kPreBlock - 1) / (2 * kPreBlock);  // k_slice partitions (2 survivors per thread)
    L.cull_parts = (n + 4 * kPreBlock - 1) / (4 * kPreBlock);  // k_cull partitions (4 Gaussians per thread)
#ifndef FDGS_SLICE_GRID
#define FDGS_SLICE_GRID 2
#endif
    // grid-stride k_slice / k_vis_emit: FDGS_SLICE_GRID blocks per SM (compile-time)
    L.slice_grid = std::max(1, std::min(L.n_parts, FDGS_SLICE_GRID * sm_count()));
    L.p_sort = sm_count();
    L.sort_parts = std::max(1, (n + kDepthTile - 1) / kDepthTile);
    L.tile_parts = (int32_t)std::max<int64_t>(1, (max_entries + kTileTile - 1) / kTileTile);
    L.max_entries = max_entries;
    const size_t nn = (size_t)std::max(n, 1);
    const size_t cap = (size_t)std::max<int64_t>(max_entries, 1);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align256(off + bytes);
        return o;
    };
    // persistent, at a FIXED offset whatever the layout: the look-back epoch.  It
    // only ever increases, so epoch-tagged status words left by frames of any
    // other layout (another n, image size or capacity) can never look current
    L.epoch = take(sizeof(uint32_t));
    // cleared per frame
    L.counters = take(sizeof(Counters));
    L.sort_gbase = take(sizeof(uint32_t) * 4 * 256);
    L.tile_cnt = take(sizeof(uint32_t) * (size_t)L.n_tiles);  // entries per tile (k_row_count totals)
    L.row_diff = take(sizeof(int) * ((size_t)L.tiles_y + 1));
    L.bin_cnt = take(sizeof(uint32_t) * ((nn + 255) / 256));  // row items per k_bin_count partition
    L.zero_end = off;
    // persistent (zero-filled once)
    L.sort_status = take(sizeof(uint64_t) * 4 * 256 * (size_t)L.sort_parts);
    L.tile_status = take(sizeof(uint64_t) * 2 * 256 * (size_t)L.tile_parts);
    // per-frame scratch, fully written before read
    L.surv = take(4 * nn);
    L.surv_bits = take(4 * ((nn + 31) / 32 + 32));                     // survivor bits (k_cull)
    L.cull_cnt = take(4 * (size_t)std::max(L.cull_parts, 1));          // survivors per k_cull partition
    L.vis = take(4 * nn);                                               // visible survivor slots, ascending
    L.vis_bits = take(4 * ((nn + 31) / 32 + 32));                      // visibility bits per survivor slot
    L.vis_cnt = take(4 * (size_t)std::max(L.n_parts, 1));              // visible per k_slice partition
    L.rec0 = take(16 * nn);
    L.rec1 = take(16 * nn);
    L.rec2 = take(16 * nn);
    L.depth = take(4 * nn);
    L.rect = take(8 * nn);
    L.rect_sorted = take(8 * nn);
    L.keys0 = take(4 * nn);
    L.keys1 = take(4 * nn);
    L.vals0 = take(4 * nn);
    L.vals1 = take(4 * nn);
    L.tile_gbase = take(sizeof(uint32_t) * 512);
    L.tile_start = take(sizeof(uint32_t) * ((size_t)L.n_tiles + 1));
    L.row_start = take(sizeof(uint32_t) * ((size_t)L.tiles_y + 1));
    L.row_hist = take(sizeof(uint32_t) * (size_t)L.tiles_y * kRowSeg * L.tiles_x);  // [tiles_y][kRowSeg][tiles_x]
    L.band_consts = take(sizeof(BandConsts) * nn);          // tile-cover constants per Gaussian
    L.item_pack = take(4 * cap);                            // (ty, txa, txb) per row item
    L.item_v = take(4 * cap);                               // visible slot per row item
    L.ekey0 = take(4 * cap);
    L.ekey1 = take(4 * cap);
    L.eval0 = take(4 * cap);
    L.eval1 = take(4 * cap);
    L.entries = take(4 * cap);
    L.total = off;
    return L;
}

bool make_camdev(const fdgs_camera &c, CamDev &o, const char **why) {
    if (c.width < 1 || c.height < 1 || c.width > 8192 || c.height > 8192) { *why = "image size outside [1,8192]"; return false; }
    if (!(c.fx > 0.f) || !(c.fy > 0.f)) { *why = "fx, fy must be > 0"; return false; }
    if (!(c.z_near > 0.f)) { *why = "z_near must be > 0"; return false; }
    for (int k = 0; k < 9; ++k)
        if (!std::isfinite(c.R[k])) { *why = "non-finite R"; return false; }
    for (int k = 0; k < 3; ++k)
        if (!std::isfinite(c.T[k]) || !std::isfinite(c.bg[k])) { *why = "non-finite T/bg"; return false; }
    double worst = 0.0;
    for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += (double)c.R[3 * r + k] * (double)c.R[3 * s + k];
            worst = std::max(worst, std::fabs(acc - (r == s ? 1.0 : 0.0)));
        }
    if (worst > 1e-5) { *why = "R is not a rotation (|R R^T - I| > 1e-5)"; return false; }
    for (int k = 0; k < 9; ++k) o.R[k] = (double)c.R[k];
    for (int k = 0; k < 3; ++k) o.T[k] = (double)c.T[k];
    o.fx = c.fx;
    o.fy = c.fy;
    o.cx = c.cx;
    o.cy = c.cy;
    // pinned: 1.3 * (W / (2 fx)) in binary64 (DESIGN.md decision path)
    volatile double two_fx = 2.0 * o.fx, two_fy = 2.0 * o.fy;
    volatile double tx = (double)c.width / two_fx, ty = (double)c.height / two_fy;
    o.limx = kJClamp * tx;
    o.limy = kJClamp * ty;
    o.z_near = (double)c.z_near;
    for (int k = 0; k < 3; ++k) {
        // camera centre C = -R^T T (value path only: SH view direction)
        const double ck = -((double)c.R[k] * c.T[0] + (double)c.R[3 + k] * c.T[1] + (double)c.R[6 + k] * c.T[2]);
        o.campos[k] = (float)ck;
        o.bg[k] = c.bg[k];
    }
    o.width = c.width;
    o.height = c.height;
    return true;
}

SceneDev make_scenedev(const fdgs_scene &s) {
    SceneDev d;
    d.n = s.n;
    d.stride = s.param_stride > 0 ? s.param_stride : 1;
    d.mean = reinterpret_cast<const float4 *>(s.mean);
    d.scale = reinterpret_cast<const float4 *>(s.scale);
    d.rot_l = reinterpret_cast<const float4 *>(s.rot_l);
    d.rot_r = reinterpret_cast<const float4 *>(s.rot_r);
    d.opacity = s.opacity;
    d.L = s.log255_opacity;
    d.sh = reinterpret_cast<const float4 *>(s.sh);
    d.sh_index = s.sh_index;
    d.sh_k = s.sh_index ? s.sh_codebook_size : 0;
    d.gid = s.gid;
    d.d_n = s.d_n;
    return d;
}

// Gaussians the render workspace layout is computed for (include/fdgs.h n_capacity)
static int32_t layout_n(const fdgs_scene &s) { return std::max(s.n, s.n_capacity); }

static fdgs_status check_scene(const fdgs_scene *s) {
    if (s == nullptr) return fail(FDGS_ERR_INVALID_ARG, "scene is NULL");
    if (s->d_n != nullptr && s->gid == nullptr)
        return fail(FDGS_ERR_INVALID_ARG, "a device count (d_n) is only allowed for a compacted working set (gid)");
    if (s->n < 0) return fail(FDGS_ERR_INVALID_ARG, "scene->n < 0");
    if (s->n == 0) return FDGS_OK;
    const void *p[] = {s->mean, s->scale, s->rot_l, s->rot_r, s->opacity, s->log255_opacity, s->sh};
    for (const void *q : p)
        if (q == nullptr) return fail(FDGS_ERR_INVALID_ARG, "scene array is NULL");
    const void *a16[] = {s->mean, s->scale, s->rot_l, s->rot_r, s->sh};
    for (const void *q : a16)
        if ((uintptr_t)q % 16 != 0) return fail(FDGS_ERR_INVALID_ARG, "scene float4 arrays must be 16-byte aligned");
    if (s->param_stride < 0 || s->param_stride > 64) return fail(FDGS_ERR_INVALID_ARG, "param_stride must lie in [0, 64]");
    if (s->n_capacity < 0) return fail(FDGS_ERR_INVALID_ARG, "n_capacity < 0");
    if (s->sh_index != nullptr && (s->sh_codebook_size < 1 || s->sh_codebook_size > 65536))
        return fail(FDGS_ERR_INVALID_ARG, "sh_codebook_size must lie in [1, 65536] with sh_index");
    return FDGS_OK;
}

static std::once_flag g_attr_once;
static cudaError_t g_attr_err = cudaSuccess;

}  // namespace fdgs

using namespace fdgs;

extern "C" {

const char *fdgs_status_string(fdgs_status s) {
    switch (s) {
        case FDGS_OK: return "ok";
        case FDGS_ERR_INVALID_ARG: return "invalid argument";
        case FDGS_ERR_INVALID_SCENE: return "invalid scene";
        case FDGS_ERR_WORKSPACE_TOO_SMALL: return "workspace too small";
        case FDGS_ERR_OVERFLOW: return "tile-entry capacity exceeded";
        case FDGS_ERR_CUDA: return "CUDA error";
        case FDGS_ERR_UNSUPPORTED: return "unsupported";
    }
    return "unknown status";
}

const char *fdgs_last_error(void) { return g_err; }
int32_t fdgs_abi_version(void) { return FDGS_ABI_VERSION; }

size_t fdgs_scene_validate_workspace_bytes(void) { return 256; }

fdgs_status fdgs_scene_validate(const fdgs_scene *scene, int64_t *first_bad, void *d_ws, size_t ws_bytes,
                                void *stream) {
    if (first_bad) *first_bad = -1;
    fdgs_status s = check_scene(scene);
    if (s != FDGS_OK) return s;
    if (d_ws == nullptr || ws_bytes < 256) return fail(FDGS_ERR_WORKSPACE_TOO_SMALL, "validate needs 256 bytes");
    cudaStream_t st = (cudaStream_t)stream;
    auto *d_bad = reinterpret_cast<unsigned long long *>(d_ws);
    cudaError_t e = cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = launch_validate(make_scenedev(*scene), d_bad, st);
    unsigned long long h = ~0ull;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d_bad, sizeof h, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "fdgs_scene_validate");
    if (h != ~0ull) {
        if (first_bad) *first_bad = (int64_t)h;
        return fail(FDGS_ERR_INVALID_SCENE, "Gaussian %llu violates the scene invariants", h);
    }
    return FDGS_OK;
}

fdgs_status fdgs_log255_opacity(const float *d_opacity, int32_t n, float *d_out, void *stream) {
    if (n < 0 || (n > 0 && (d_opacity == nullptr || d_out == nullptr))) return fail(FDGS_ERR_INVALID_ARG, "bad args");
    cudaError_t e = launch_log255(d_opacity, n, d_out, (cudaStream_t)stream);
    return e == cudaSuccess ? FDGS_OK : cuda_fail(e, "fdgs_log255_opacity");
}

size_t fdgs_render_workspace_bytes(int32_t n, int32_t width, int32_t height, int64_t max_entries) {
    if (n < 0 || width < 1 || height < 1 || max_entries < 0) return 0;
    return render_layout(n, width, height, max_entries).total;
}

static fdgs_status render_impl(const fdgs_scene *scene, const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                               const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T, void *d_ws,
                               size_t ws_bytes, int64_t max_entries, fdgs_frame_stats *d_stats, void *stream,
                               void *const *stage_events, void *blend_stream, void *split_event) {
    fdgs_status s = check_scene(scene);
    if (s != FDGS_OK) return s;
    if (cam == nullptr || d_out_rgb == nullptr) return fail(FDGS_ERR_INVALID_ARG, "camera / output is NULL");
    if (!std::isfinite(t)) return fail(FDGS_ERR_INVALID_ARG, "t is not finite");
    if (max_entries < 0 || max_entries > 0xffffffffll) return fail(FDGS_ERR_INVALID_ARG, "max_entries out of range");
    CamDev cd;
    const char *why = nullptr;
    if (!make_camdev(*cam, cd, &why)) return fail(FDGS_ERR_INVALID_ARG, "camera: %s", why);
    const RenderLayout L = render_layout(layout_n(*scene), cam->width, cam->height, max_entries);
    if (L.n_tiles > FDGS_MAX_TILES) return fail(FDGS_ERR_UNSUPPORTED, "tile grid %d > %d", L.n_tiles, FDGS_MAX_TILES);
    if (d_ws == nullptr || ws_bytes < L.total || (uintptr_t)d_ws % 256 != 0)
        return fail(FDGS_ERR_WORKSPACE_TOO_SMALL, "workspace needs %zu bytes (256-aligned), got %zu", L.total, ws_bytes);
    if (d_mask_l == nullptr && d_mask_r != nullptr) d_mask_l = d_mask_r, d_mask_r = nullptr;
    std::call_once(g_attr_once, [] { g_attr_err = render_set_smem_attrs(); });
    if (g_attr_err != cudaSuccess) return cuda_fail(g_attr_err, "cudaFuncSetAttribute");
    cudaError_t e = launch_render(make_scenedev(*scene), d_mask_l, d_mask_r, cd, t, d_out_rgb, d_out_T,
                                  reinterpret_cast<char *>(d_ws), L, d_stats, (cudaStream_t)stream,
                                  reinterpret_cast<cudaEvent_t const *>(stage_events), (cudaStream_t)blend_stream,
                                  (cudaEvent_t)split_event);
    return e == cudaSuccess ? FDGS_OK : cuda_fail(e, "fdgs_render");
}

fdgs_status fdgs_render_timed(const fdgs_scene *scene, const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                              const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T, void *d_ws,
                              size_t ws_bytes, int64_t max_entries, fdgs_frame_stats *d_stats, void *stream,
                              void *const *stage_events) {
    return render_impl(scene, d_mask_l, d_mask_r, cam, t, d_out_rgb, d_out_T, d_ws, ws_bytes, max_entries, d_stats,
                       stream, stage_events, nullptr, nullptr);
}

fdgs_status fdgs_render_split(const fdgs_scene *scene, const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                              const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T, void *d_ws,
                              size_t ws_bytes, int64_t max_entries, fdgs_frame_stats *d_stats, void *stream,
                              void *blend_stream, void *split_event, void *const *stage_events) {
    if (blend_stream == nullptr || split_event == nullptr)
        return fail(FDGS_ERR_INVALID_ARG, "fdgs_render_split needs a blend stream and an event");
    return render_impl(scene, d_mask_l, d_mask_r, cam, t, d_out_rgb, d_out_T, d_ws, ws_bytes, max_entries, d_stats,
                       stream, stage_events, blend_stream, split_event);
}

fdgs_status fdgs_render(const fdgs_scene *scene, const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                        const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T, void *d_ws,
                        size_t ws_bytes, int64_t max_entries, fdgs_frame_stats *d_stats, void *stream) {
    return fdgs_render_timed(scene, d_mask_l, d_mask_r, cam, t, d_out_rgb, d_out_T, d_ws, ws_bytes, max_entries,
                             d_stats, stream, nullptr);
}

fdgs_status fdgs_render_checked(const fdgs_scene *scene, const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                                const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T, void *d_ws,
                                size_t ws_bytes, int64_t max_entries, fdgs_frame_stats *host_stats,
                                void *stream) {
    fdgs_status s = fdgs_render(scene, d_mask_l, d_mask_r, cam, t, d_out_rgb, d_out_T, d_ws, ws_bytes, max_entries,
                                nullptr, stream);
    if (s != FDGS_OK) return s;
    const RenderLayout L = render_layout(layout_n(*scene), cam->width, cam->height, max_entries);
    Counters c;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(&c, reinterpret_cast<char *>(d_ws) + L.counters, sizeof c, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "fdgs_render_checked");
    const uint32_t h[4] = {c.n_act, c.n_vis, c.n_entries, c.status};
    if (host_stats) {
        host_stats->n_act = h[0];
        host_stats->n_vis = h[1];
        host_stats->n_entries = h[2];
        host_stats->status = h[3];
        host_stats->n_evaluated = c.n_eval;
        host_stats->n_blended = c.n_blend;
    }
    if (h[3] != FDGS_OK)
        return fail((fdgs_status)h[3], "frame status %u: %u entries > capacity %lld", h[3], h[2], (long long)max_entries);
    return FDGS_OK;
}

struct fdgs_render_graph {
    fdgs::RenderGraphImpl *impl;
    int32_t layout_n, width, height;
    int64_t max_entries;
};

fdgs_status fdgs_render_graph_create(const fdgs_scene *scene, int32_t width, int32_t height, void *d_ws,
                                     size_t ws_bytes, int64_t max_entries, fdgs_render_graph **out) {
    if (out == nullptr) return fail(FDGS_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    fdgs_status s = check_scene(scene);
    if (s != FDGS_OK) return s;
    if (width < 1 || height < 1 || width > 8192 || height > 8192) return fail(FDGS_ERR_INVALID_ARG, "image size");
    if (max_entries < 0 || max_entries > 0xffffffffll) return fail(FDGS_ERR_INVALID_ARG, "max_entries out of range");
    const RenderLayout L = render_layout(layout_n(*scene), width, height, max_entries);
    if (L.n_tiles > FDGS_MAX_TILES) return fail(FDGS_ERR_UNSUPPORTED, "tile grid %d > %d", L.n_tiles, FDGS_MAX_TILES);
    if (d_ws == nullptr || ws_bytes < L.total || (uintptr_t)d_ws % 256 != 0)
        return fail(FDGS_ERR_WORKSPACE_TOO_SMALL, "workspace needs %zu bytes (256-aligned), got %zu", L.total, ws_bytes);
    std::call_once(g_attr_once, [] { g_attr_err = render_set_smem_attrs(); });
    if (g_attr_err != cudaSuccess) return cuda_fail(g_attr_err, "cudaFuncSetAttribute");
    CamDev cd{};  // placeholder camera: the arguments are replaced at every launch
    cd.width = width;
    cd.height = height;
    RenderGraphImpl *impl = render_graph_new();
    if (impl == nullptr) return fail(FDGS_ERR_CUDA, "out of host memory");
    cudaError_t e = render_graph_build(*impl, make_scenedev(*scene), cd, reinterpret_cast<char *>(d_ws), L);
    if (e != cudaSuccess) {
        render_graph_delete(impl);
        return cuda_fail(e, "fdgs_render_graph_create");
    }
    *out = new (std::nothrow) fdgs_render_graph{impl, layout_n(*scene), width, height, max_entries};
    if (*out == nullptr) {
        render_graph_delete(impl);
        return fail(FDGS_ERR_CUDA, "out of host memory");
    }
    return FDGS_OK;
}

fdgs_status fdgs_render_graph_launch(fdgs_render_graph *graph, const fdgs_scene *scene, const uint32_t *d_mask_l,
                                     const uint32_t *d_mask_r, const fdgs_camera *cam, float t, float *d_out_rgb,
                                     float *d_out_T, void *stream) {
    return fdgs_render_graph_launch_split(graph, scene, d_mask_l, d_mask_r, cam, t, d_out_rgb, d_out_T, stream,
                                          nullptr, nullptr);
}

fdgs_status fdgs_render_graph_launch_split(fdgs_render_graph *graph, const fdgs_scene *scene,
                                           const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                                           const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T,
                                           void *stream, void *blend_stream, void *split_event) {
    return fdgs_render_graph_launch_timed(graph, scene, d_mask_l, d_mask_r, cam, t, d_out_rgb, d_out_T, stream,
                                          blend_stream, split_event, nullptr);
}

fdgs_status fdgs_render_graph_launch_timed(fdgs_render_graph *graph, const fdgs_scene *scene,
                                           const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                                           const fdgs_camera *cam, float t, float *d_out_rgb, float *d_out_T,
                                           void *stream, void *blend_stream, void *split_event,
                                           void *const *stage_events) {
    if ((blend_stream == nullptr) != (split_event == nullptr))
        return fail(FDGS_ERR_INVALID_ARG, "blend_stream and split_event go together");
    if (graph == nullptr) return fail(FDGS_ERR_INVALID_ARG, "graph is NULL");
    fdgs_status s = check_scene(scene);
    if (s != FDGS_OK) return s;
    if (cam == nullptr || d_out_rgb == nullptr) return fail(FDGS_ERR_INVALID_ARG, "camera / output is NULL");
    if (!std::isfinite(t)) return fail(FDGS_ERR_INVALID_ARG, "t is not finite");
    if (layout_n(*scene) != graph->layout_n || cam->width != graph->width || cam->height != graph->height)
        return fail(FDGS_ERR_INVALID_ARG, "scene layout / image size differ from the graph's");
    CamDev cd;
    const char *why = nullptr;
    if (!make_camdev(*cam, cd, &why)) return fail(FDGS_ERR_INVALID_ARG, "camera: %s", why);
    if (d_mask_l == nullptr && d_mask_r != nullptr) d_mask_l = d_mask_r, d_mask_r = nullptr;
    cudaError_t e = render_graph_launch(*graph->impl, make_scenedev(*scene), d_mask_l, d_mask_r, cd, t, d_out_rgb,
                                        d_out_T, (cudaStream_t)stream, (cudaStream_t)blend_stream,
                                        (cudaEvent_t)split_event, reinterpret_cast<cudaEvent_t const *>(stage_events));
    return e == cudaSuccess ? FDGS_OK : cuda_fail(e, "fdgs_render_graph_launch");
}

fdgs_status fdgs_render_graph_destroy(fdgs_render_graph *graph) {
    if (graph) {
        render_graph_delete(graph->impl);
        delete graph;
    }
    return FDGS_OK;
}

fdgs_status fdgs_render_debug_views(void *d_ws, size_t ws_bytes, int32_t n, int32_t width, int32_t height,
                                    int64_t max_entries, fdgs_debug_views *out) {
    if (d_ws == nullptr || out == nullptr) return fail(FDGS_ERR_INVALID_ARG, "NULL");
    const RenderLayout L = render_layout(n, width, height, max_entries);
    if (ws_bytes < L.total) return fail(FDGS_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
    char *w = reinterpret_cast<char *>(d_ws);
    out->rec0 = w + L.rec0;
    out->rec1 = w + L.rec1;
    out->rec2 = w + L.rec2;
    out->depth = reinterpret_cast<const uint32_t *>(w + L.depth);
    out->vis = reinterpret_cast<const uint32_t *>(w + L.vis);
    out->order = reinterpret_cast<const uint32_t *>(w + L.vals1);
    out->tile_start = reinterpret_cast<const uint32_t *>(w + L.tile_start);
    out->entries = reinterpret_cast<const uint32_t *>(w + L.entries);
    out->counters = reinterpret_cast<const uint32_t *>(w + L.counters);
    out->n_tiles = L.n_tiles;
    return FDGS_OK;
}

fdgs_status fdgs_debug_strip_reach(void *d_ws, size_t ws_bytes, int32_t n, int32_t width, int32_t height,
                                   int64_t max_entries, uint8_t *d_out, void *stream) {
    if (d_ws == nullptr || d_out == nullptr || n < 0 || width < 1 || height < 1 || max_entries < 0)
        return fail(FDGS_ERR_INVALID_ARG, "bad args");
    const RenderLayout L = render_layout(n, width, height, max_entries);
    if (ws_bytes < L.total) return fail(FDGS_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
    cudaError_t e = launch_debug_strip_reach(reinterpret_cast<char *>(d_ws), L, d_out, (cudaStream_t)stream);
    return e == cudaSuccess ? FDGS_OK : cuda_fail(e, "fdgs_debug_strip_reach");
}

size_t fdgs_keyframe_workspace_bytes(int32_t n_cams) {
    return n_cams <= 0 ? 256 : align256(sizeof(CamDev) * (size_t)n_cams);
}

fdgs_status fdgs_keyframe_mask(const fdgs_scene *scene, const fdgs_camera *cams, int32_t n_cams, float t_key,
                               uint32_t *d_out_mask, void *d_ws, size_t ws_bytes, void *stream) {
    fdgs_status s = check_scene(scene);
    if (s != FDGS_OK) return s;
    if (cams == nullptr || n_cams <= 0 || n_cams > 1024 || d_out_mask == nullptr)
        return fail(FDGS_ERR_INVALID_ARG, "cameras / output");
    if (scene->gid != nullptr) return fail(FDGS_ERR_INVALID_ARG, "masks index the full scene, not a working set");
    if (!std::isfinite(t_key)) return fail(FDGS_ERR_INVALID_ARG, "t_key is not finite");
    if (d_ws == nullptr || ws_bytes < fdgs_keyframe_workspace_bytes(n_cams))
        return fail(FDGS_ERR_WORKSPACE_TOO_SMALL, "keyframe workspace");
    std::vector<CamDev> h(n_cams);
    for (int c = 0; c < n_cams; ++c) {
        const char *why = nullptr;
        if (!make_camdev(cams[c], h[c], &why)) return fail(FDGS_ERR_INVALID_ARG, "camera %d: %s", c, why);
    }
    cudaStream_t st = (cudaStream_t)stream;
    // pageable source: cudaMemcpyAsync returns once `h` has been staged
    cudaError_t e = cudaMemcpyAsync(d_ws, h.data(), sizeof(CamDev) * n_cams, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = launch_keyframe(make_scenedev(*scene), reinterpret_cast<CamDev *>(d_ws), n_cams, t_key,
                                              d_out_mask, st);
    return e == cudaSuccess ? FDGS_OK : cuda_fail(e, "fdgs_keyframe_mask");
}

size_t fdgs_keyframe_mask_contrib_workspace_bytes(int32_t n, const fdgs_camera *cams, int32_t n_cams,
                                                  int64_t max_entries) {
    return fdgs_stv_workspace_bytes(n, cams, n_cams, max_entries);
}

fdgs_status fdgs_keyframe_mask_contrib(const fdgs_scene *scene, const fdgs_camera *cams, int32_t n_cams,
                                       float t_key, double threshold, int64_t max_entries, uint32_t *d_out_mask,
                                       void *d_ws, size_t ws_bytes, uint32_t *h_max_entries, void *stream) {
    if (h_max_entries) *h_max_entries = 0;
    fdgs_status s = check_scene(scene);
    if (s != FDGS_OK) return s;
    if (cams == nullptr || n_cams < 1 || (scene->n > 0 && d_out_mask == nullptr))
        return fail(FDGS_ERR_INVALID_ARG, "cameras / output");
    if (scene->gid != nullptr) return fail(FDGS_ERR_INVALID_ARG, "masks index the full scene, not a working set");
    if (!std::isfinite(t_key)) return fail(FDGS_ERR_INVALID_ARG, "t_key is not finite");
    if (!(threshold >= 0.0) || !std::isfinite(threshold) || threshold > 1e11)
        return fail(FDGS_ERR_INVALID_ARG, "threshold must be finite, >= 0 and <= 1e11");
    if (max_entries < 0 || max_entries > 0xffffffffll) return fail(FDGS_ERR_INVALID_ARG, "max_entries");
    std::vector<CamDev> cd(n_cams);
    for (int c = 0; c < n_cams; ++c) {
        const char *why = nullptr;
        if (!make_camdev(cams[c], cd[c], &why)) return fail(FDGS_ERR_INVALID_ARG, "camera %d: %s", c, why);
        const RenderLayout L = render_layout(std::max(scene->n, 0), cams[c].width, cams[c].height, max_entries);
        if (L.n_tiles > FDGS_MAX_TILES) return fail(FDGS_ERR_UNSUPPORTED, "tile grid %d > %d", L.n_tiles, FDGS_MAX_TILES);
    }
    if (scene->n == 0) return FDGS_OK;
    const StvLayout SL = stv_layout(scene->n, cams, n_cams, max_entries);
    if (d_ws == nullptr || ws_bytes < SL.total || (uintptr_t)d_ws % 256 != 0)
        return fail(FDGS_ERR_WORKSPACE_TOO_SMALL, "workspace needs %zu bytes (256-aligned), got %zu", SL.total,
                    ws_bytes);
    std::call_once(g_attr_once, [] { g_attr_err = render_set_smem_attrs(); });
    if (g_attr_err != cudaSuccess) return cuda_fail(g_attr_err, "cudaFuncSetAttribute");
    const unsigned long long thr_fixed = (unsigned long long)std::floor(threshold * 16777216.0);
    cudaStream_t st = (cudaStream_t)stream;
    char *ws = reinterpret_cast<char *>(d_ws);
    cudaError_t e = launch_keyframe_contrib(make_scenedev(*scene), cd.data(), cams, n_cams, t_key, thr_fixed,
                                            max_entries, ws, SL, d_out_mask, st);
    uint32_t info[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(info, ws + SL.state, sizeof info, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "fdgs_keyframe_mask_contrib");
    if (h_max_entries) *h_max_entries = info[1];
    if (info[0] != FDGS_OK)
        return fail((fdgs_status)info[0], "a view needed %u tile entries > capacity %lld", info[1],
                    (long long)max_entries);
    return FDGS_OK;
}

size_t fdgs_scene_compact_workspace_bytes(int32_t n) {
    if (n < 0) return 0;
    return align256(sizeof(uint32_t) * (size_t)n) + fdgs_mask_compact_workspace_bytes(n);
}

fdgs_status fdgs_scene_compact(const fdgs_scene *scene, const uint32_t *d_mask_l, const uint32_t *d_mask_r,
                               float *d_params, float *d_opacity, float *d_L, float *d_sh, uint16_t *d_sh_index,
                               uint32_t *d_gid, uint32_t *d_count, void *d_ws, size_t ws_bytes, void *stream) {
    fdgs_status s = check_scene(scene);
    if (s != FDGS_OK) return s;
    if (scene->gid != nullptr) return fail(FDGS_ERR_INVALID_ARG, "the scene is already a compacted working set");
    if (d_count == nullptr || (scene->n > 0 && (d_mask_l == nullptr || d_params == nullptr || d_opacity == nullptr ||
                                                d_L == nullptr || d_gid == nullptr)))
        return fail(FDGS_ERR_INVALID_ARG, "NULL mask / output");
    if (scene->n > 0 && ((scene->sh_index == nullptr) != (d_sh_index == nullptr) ||
                         (scene->sh_index == nullptr && d_sh == nullptr)))
        return fail(FDGS_ERR_INVALID_ARG, "SH output must match the scene's storage (dense d_sh or VQ d_sh_index)");
    if ((uintptr_t)d_params % 16 != 0 || (d_sh && (uintptr_t)d_sh % 16 != 0))
        return fail(FDGS_ERR_INVALID_ARG, "d_params / d_sh must be 16-byte aligned");
    if (d_ws == nullptr || ws_bytes < fdgs_scene_compact_workspace_bytes(scene->n))
        return fail(FDGS_ERR_WORKSPACE_TOO_SMALL, "compact workspace");
    cudaError_t e = launch_scene_compact(make_scenedev(*scene), d_mask_l, d_mask_r, reinterpret_cast<float4 *>(d_params),
                                         d_opacity, d_L, reinterpret_cast<float4 *>(d_sh), d_sh_index, d_gid, d_count,
                                         reinterpret_cast<uint32_t *>(d_ws), (cudaStream_t)stream);
    return e == cudaSuccess ? FDGS_OK : cuda_fail(e, "fdgs_scene_compact");
}

fdgs_status fdgs_mask_or(const uint32_t *d_a, const uint32_t *d_b, int32_t n, uint32_t *d_out, void *stream) {
    if (n < 0 || (n > 0 && (d_a == nullptr || d_b == nullptr || d_out == nullptr)))
        return fail(FDGS_ERR_INVALID_ARG, "bad args");
    cudaError_t e = launch_mask_or(d_a, d_b, n, d_out, (cudaStream_t)stream);
    return e == cudaSuccess ? FDGS_OK : cuda_fail(e, "fdgs_mask_or");
}

size_t fdgs_mask_compact_workspace_bytes(int32_t n) {
    return align256(sizeof(uint32_t) * (32 + (size_t)(std::max(n, 0) + 255) / 256));
}

fdgs_status fdgs_mask_compact(const uint32_t *d_a, const uint32_t *d_b, int32_t n, int32_t *d_out_idx,
                              uint32_t *d_count, void *d_ws, size_t ws_bytes, void *stream) {
    if (n < 0 || (n > 0 && (d_a == nullptr || d_out_idx == nullptr)) || d_count == nullptr)
        return fail(FDGS_ERR_INVALID_ARG, "bad args");
    if (d_ws == nullptr || ws_bytes < fdgs_mask_compact_workspace_bytes(n))
        return fail(FDGS_ERR_WORKSPACE_TOO_SMALL, "compact workspace");
    cudaError_t e = launch_mask_compact(d_a, d_b, n, d_out_idx, d_count, reinterpret_cast<uint32_t *>(d_ws),
                                        (cudaStream_t)stream);
    return e == cudaSuccess ? FDGS_OK : cuda_fail(e, "fdgs_mask_compact");
}

size_t fdgs_prune_workspace_bytes(int32_t n) { return n < 0 ? 0 : prune_workspace_bytes(n); }

fdgs_status fdgs_prune_mask(const float *d_score, int32_t n, int64_t keep, uint32_t *d_out_mask, void *d_ws,
                            size_t ws_bytes, void *stream) {
    if (n < 0 || keep < 0 || (n > 0 && (d_score == nullptr || d_out_mask == nullptr)))
        return fail(FDGS_ERR_INVALID_ARG, "bad args");
    if (d_ws == nullptr || ws_bytes < prune_workspace_bytes(n))
        return fail(FDGS_ERR_WORKSPACE_TOO_SMALL, "prune workspace needs %zu bytes", prune_workspace_bytes(n));
    cudaError_t e = launch_prune_mask(d_score, n, keep, d_out_mask, reinterpret_cast<char *>(d_ws), (cudaStream_t)stream);
    return e == cudaSuccess ? FDGS_OK : cuda_fail(e, "fdgs_prune_mask");
}

size_t fdgs_stv_workspace_bytes(int32_t n, const fdgs_camera *cams, int32_t n_cams, int64_t max_entries) {
    if (n < 0 || cams == nullptr || n_cams < 1 || max_entries < 0) return 0;
    for (int c = 0; c < n_cams; ++c)
        if (cams[c].width < 1 || cams[c].height < 1) return 0;
    return stv_layout(n, cams, n_cams, max_entries).total;
}

fdgs_status fdgs_stv_score(const fdgs_scene *scene, const fdgs_camera *cams, int32_t n_cams, const float *ts,
                           int32_t n_ts, const fdgs_stv_opts *opts, float *d_out_score, float *d_out_spatial,
                           float *d_out_gamma, void *d_ws, size_t ws_bytes, uint32_t *h_max_entries, void *stream) {
    if (h_max_entries) *h_max_entries = 0;
    fdgs_status s = check_scene(scene);
    if (s != FDGS_OK) return s;
    if (opts == nullptr || cams == nullptr || n_cams < 1 || n_ts < 0 || (n_ts > 0 && ts == nullptr))
        return fail(FDGS_ERR_INVALID_ARG, "opts / cameras / timestamps");
    if (scene->gid != nullptr) return fail(FDGS_ERR_INVALID_ARG, "score the full scene, not a compacted working set");
    if (scene->n > 0 && d_out_score == nullptr) return fail(FDGS_ERR_INVALID_ARG, "d_out_score is NULL");
    if (!(opts->volume_percentile > 0.0 && opts->volume_percentile <= 1.0))
        return fail(FDGS_ERR_INVALID_ARG, "volume_percentile must lie in (0, 1]");
    if (opts->combine_mode != 0 && opts->combine_mode != 1) return fail(FDGS_ERR_INVALID_ARG, "combine_mode");
    if (opts->variant < 0 || opts->variant > 4) return fail(FDGS_ERR_INVALID_ARG, "variant must lie in [0, 4]");
    if (opts->max_entries < 0 || opts->max_entries > 0xffffffffll) return fail(FDGS_ERR_INVALID_ARG, "max_entries");
    for (int k = 0; k < n_ts; ++k)
        if (!std::isfinite(ts[k])) return fail(FDGS_ERR_INVALID_ARG, "ts[%d] is not finite", k);
    std::vector<CamDev> cd(n_cams);
    for (int c = 0; c < n_cams; ++c) {
        const char *why = nullptr;
        if (!make_camdev(cams[c], cd[c], &why)) return fail(FDGS_ERR_INVALID_ARG, "camera %d: %s", c, why);
        const RenderLayout L = render_layout(std::max(scene->n, 0), cams[c].width, cams[c].height, opts->max_entries);
        if (L.n_tiles > FDGS_MAX_TILES) return fail(FDGS_ERR_UNSUPPORTED, "tile grid %d > %d", L.n_tiles, FDGS_MAX_TILES);
    }
    const int n = scene->n;
    if (n == 0) return FDGS_OK;
    const StvLayout SL = stv_layout(n, cams, n_cams, opts->max_entries);
    if (d_ws == nullptr || ws_bytes < SL.total || (uintptr_t)d_ws % 256 != 0)
        return fail(FDGS_ERR_WORKSPACE_TOO_SMALL, "stv workspace needs %zu bytes (256-aligned), got %zu", SL.total,
                    ws_bytes);
    cudaStream_t st = (cudaStream_t)stream;
    if (n_ts == 0 && d_out_gamma == nullptr) {  // empty sums (gamma does not depend on t)
        cudaError_t e = cudaMemsetAsync(d_out_score, 0, sizeof(float) * (size_t)n, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        return e == cudaSuccess ? FDGS_OK : cuda_fail(e, "fdgs_stv_score");
    }
    std::call_once(g_attr_once, [] { g_attr_err = render_set_smem_attrs(); });
    if (g_attr_err != cudaSuccess) return cuda_fail(g_attr_err, "cudaFuncSetAttribute");
    // nearest rank, 0-based: ceil(p n) - 1 (as the oracle)
    long long rank = (long long)std::ceil(opts->volume_percentile * (double)n) - 1;
    rank = std::min<long long>(std::max<long long>(rank, 0), n - 1);
    char *ws = reinterpret_cast<char *>(d_ws);
    // camera constants go to the device by value (kernel arguments), so cd is host-only
    cudaError_t e = launch_stv(make_scenedev(*scene), cd.data(), cams, n_cams, ts, n_ts, (uint32_t)rank,
                               opts->combine_mode, opts->variant, opts->max_entries, ws, SL, d_out_score, d_out_spatial, d_out_gamma,
                               st);
    uint32_t info[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(info, ws + SL.state, sizeof info, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "fdgs_stv_score");
    if (h_max_entries) *h_max_entries = info[1];
    if (info[0] != FDGS_OK)
        return fail((fdgs_status)info[0], "a view needed %u tile entries > capacity %lld", info[1],
                    (long long)opts->max_entries);
    return FDGS_OK;
}

}  // extern "C"
