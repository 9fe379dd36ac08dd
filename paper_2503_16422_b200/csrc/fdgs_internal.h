// fdgs_internal.h -- host-side launchers shared by the .cu files of libfdgs.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/fdgs.h"
#include "fdgs_device.cuh"

namespace fdgs {

constexpr int kPreBlock = 256;         // Gaussians per preprocess partition
#ifndef FDGS_SORT_ITEMS
#define FDGS_SORT_ITEMS 4
#endif
constexpr int kDepthItems = FDGS_SORT_ITEMS;
constexpr int kDepthTile = 256 * kDepthItems;  // keys per depth-sort partition (256 threads x items)
constexpr int kTileSortItems = 4;      // row items per thread in the row-partition passes
constexpr int kTileTile = 256 * kTileSortItems;
#ifndef FDGS_ROWSEG
#define FDGS_ROWSEG 16
#endif
constexpr int kRowSeg = FDGS_ROWSEG;   // blocks per tile row in the row count / scatter
constexpr int kMaxTilesY = 512;        // 8192 px / 16
constexpr uint32_t kFlagA = 1u << 30;  // look-back: aggregate available
constexpr uint32_t kFlagP = 2u << 30;  // look-back: inclusive prefix available
constexpr uint32_t kValMask = (1u << 30) - 1;

// Counter block at the head of the render workspace (zeroed per frame).
struct Counters {
    uint32_t n_act, n_vis, n_entries, status;  // mirrors fdgs_frame_stats
    uint32_t part_ticket;
    uint32_t sort_ticket[5];  // [0] histogram kernel, [1 + pass] onesweep partitions
    uint32_t bin_ticket;
    uint32_t blend_ticket;
    uint32_t tile_ticket[2];
    uint32_t n_sort_entries;     // E when it fits the capacity, else 0
    uint32_t pad[1];
    unsigned long long n_eval;   // (pixel, Gaussian) pairs tested before termination
    unsigned long long n_blend;  // pairs composited
    uint32_t row_ticket;         // row-item scan partitions
    uint32_t n_items;            // (Gaussian, tile row) items
    uint32_t n_surv;             // Gaussians passing the mask and the temporal cull (k_cull)
    uint32_t cull_ticket;        // k_cull partitions
    uint32_t n_items_part;       // row items the row partition sorts: n_items if <= capacity, else 0
    uint32_t pad2[7];
};
static_assert(sizeof(Counters) == 128, "Counters layout");

struct SceneDev {
    int32_t n;
    int32_t stride;  // float4 elements between consecutive Gaussians of mean/scale/rot_l/rot_r
    const float4 *mean, *scale, *rot_l, *rot_r;
    __device__ __forceinline__ float4 ld_mean(int i) const { return __ldg(mean + (size_t)i * stride); }
    __device__ __forceinline__ float4 ld_scale(int i) const { return __ldg(scale + (size_t)i * stride); }
    __device__ __forceinline__ float4 ld_rot_l(int i) const { return __ldg(rot_l + (size_t)i * stride); }
    __device__ __forceinline__ float4 ld_rot_r(int i) const { return __ldg(rot_r + (size_t)i * stride); }
    const float *opacity, *L;
    const float4 *sh;  // [n][12] float4 = 48 floats, or the VQ codebook [K][12]
    const uint16_t *sh_index;  // VQ: codebook entry per Gaussian (nullable)
    int32_t sh_k;              // VQ codebook entries
    const uint32_t *gid;       // compacted working set: original index of Gaussian i (nullable)
    const uint32_t *d_n;       // device count (nullable): Gaussians [0, min(*d_n, n)) are the scene
    __device__ __forceinline__ uint32_t orig(int i) const { return gid ? __ldg(gid + i) : (uint32_t)i; }
};

// Workspace layout of fdgs_render (all offsets 256-byte aligned).  The
// region [counters, zero_end) is cleared per frame; the epoch word and the
// epoch-tagged look-back tables persist (the workspace must be zero-filled
// once before first use).
struct RenderLayout {
    int32_t n, width, height, tiles_x, tiles_y, n_tiles;
    int32_t n_parts;     // k_slice partitions (upper bound: every Gaussian survives)
    int32_t cull_parts;  // k_cull partitions
    int32_t slice_grid;  // persistent k_slice grid
    int32_t p_sort;      // SM count (grid of the histogram kernels)
    int32_t sort_parts;  // depth-sort partitions (upper bound from n)
    int32_t tile_parts;  // row-partition partitions (upper bound from max_entries)
    int64_t max_entries;
    size_t counters, sort_gbase, tile_cnt, row_diff, bin_cnt, zero_end;
    size_t epoch, sort_status, tile_status;
    size_t surv, surv_bits, cull_cnt, vis, vis_bits, vis_cnt, rec0, rec1, rec2, depth, rect, rect_sorted, keys0, keys1, vals0, vals1;
    size_t tile_gbase, tile_start, row_start, row_hist, band_consts, item_pack, item_v, ekey0, ekey1, eval0, eval1, entries, total;
};
RenderLayout render_layout(int32_t n, int32_t width, int32_t height, int64_t max_entries);
// Sets the calling thread's fdgs_last_error() message; returns s.
fdgs_status set_error(fdgs_status s, const char *msg);

bool make_camdev(const fdgs_camera &c, CamDev &out, const char **why);
SceneDev make_scenedev(const fdgs_scene &s);

// launchers (return cudaGetLastError())
cudaError_t launch_render(const SceneDev &sc, const uint32_t *mask_l, const uint32_t *mask_r, const CamDev &cam,
                          float t, float *out_rgb, float *out_T, char *ws, const RenderLayout &L,
                          fdgs_frame_stats *stats, cudaStream_t st, cudaEvent_t const *stage_events,
                          cudaStream_t blend_st = nullptr, cudaEvent_t split_ev = nullptr,
                          unsigned long long *contrib = nullptr, uint32_t *stv_info = nullptr,
                          bool front_only = false);
// Head of the fdgs_stv_score workspace.
struct StvState {
    uint32_t info[2];  // [0] worst frame status, [1] largest per-view entry count
    uint32_t prefix;   // radix select: selected high bits of V_p (finally V_p's bits)
    uint32_t rank;     // radix select: remaining rank within the prefix
    uint32_t hist[256];
};
struct StvLayout {
    size_t state, contrib, acc_a, acc_b, acc_c, render, total;
};
StvLayout stv_layout(int32_t n, const fdgs_camera *cams, int32_t n_cams, int64_t max_entries);
cudaError_t launch_stv(const SceneDev &sc, const CamDev *cams, const fdgs_camera *hcams, int n_cams, const float *ts,
                       int n_ts, uint32_t rank, int mode, int variant, int64_t max_entries, char *ws,
                       const StvLayout &SL, float *out_score, float *out_spatial, float *out_gamma,
                       cudaStream_t st);

__global__ void k_count_scan(uint32_t *__restrict__ cnt, int parts_ub, const uint32_t *items, int per_part,
                             uint32_t *total);
size_t prune_workspace_bytes(int32_t n);
cudaError_t launch_prune_mask(const float *score, int n, int64_t keep, uint32_t *mask, char *ws, cudaStream_t st);
cudaError_t launch_keyframe_contrib(const SceneDev &sc, const CamDev *cams, const fdgs_camera *hcams, int n_cams,
                                    float t_key, unsigned long long thr_fixed, int64_t max_entries, char *ws,
                                    const StvLayout &SL, uint32_t *out_mask, cudaStream_t st);

struct RenderGraphImpl;
cudaError_t render_graph_build(RenderGraphImpl &g, const SceneDev &sc, const CamDev &cam, char *ws,
                               const RenderLayout &L);
cudaError_t render_graph_launch(RenderGraphImpl &g, const SceneDev &sc, const uint32_t *mask_l,
                                const uint32_t *mask_r, const CamDev &cam, float t, float *out_rgb, float *out_T,
                                cudaStream_t st, cudaStream_t blend_st = nullptr, cudaEvent_t split_ev = nullptr,
                                cudaEvent_t const *ev = nullptr);
void render_graph_free(RenderGraphImpl &g);
RenderGraphImpl *render_graph_new();
void render_graph_delete(RenderGraphImpl *g);
const RenderLayout &render_graph_layout(const RenderGraphImpl &g);

cudaError_t launch_debug_strip_reach(char *ws, const RenderLayout &L, uint8_t *out, cudaStream_t st);
cudaError_t launch_keyframe(const SceneDev &sc, const CamDev *d_cams, int n_cams, float t, uint32_t *out,
                            cudaStream_t st);
cudaError_t launch_mask_or(const uint32_t *a, const uint32_t *b, int n, uint32_t *out, cudaStream_t st);
cudaError_t launch_mask_compact(const uint32_t *a, const uint32_t *b, int n, int32_t *idx, uint32_t *count,
                                uint32_t *ws_ticket_and_status, cudaStream_t st);
cudaError_t launch_scene_compact(const SceneDev &sc, const uint32_t *mask_l, const uint32_t *mask_r, float4 *params,
                                 float *opacity, float *L, float4 *sh, uint16_t *sh_index, uint32_t *gid,
                                 uint32_t *count, uint32_t *ws, cudaStream_t st);
cudaError_t launch_validate(const SceneDev &sc, unsigned long long *d_first_bad, cudaStream_t st);
cudaError_t launch_log255(const float *op, int n, float *out, cudaStream_t st);

}  // namespace fdgs
