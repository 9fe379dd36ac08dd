// render.cu -- the per-frame hot path of fdgs_render.
//
//   k_preprocess     rows 1-4: active mask OR + cull-first slice
//                    (Eq. 1) + temporal marginal (Eq. 3)
//                    + EWA projection + SH3 colour + order-preserving
//                    compaction (warp ballot, block scan, decoupled look-back)
//   k_sort_*         row 5a: stable LSD radix sort (4 x 8-bit) of the fp32 depth
//                    keys -> canonical (depth, index) order ("sorted by
//                    their depth", reading R8)
//   k_bin_*          row 5b: stable counting sort of (tile, canonical rank)
//                    entries: per-block tile histograms, column scan, scatter
//   k_blend          row 6: per-tile front-to-back Eq. 2 with warp-uniform
//                    early exit
#include <cstdio>

#include "fdgs_internal.h"

namespace fdgs {

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) { return *(const volatile uint32_t *)p; }
__device__ __forceinline__ void st_volatile(uint32_t *p, uint32_t v) { *(volatile uint32_t *)p = v; }
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Decoupled look-back (single thread): publish `total` for partition `part`,
// return the exclusive prefix.  Status word = flag(2 bits) | value(30 bits).
__device__ __forceinline__ uint32_t lookback_exclusive(uint32_t *status, uint32_t part, uint32_t total) {
    if (part == 0) {
        st_volatile(&status[0], kFlagP | total);
        return 0;
    }
    st_volatile(&status[part], kFlagA | total);
    uint32_t excl = 0;
    int j = (int)part - 1;
    while (true) {
        const uint32_t s = ld_volatile(&status[j]);
        const uint32_t f = s & ~kValMask;
        if (f == 0) continue;
        excl += s & kValMask;
        if (f == kFlagP) break;
        --j;
    }
    st_volatile(&status[part], kFlagP | (excl + total));
    return excl;
}

// ---------------------------------------------------------------- rows 1-4
__global__ void __launch_bounds__(kPreBlock) k_preprocess(SceneDev sc, const uint32_t *__restrict__ mask_l,
                                                          const uint32_t *__restrict__ mask_r, CamDev cam, float t,
                                                          Counters *ctr, uint32_t *lb, float4 *__restrict__ rec0,
                                                          float4 *__restrict__ rec1, float4 *__restrict__ rec2,
                                                          uint32_t *__restrict__ depth) {
    __shared__ uint32_t s_part, s_excl;
    __shared__ uint32_t s_wvis[kPreBlock / 32], s_wact[kPreBlock / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_part = atomicAdd(&ctr->part_ticket, 1u);
    __syncthreads();
    const uint32_t part = s_part;
    const int i = (int)part * kPreBlock + tid;
    bool act = false;
    if (i < sc.n) {
        uint32_t w = 0xffffffffu;
        if (mask_l != nullptr) {
            w = __ldg(mask_l + (i >> 5));
            if (mask_r != nullptr) w |= __ldg(mask_r + (i >> 5));
        }
        act = (w >> (i & 31)) & 1u;
    }
    Slice sl;
    Proj pj;
    int st = -1;
    if (act) {
        st = slice_gaussian(__ldg(sc.mean + i), __ldg(sc.scale + i), __ldg(sc.rot_l + i), __ldg(sc.rot_r + i),
                            __ldg(sc.L + i), t, sl);
        if (st == kNear) st = project_gaussian(sl, cam, pj);
    }
    const bool vis = st == kVisible;
    const uint32_t bvis = __ballot_sync(0xffffffffu, vis);
    const uint32_t bact = __ballot_sync(0xffffffffu, act);
    if (lane == 0) {
        s_wvis[warp] = __popc(bvis);
        s_wact[warp] = __popc(bact);
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t tot = 0, act_tot = 0;
#pragma unroll
        for (int w = 0; w < kPreBlock / 32; ++w) {
            const uint32_t c = s_wvis[w];
            s_wvis[w] = tot;
            tot += c;
            act_tot += s_wact[w];
        }
        if (act_tot) atomicAdd(&ctr->n_act, act_tot);
        const uint32_t excl = lookback_exclusive(lb, part, tot);
        s_excl = excl;
        if (part == gridDim.x - 1) ctr->n_vis = excl + tot;
    }
    __syncthreads();
    if (vis) {
        const uint32_t pos = s_excl + s_wvis[warp] + __popc(bvis & lanemask_lt());
        float rgb[3];
        sh_color(sc.sh + (size_t)i * 12, (float)sl.mu3[0] - cam.campos[0], (float)sl.mu3[1] - cam.campos[1],
                 (float)sl.mu3[2] - cam.campos[2], rgb);
        rec0[pos] = make_float4(pj.u, pj.v, pj.Ap, pj.Bp);
        rec1[pos] = make_float4(pj.Cp, pj.Q2, __int_as_float(pj.px0 | (pj.px1 << 16)),
                                __int_as_float(pj.py0 | (pj.py1 << 16)));
        rec2[pos] = make_float4(rgb[0], rgb[1], rgb[2], __int_as_float(i));
        depth[pos] = pj.depth_bits;
    }
}

// ---------------------------------------------------------------- row 5a
constexpr int kSortThreads = 256;

__device__ __forceinline__ void part_range(uint32_t n, int parts, int b, uint32_t &lo, uint32_t &hi) {
    const uint32_t chunk = (n + parts - 1) / parts;
    lo = min((uint32_t)b * chunk, n);
    hi = min(lo + chunk, n);
}

// Per-partition digit histogram; the last block to finish turns the [P][256]
// table into global exclusive offsets (digit-major, partition-minor).
__global__ void __launch_bounds__(kSortThreads) k_sort_upsweep(const uint32_t *__restrict__ keys,
                                                               const Counters *ctrc, Counters *ctr, int pass,
                                                               uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[256];
    __shared__ bool s_last;
    const int tid = threadIdx.x, P = gridDim.x, b = blockIdx.x;
    const uint32_t n = ctrc->n_vis;
    const int shift = 8 * pass;
    uint32_t lo, hi;
    part_range(n, P, b, lo, hi);
    h[tid] = 0;
    __syncthreads();
    for (uint32_t i = lo + tid; i < hi; i += kSortThreads) atomicAdd(&h[(__ldg(keys + i) >> shift) & 255u], 1u);
    __syncthreads();
    hist[(size_t)b * 256 + tid] = h[tid];
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&ctr->sort_ticket[pass], 1u) == (uint32_t)P - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // digit tid: total over partitions, block-exclusive-scan over digits, then
    // per-partition running offsets.
    uint32_t tot = 0;
    for (int p = 0; p < P; ++p) tot += ld_volatile(&hist[(size_t)p * 256 + tid]);
    __shared__ uint32_t s_scan[256];
    s_scan[tid] = tot;
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {
        const uint32_t v = tid >= off ? s_scan[tid - off] : 0;
        __syncthreads();
        s_scan[tid] += v;
        __syncthreads();
    }
    uint32_t run = s_scan[tid] - tot;
    for (int p = 0; p < P; ++p) {
        const uint32_t c = ld_volatile(&hist[(size_t)p * 256 + tid]);
        hist[(size_t)p * 256 + tid] = run;
        run += c;
    }
}

// Stable scatter: 256-item tiles, within-warp ranks by match_any, cross-warp
// prefix per digit in shared memory.
__global__ void __launch_bounds__(kSortThreads) k_sort_downsweep(const uint32_t *__restrict__ keys_in,
                                                                 const uint32_t *__restrict__ vals_in,
                                                                 uint32_t *__restrict__ keys_out,
                                                                 uint32_t *__restrict__ vals_out, const Counters *ctrc,
                                                                 int pass, const uint32_t *__restrict__ hist) {
    constexpr int NW = kSortThreads / 32;
    __shared__ uint32_t s_off[256];
    __shared__ uint32_t s_w[NW][256];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, P = gridDim.x, b = blockIdx.x;
    const uint32_t n = ctrc->n_vis;
    const int shift = 8 * pass;
    uint32_t lo, hi;
    part_range(n, P, b, lo, hi);
    if (lo >= hi) return;
    s_off[tid] = hist[(size_t)b * 256 + tid];
    for (uint32_t base = lo; base < hi; base += kSortThreads) {
        const uint32_t i = base + tid;
        const bool valid = i < hi;
        const uint32_t key = valid ? __ldg(keys_in + i) : 0u;
        const uint32_t val = valid ? (vals_in ? __ldg(vals_in + i) : i) : 0u;
        const uint32_t d = valid ? (key >> shift) & 255u : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & lanemask_lt());
#pragma unroll
        for (int k = 0; k < 8; ++k) s_w[warp][lane + 32 * k] = 0;
        __syncwarp();
        if (valid && (__ffs(peers) - 1) == lane) s_w[warp][d] = __popc(peers);
        __syncthreads();
        {
            uint32_t run = s_off[tid];
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const uint32_t c = s_w[w][tid];
                s_w[w][tid] = run;
                run += c;
            }
            s_off[tid] = run;
        }
        __syncthreads();
        if (valid) {
            const uint32_t pos = s_w[warp][d] + rank;
            if (keys_out) keys_out[pos] = key;
            vals_out[pos] = val;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- row 5b
__device__ __forceinline__ void unpack_rect(float4 r1, int &px0, int &px1, int &py0, int &py1) {
    const uint32_t ax = __float_as_uint(r1.z), ay = __float_as_uint(r1.w);
    px0 = ax & 0xffff;
    px1 = ax >> 16;
    py0 = ay & 0xffff;
    py1 = ay >> 16;
}

// Per-partition (canonical-rank range) histogram over tiles -> hist[b][T].
__global__ void __launch_bounds__(256) k_bin_count(const uint32_t *__restrict__ order, const float4 *__restrict__ rec1,
                                                   const Counters *ctrc, int tiles_x, int n_tiles,
                                                   uint32_t *__restrict__ hist) {
    extern __shared__ uint32_t sh_cnt[];
    const int tid = threadIdx.x, P = gridDim.x, b = blockIdx.x;
    for (int k = tid; k < n_tiles; k += blockDim.x) sh_cnt[k] = 0;
    __syncthreads();
    uint32_t lo, hi;
    part_range(ctrc->n_vis, P, b, lo, hi);
    for (uint32_t r = lo + tid; r < hi; r += blockDim.x) {
        const uint32_t v = __ldg(order + r);
        int px0, px1, py0, py1;
        unpack_rect(__ldg(rec1 + v), px0, px1, py0, py1);
        for (int ty = py0 >> 4; ty <= (py1 >> 4); ++ty)
            for (int tx = px0 >> 4; tx <= (px1 >> 4); ++tx) atomicAdd(&sh_cnt[ty * tiles_x + tx], 1u);
    }
    __syncthreads();
    for (int k = tid; k < n_tiles; k += blockDim.x) hist[(size_t)b * n_tiles + k] = sh_cnt[k];
}

// Column scan: for 32 consecutive tiles, exclusive prefix over partitions
// (in place) + per-tile totals; the last block scans the totals into
// tile_start[0..T] and checks the entry capacity.
__global__ void __launch_bounds__(256) k_bin_colscan(uint32_t *__restrict__ hist, int P, int n_tiles,
                                                     uint32_t *__restrict__ tile_total,
                                                     uint32_t *__restrict__ tile_start, Counters *ctr,
                                                     int64_t max_entries) {
    __shared__ uint32_t s_part[8][32];
    __shared__ bool s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t = blockIdx.x * 32 + lane;
    const int per = (P + 7) / 8;
    const int b0 = min(warp * per, P), b1 = min(b0 + per, P);
    uint32_t sum = 0;
    if (t < n_tiles)
        for (int b = b0; b < b1; ++b) sum += hist[(size_t)b * n_tiles + t];
    s_part[warp][lane] = sum;
    __syncthreads();
    if (warp == 0) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const uint32_t c = s_part[w][lane];
            s_part[w][lane] = run;
            run += c;
        }
        if (t < n_tiles) tile_total[t] = run;
    }
    __syncthreads();
    if (t < n_tiles) {
        uint32_t run = s_part[warp][lane];
        for (int b = b0; b < b1; ++b) {
            const uint32_t c = hist[(size_t)b * n_tiles + t];
            hist[(size_t)b * n_tiles + t] = run;
            run += c;
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&ctr->bin_ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // exclusive scan of tile_total -> tile_start (block-wide, chunked)
    __shared__ uint32_t s_sum[256];
    const int chunk = (n_tiles + 255) / 256;
    const int k0 = min(tid * chunk, n_tiles), k1 = min(k0 + chunk, n_tiles);
    uint32_t local = 0;
    for (int k = k0; k < k1; ++k) local += ld_volatile(&tile_total[k]);
    s_sum[tid] = local;
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {
        const uint32_t v = tid >= off ? s_sum[tid - off] : 0;
        __syncthreads();
        s_sum[tid] += v;
        __syncthreads();
    }
    uint32_t run = s_sum[tid] - local;
    for (int k = k0; k < k1; ++k) {
        tile_start[k] = run;
        run += ld_volatile(&tile_total[k]);
    }
    if (tid == 255) {
        const uint32_t E = s_sum[255];
        tile_start[n_tiles] = E;
        ctr->n_entries = E;
        if ((int64_t)E > max_entries) ctr->status = FDGS_ERR_OVERFLOW;
    }
}

// Stable scatter of entries: warp-private u16 counters per tile; warp w owns a
// contiguous sub-range of the block's canonical ranks and walks it in order.
__global__ void k_bin_scatter(const uint32_t *__restrict__ order, const float4 *__restrict__ rec1,
                              const Counters *ctrc, int tiles_x, int n_tiles, const uint32_t *__restrict__ hist,
                              const uint32_t *__restrict__ tile_start, uint32_t *__restrict__ entries) {
    extern __shared__ uint32_t sh_base[];  // [n_tiles] u32 global base, then [NW][n_tiles] u16
    const int NW = blockDim.x >> 5;
    uint16_t *cnt = reinterpret_cast<uint16_t *>(sh_base + n_tiles);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, P = gridDim.x, b = blockIdx.x;
    if (ctrc->status != FDGS_OK) return;
    uint32_t lo, hi;
    part_range(ctrc->n_vis, P, b, lo, hi);
    if (lo >= hi) return;
    for (int k = tid; k < n_tiles * NW; k += blockDim.x) cnt[k] = 0;
    __syncthreads();
    const uint32_t per = (hi - lo + NW - 1) / NW;
    const uint32_t w0 = min(lo + warp * per, hi), w1 = min(w0 + per, hi);
    uint16_t *my = cnt + warp * n_tiles;
    for (uint32_t r = w0; r < w1; ++r) {
        int px0, px1, py0, py1;
        unpack_rect(__ldg(rec1 + __ldg(order + r)), px0, px1, py0, py1);
        const int tx0 = px0 >> 4, ty0 = py0 >> 4, nx = (px1 >> 4) - tx0 + 1, ny = (py1 >> 4) - ty0 + 1;
        for (int e = lane; e < nx * ny; e += 32) {
            const int ty = ty0 + e / nx, tx = tx0 + e % nx;
            my[ty * tiles_x + tx] += 1;
        }
        __syncwarp();
    }
    __syncthreads();
    for (int k = tid; k < n_tiles; k += blockDim.x) {
        sh_base[k] = __ldg(tile_start + k) + __ldg(hist + (size_t)b * n_tiles + k);
        uint16_t run = 0;
        for (int w = 0; w < NW; ++w) {
            const uint16_t c = cnt[w * n_tiles + k];
            cnt[w * n_tiles + k] = run;
            run = (uint16_t)(run + c);
        }
    }
    __syncthreads();
    for (uint32_t r = w0; r < w1; ++r) {
        const uint32_t v = __ldg(order + r);
        int px0, px1, py0, py1;
        unpack_rect(__ldg(rec1 + v), px0, px1, py0, py1);
        const int tx0 = px0 >> 4, ty0 = py0 >> 4, nx = (px1 >> 4) - tx0 + 1, ny = (py1 >> 4) - ty0 + 1;
        for (int e = lane; e < nx * ny; e += 32) {
            const int tile = (ty0 + e / nx) * tiles_x + tx0 + e % nx;
            const uint32_t pos = sh_base[tile] + my[tile];
            my[tile] += 1;
            entries[pos] = v;
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- row 6
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

constexpr int kBlendThreads = 256;

__global__ void __launch_bounds__(kBlendThreads) k_blend(const uint32_t *__restrict__ tile_start,
                                                         const uint32_t *__restrict__ entries,
                                                         const float4 *__restrict__ rec0,
                                                         const float4 *__restrict__ rec1,
                                                         const float4 *__restrict__ rec2, Counters *ctr,
                                                         int tiles_x, int width, int height, float bg0, float bg1,
                                                         float bg2, float *__restrict__ out_rgb,
                                                         float *__restrict__ out_T, fdgs_frame_stats *stats) {
    __shared__ float4 s0[kBlendThreads];
    __shared__ float4 s1[kBlendThreads];
    __shared__ float2 s2[kBlendThreads];
    __shared__ bool s_last;
    const bool ok = ctr->status == FDGS_OK;
    const int tile = blockIdx.x, tx = tile % tiles_x, ty = tile / tiles_x;
    const int tid = threadIdx.x, lx = tid & 15, ly = tid >> 4;
    const int i = tx * 16 + lx, j = ty * 16 + ly;
    const bool inside = i < width && j < height;
    const uint32_t start = __ldg(tile_start + tile), end = __ldg(tile_start + tile + 1);
    const float pxf = (float)i + 0.5f, pyf = (float)j + 0.5f;
    const uint32_t pix = (1u << lx) | (1u << (16 + ly));
    float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
    bool done = !inside;
    uint32_t n_eval = 0, n_blend = 0;
    for (uint32_t base = ok ? start : end; base < end; base += kBlendThreads) {
        const uint32_t k = base + tid;
        if (k < end) {
            const uint32_t v = __ldg(entries + k);
            const float4 r0 = __ldg(rec0 + v), r1 = __ldg(rec1 + v), r2 = __ldg(rec2 + v);
            int px0, px1, py0, py1;
            unpack_rect(r1, px0, px1, py0, py1);
            const int x0 = max(px0 - tx * 16, 0), x1 = min(px1 - tx * 16, 15);
            const int y0 = max(py0 - ty * 16, 0), y1 = min(py1 - ty * 16, 15);
            const uint32_t xm = ((2u << x1) - 1u) & ~((1u << x0) - 1u);
            const uint32_t ym = ((2u << y1) - 1u) & ~((1u << y0) - 1u);
            s0[tid] = r0;
            s1[tid] = make_float4(r1.x, r1.y, r2.x, r2.y);
            s2[tid] = make_float2(r2.z, __uint_as_float(xm | (ym << 16)));
        }
        __syncthreads();
        if (!done) {
            const int cnt = (int)min((uint32_t)kBlendThreads, end - base);
            for (int q = 0; q < cnt; ++q) {
                const float2 c2 = s2[q];
                const uint32_t m = __float_as_uint(c2.y);
                if ((m & pix) != pix) continue;
                ++n_eval;
                const float4 a = s0[q];
                const float4 c = s1[q];
                const float dx = __fsub_rn(pxf, a.x);
                const float dy = __fsub_rn(pyf, a.y);
                const float t1 = __fmul_rn(a.w, dy);
                const float t2 = __fmaf_rn(a.z, dx, t1);
                const float t3 = __fmul_rn(c.x, dy);
                const float t4 = __fmaf_rn(t3, dy, c.y);
                const float e2 = __fmaf_rn(dx, t2, t4);
                if (!(e2 >= 0.0f)) continue;
                const float alpha = fminf(0.99f, ex2_approx(e2) * (1.0f / 255.0f));
                const float test = T * (1.0f - alpha);
                if (test < 1e-4f) {
                    done = true;
                    break;
                }
                const float w = alpha * T;
                C0 = fmaf(c.z, w, C0);
                C1 = fmaf(c.w, w, C1);
                C2 = fmaf(c2.x, w, C2);
                T = test;
                ++n_blend;
            }
        }
        if (__syncthreads_count(done) == kBlendThreads) break;
    }
    // Eq. 2 work counters (algorithmic pairs), one atomic per warp
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n_eval += __shfl_xor_sync(0xffffffffu, n_eval, o);
        n_blend += __shfl_xor_sync(0xffffffffu, n_blend, o);
    }
    if ((tid & 31) == 0 && n_eval) {
        atomicAdd(&ctr->n_eval, (unsigned long long)n_eval);
        atomicAdd(&ctr->n_blend, (unsigned long long)n_blend);
    }
    if (stats) {
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(&ctr->blend_ticket, 1u) == gridDim.x - 1;
        __syncthreads();
        if (s_last && tid == 0) {
            __threadfence();
            volatile Counters *vc = ctr;
            stats->n_act = vc->n_act;
            stats->n_vis = vc->n_vis;
            stats->n_entries = vc->n_entries;
            stats->status = vc->status;
            stats->n_evaluated = vc->n_eval;
            stats->n_blended = vc->n_blend;
        }
    }
    if (!ok) return;
    if (inside) {
        const size_t hw = (size_t)width * height, p = (size_t)j * width + i;
        out_rgb[p] = fmaf(T, bg0, C0);
        out_rgb[hw + p] = fmaf(T, bg1, C1);
        out_rgb[2 * hw + p] = fmaf(T, bg2, C2);
        if (out_T) out_T[p] = T;
    }
}

// ---------------------------------------------------------------- launcher
cudaError_t launch_render(const SceneDev &sc, const uint32_t *mask_l, const uint32_t *mask_r, const CamDev &cam,
                          float t, float *out_rgb, float *out_T, char *ws, const RenderLayout &L,
                          fdgs_frame_stats *stats, cudaStream_t st, cudaEvent_t const *ev) {
    Counters *ctr = reinterpret_cast<Counters *>(ws + L.counters);
    uint32_t *lb = reinterpret_cast<uint32_t *>(ws + L.lookback);
    float4 *rec0 = reinterpret_cast<float4 *>(ws + L.rec0);
    float4 *rec1 = reinterpret_cast<float4 *>(ws + L.rec1);
    float4 *rec2 = reinterpret_cast<float4 *>(ws + L.rec2);
    uint32_t *depth = reinterpret_cast<uint32_t *>(ws + L.depth);
    uint32_t *keys[2] = {reinterpret_cast<uint32_t *>(ws + L.keys0), reinterpret_cast<uint32_t *>(ws + L.keys1)};
    uint32_t *vals[2] = {reinterpret_cast<uint32_t *>(ws + L.vals0), reinterpret_cast<uint32_t *>(ws + L.vals1)};
    uint32_t *shist = reinterpret_cast<uint32_t *>(ws + L.sort_hist);
    uint32_t *bhist = reinterpret_cast<uint32_t *>(ws + L.bin_hist);
    uint32_t *ttot = reinterpret_cast<uint32_t *>(ws + L.tile_total);
    uint32_t *tstart = reinterpret_cast<uint32_t *>(ws + L.tile_start);
    uint32_t *entries = reinterpret_cast<uint32_t *>(ws + L.entries);

    cudaError_t e = cudaSuccess;
    if (ev && (e = cudaEventRecord(ev[0], st)) != cudaSuccess) return e;
    e = cudaMemsetAsync(ws + L.counters, 0, L.rec0 - L.counters, st);  // counters + look-back
    if (e != cudaSuccess) return e;
    if (L.n_parts > 0)
        k_preprocess<<<L.n_parts, kPreBlock, 0, st>>>(sc, mask_l, mask_r, cam, t, ctr, lb, rec0, rec1, rec2, depth);
    if (ev && (e = cudaEventRecord(ev[1], st)) != cudaSuccess) return e;
    for (int pass = 0; pass < 4; ++pass) {
        const uint32_t *kin = pass == 0 ? depth : keys[(pass - 1) & 1];
        const uint32_t *vin = pass == 0 ? nullptr : vals[(pass - 1) & 1];
        k_sort_upsweep<<<L.p_sort, kSortThreads, 0, st>>>(kin, ctr, ctr, pass, shist + (size_t)pass * L.p_sort * 256);
        k_sort_downsweep<<<L.p_sort, kSortThreads, 0, st>>>(kin, vin, pass == 3 ? nullptr : keys[pass & 1],
                                                             vals[pass & 1], ctr, pass,
                                                             shist + (size_t)pass * L.p_sort * 256);
    }
    const uint32_t *order = vals[1];
    if (ev && (e = cudaEventRecord(ev[2], st)) != cudaSuccess) return e;
    k_bin_count<<<L.p_bin, 256, (size_t)L.n_tiles * 4, st>>>(order, rec1, ctr, L.tiles_x, L.n_tiles, bhist);
    k_bin_colscan<<<(L.n_tiles + 31) / 32, 256, 0, st>>>(bhist, L.p_bin, L.n_tiles, ttot, tstart, ctr, L.max_entries);
    const size_t scat_smem = (size_t)L.n_tiles * 4 + (size_t)L.bin_warps * L.n_tiles * 2;
    k_bin_scatter<<<L.p_bin, 32 * L.bin_warps, scat_smem, st>>>(order, rec1, ctr, L.tiles_x, L.n_tiles, bhist, tstart,
                                                                 entries);
    if (ev && (e = cudaEventRecord(ev[3], st)) != cudaSuccess) return e;
    k_blend<<<L.n_tiles, kBlendThreads, 0, st>>>(tstart, entries, rec0, rec1, rec2, ctr, L.tiles_x, L.width, L.height,
                                                 cam.bg[0], cam.bg[1], cam.bg[2], out_rgb, out_T, stats);
    if (ev && (e = cudaEventRecord(ev[4], st)) != cudaSuccess) return e;
    return cudaGetLastError();
}

// Opt-in to large dynamic shared memory once per process.
__host__ cudaError_t render_set_smem_attrs() {
    cudaError_t e = cudaFuncSetAttribute(k_bin_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_bin_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

}  // namespace fdgs
