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

// Decoupled look-back, one warp: publish `total` for partition `part`, return
// the exclusive prefix (all lanes).  Status word = flag(2 bits) | value(30
// bits); the warp inspects 32 predecessors per round trip.
__device__ __forceinline__ uint32_t lookback_warp(uint32_t *status, uint32_t part, uint32_t total, int lane) {
    if (part == 0) {
        if (lane == 0) st_volatile(&status[0], kFlagP | total);
        return 0;
    }
    if (lane == 0) st_volatile(&status[part], kFlagA | total);
    uint32_t excl = 0;
    int base = (int)part - 1;
    while (true) {
        const int j = base - lane;
        uint32_t s = j >= 0 ? ld_volatile(&status[j]) : (kFlagP | 0u);
        if (__any_sync(0xffffffffu, (s & ~kValMask) == 0)) continue;  // a predecessor is not published yet
        const uint32_t pmask = __ballot_sync(0xffffffffu, (s & ~kValMask) == kFlagP);
        const int stop = pmask ? __ffs(pmask) - 1 : 31;
        uint32_t v = lane <= stop ? (s & kValMask) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (pmask) break;
        base -= 32;
    }
    if (lane == 0) st_volatile(&status[part], kFlagP | (excl + total));
    return excl;
}

// ---------------------------------------------------------------- rows 1-4
__global__ void __launch_bounds__(kPreBlock) k_preprocess(SceneDev sc, const uint32_t *__restrict__ mask_l,
                                                          const uint32_t *__restrict__ mask_r, CamDev cam, float t,
                                                          Counters *ctr, uint32_t *lb, float4 *__restrict__ rec0,
                                                          float4 *__restrict__ rec1, float4 *__restrict__ rec2,
                                                          uint32_t *__restrict__ depth, uint2 *__restrict__ rect) {
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
    if (warp == 0) {
        uint32_t tot = 0, act_tot = 0, mine = 0;
#pragma unroll
        for (int w = 0; w < kPreBlock / 32; ++w) {
            const uint32_t c = s_wvis[w];
            if (w == lane) mine = tot;
            tot += c;
            act_tot += s_wact[w];
        }
        __syncwarp();
        if (lane < kPreBlock / 32) s_wvis[lane] = mine;
        if (lane == 0 && act_tot) atomicAdd(&ctr->n_act, act_tot);
        const uint32_t excl = lookback_warp(lb, part, tot, lane);
        if (lane == 0) {
            s_excl = excl;
            if (part == gridDim.x - 1) ctr->n_vis = excl + tot;
        }
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
        rect[pos] = make_uint2(pj.px0 | (pj.px1 << 16), pj.py0 | (pj.py1 << 16));
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
__global__ void __launch_bounds__(kSortThreads) k_sort_upsweep(const uint32_t *__restrict__ keys, Counters *ctr,
                                                               int pass, uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[256];
    __shared__ uint32_t s_scan[256];
    __shared__ bool s_last;
    const int tid = threadIdx.x, P = gridDim.x, b = blockIdx.x;
    const uint32_t n = ctr->n_vis;
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
    // digit tid: total over partitions (L2 loads, pipelined), block scan over
    // digits, then per-partition running offsets.
    uint32_t tot = 0;
    int p = 0;
    for (; p + 8 <= P; p += 8) {
        uint32_t c[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k] = __ldcg(&hist[(size_t)(p + k) * 256 + tid]);
#pragma unroll
        for (int k = 0; k < 8; ++k) tot += c[k];
    }
    for (; p < P; ++p) tot += __ldcg(&hist[(size_t)p * 256 + tid]);
    s_scan[tid] = tot;
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {
        const uint32_t v = tid >= off ? s_scan[tid - off] : 0;
        __syncthreads();
        s_scan[tid] += v;
        __syncthreads();
    }
    uint32_t run = s_scan[tid] - tot;
    for (p = 0; p + 8 <= P; p += 8) {
        uint32_t c[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k] = __ldcg(&hist[(size_t)(p + k) * 256 + tid]);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            hist[(size_t)(p + k) * 256 + tid] = run;
            run += c[k];
        }
    }
    for (; p < P; ++p) {
        const uint32_t c = __ldcg(&hist[(size_t)p * 256 + tid]);
        hist[(size_t)p * 256 + tid] = run;
        run += c;
    }
}

// Stable scatter: 256-item tiles, within-warp ranks by match_any, cross-warp
// prefix per digit in shared memory.  The last pass also gathers the packed
// pixel AABB of each Gaussian into canonical order (rect_out) for binning.
__global__ void __launch_bounds__(kSortThreads) k_sort_downsweep(const uint32_t *__restrict__ keys_in,
                                                                 const uint32_t *__restrict__ vals_in,
                                                                 uint32_t *__restrict__ keys_out,
                                                                 uint32_t *__restrict__ vals_out, const Counters *ctrc,
                                                                 int pass, const uint32_t *__restrict__ hist,
                                                                 const uint2 *__restrict__ rect_in,
                                                                 uint2 *__restrict__ rect_out) {
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
        uint2 rc = make_uint2(0, 0);
        if (rect_out != nullptr && valid) rc = __ldg(rect_in + val);
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
            if (rect_out) rect_out[pos] = rc;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- row 5b
// Tile rectangle of a packed pixel AABB (16x16 tiles).
struct TileRect {
    int tx0, ty0, nx, ny;
};
__device__ __forceinline__ TileRect tile_rect(uint2 r) {
    TileRect t;
    t.tx0 = (r.x & 0xffff) >> 4;
    t.ty0 = (r.y & 0xffff) >> 4;
    t.nx = (int)(r.x >> 20) - t.tx0 + 1;
    t.ny = (int)(r.y >> 20) - t.ty0 + 1;
    return t;
}

// Per-partition tile histogram via a 2D difference array: 4 shared atomics per
// Gaussian, then row and column prefix sums -> hist[b][T].
__global__ void __launch_bounds__(256) k_bin_count(const uint2 *__restrict__ rects, const Counters *ctrc, int tiles_x,
                                                   int tiles_y, uint32_t *__restrict__ hist) {
    extern __shared__ int sh_diff[];  // (tiles_y + 1) x (tiles_x + 1)
    const int tid = threadIdx.x, P = gridDim.x, b = blockIdx.x;
    const int gx = tiles_x + 1, gy = tiles_y + 1;
    for (int k = tid; k < gx * gy; k += blockDim.x) sh_diff[k] = 0;
    __syncthreads();
    uint32_t lo, hi;
    part_range(ctrc->n_vis, P, b, lo, hi);
    for (uint32_t r = lo + tid; r < hi; r += blockDim.x) {
        const TileRect t = tile_rect(__ldg(rects + r));
        const int x1 = t.tx0 + t.nx, y1 = t.ty0 + t.ny;
        atomicAdd(&sh_diff[t.ty0 * gx + t.tx0], 1);
        atomicAdd(&sh_diff[t.ty0 * gx + x1], -1);
        atomicAdd(&sh_diff[y1 * gx + t.tx0], -1);
        atomicAdd(&sh_diff[y1 * gx + x1], 1);
    }
    __syncthreads();
    for (int y = tid; y < tiles_y; y += blockDim.x) {  // prefix along x
        int run = 0;
        for (int x = 0; x < tiles_x; ++x) {
            run += sh_diff[y * gx + x];
            sh_diff[y * gx + x] = run;
        }
    }
    __syncthreads();
    for (int x = tid; x < tiles_x; x += blockDim.x) {  // prefix along y
        int run = 0;
        for (int y = 0; y < tiles_y; ++y) {
            run += sh_diff[y * gx + x];
            sh_diff[y * gx + x] = run;
        }
    }
    __syncthreads();
    const int n_tiles = tiles_x * tiles_y;
    for (int k = tid; k < n_tiles; k += blockDim.x)
        hist[(size_t)b * n_tiles + k] = (uint32_t)sh_diff[(k / tiles_x) * gx + (k % tiles_x)];
}

// Column scan: tile t's exclusive prefix over partitions (in place) and its
// total; the last block scans the totals into tile_start[0..T] and checks the
// entry capacity.  Block = 32 tiles x 32 partition slices.
__global__ void __launch_bounds__(1024) k_bin_colscan(uint32_t *__restrict__ hist, int P, int n_tiles,
                                                      uint32_t *__restrict__ tile_total,
                                                      uint32_t *__restrict__ tile_start, Counters *ctr,
                                                      int64_t max_entries) {
    __shared__ uint32_t s_part[32][33];
    __shared__ uint32_t s_sum[1024];
    __shared__ bool s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t = blockIdx.x * 32 + lane;
    const int per = (P + 31) / 32;
    const int b0 = min(warp * per, P), b1 = min(b0 + per, P);
    uint32_t sum = 0;
    if (t < n_tiles)
        for (int b = b0; b < b1; ++b) sum += __ldcg(&hist[(size_t)b * n_tiles + t]);
    s_part[warp][lane] = sum;
    __syncthreads();
    if (warp == 0) {
        uint32_t run = 0;
        for (int w = 0; w < 32; ++w) {
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
            const uint32_t c = __ldcg(&hist[(size_t)b * n_tiles + t]);
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
    const int chunk = (n_tiles + 1023) / 1024;
    const int k0 = min(tid * chunk, n_tiles), k1 = min(k0 + chunk, n_tiles);
    uint32_t local = 0;
    for (int k = k0; k < k1; ++k) local += __ldcg(&tile_total[k]);
    s_sum[tid] = local;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const uint32_t v = tid >= off ? s_sum[tid - off] : 0;
        __syncthreads();
        s_sum[tid] += v;
        __syncthreads();
    }
    uint32_t run = s_sum[tid] - local;
    for (int k = k0; k < k1; ++k) {
        tile_start[k] = run;
        run += __ldcg(&tile_total[k]);
    }
    if (tid == 1023) {
        const uint32_t E = s_sum[1023];
        tile_start[n_tiles] = E;
        ctr->n_entries = E;
        if ((int64_t)E > max_entries) ctr->status = FDGS_ERR_OVERFLOW;
    }
}

// Stable scatter of entries.  Warp w owns a contiguous sub-range of the
// block's canonical ranks and walks it in order with warp-private u16 tile
// counters; each round loads 32 rects at once and broadcasts them by shuffle.
__global__ void k_bin_scatter(const uint32_t *__restrict__ order, const uint2 *__restrict__ rects,
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
    for (uint32_t r0 = w0; r0 < w1; r0 += 32) {
        const uint32_t r = r0 + lane;
        const uint2 rc = r < w1 ? __ldg(rects + r) : make_uint2(0, 0);
        const int m = min(32u, w1 - r0);
        for (int j = 0; j < m; ++j) {
            const uint2 q = make_uint2(__shfl_sync(0xffffffffu, rc.x, j), __shfl_sync(0xffffffffu, rc.y, j));
            const TileRect t = tile_rect(q);
            for (int e = lane; e < t.nx * t.ny; e += 32) {
                const int ty = t.ty0 + e / t.nx, tx = t.tx0 + e % t.nx;
                my[ty * tiles_x + tx] += 1;
            }
            __syncwarp();
        }
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
    for (uint32_t r0 = w0; r0 < w1; r0 += 32) {
        const uint32_t r = r0 + lane;
        uint2 rc = make_uint2(0, 0);
        uint32_t v = 0;
        if (r < w1) {
            rc = __ldg(rects + r);
            v = __ldg(order + r);
        }
        const int m = min(32u, w1 - r0);
        for (int j = 0; j < m; ++j) {
            const uint2 q = make_uint2(__shfl_sync(0xffffffffu, rc.x, j), __shfl_sync(0xffffffffu, rc.y, j));
            const uint32_t vj = __shfl_sync(0xffffffffu, v, j);
            const TileRect t = tile_rect(q);
            for (int e = lane; e < t.nx * t.ny; e += 32) {
                const int tile = (t.ty0 + e / t.nx) * tiles_x + t.tx0 + e % t.nx;
                const uint32_t pos = sh_base[tile] + my[tile];
                my[tile] += 1;
                entries[pos] = vj;
            }
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------- row 6
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Packed fp32x2 (Blackwell FADD2/FFMA2), IEEE RN per lane.  Used only where
// no product feeds an add (no contraction hazard), see DESIGN.md.
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    float2 d;
    asm("sub.rn.f32x2 %0, %1, %2;"
        : "=l"(*reinterpret_cast<unsigned long long *>(&d))
        : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)));
    return d;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(*reinterpret_cast<unsigned long long *>(&d))
        : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)),
          "l"(*reinterpret_cast<unsigned long long *>(&c)));
    return d;
}

constexpr int kBlendThreads = 128;  // one 16x16 tile, 2 horizontally adjacent pixels per thread

// Staged splat record in shared memory (double-buffered batches).
struct BlendBatch {
    float4 a[kBlendThreads];  // u, v, A', B'
    float4 c[kBlendThreads];  // C', Q2, r, g
    float2 d[kBlendThreads];  // b, tile-local AABB mask (x bits 0-15, y bits 16-31)
};

__device__ __forceinline__ void stage_load(const uint32_t *__restrict__ entries, const float4 *__restrict__ rec0,
                                           const float4 *__restrict__ rec1, const float4 *__restrict__ rec2,
                                           uint32_t k, uint32_t end, float4 &r0, float4 &r1, float4 &r2) {
    if (k < end) {
        const uint32_t v = __ldg(entries + k);
        r0 = __ldg(rec0 + v);
        r1 = __ldg(rec1 + v);
        r2 = __ldg(rec2 + v);
    }
}

__device__ __forceinline__ void stage_store(BlendBatch &B, int tid, uint32_t k, uint32_t end, int tx, int ty,
                                            const float4 &r0, const float4 &r1, const float4 &r2) {
    if (k < end) {
        const uint32_t ax = __float_as_uint(r1.z), ay = __float_as_uint(r1.w);
        const int x0 = max((int)(ax & 0xffff) - tx * 16, 0), x1 = min((int)(ax >> 16) - tx * 16, 15);
        const int y0 = max((int)(ay & 0xffff) - ty * 16, 0), y1 = min((int)(ay >> 16) - ty * 16, 15);
        const uint32_t xm = ((2u << x1) - 1u) & ~((1u << x0) - 1u);
        const uint32_t ym = ((2u << y1) - 1u) & ~((1u << y0) - 1u);
        B.a[tid] = r0;
        B.c[tid] = make_float4(r1.x, r1.y, r2.x, r2.y);
        B.d[tid] = make_float2(r2.z, __uint_as_float(xm | (ym << 16)));
    }
}

template <bool kCount>
__global__ void __launch_bounds__(kBlendThreads) k_blend(const uint32_t *__restrict__ tile_start,
                                                         const uint32_t *__restrict__ entries,
                                                         const float4 *__restrict__ rec0,
                                                         const float4 *__restrict__ rec1,
                                                         const float4 *__restrict__ rec2, Counters *ctr,
                                                         int tiles_x, int width, int height, float bg0, float bg1,
                                                         float bg2, float *__restrict__ out_rgb,
                                                         float *__restrict__ out_T, fdgs_frame_stats *stats) {
    __shared__ BlendBatch sb[2];
    __shared__ bool s_last;
    const bool ok = ctr->status == FDGS_OK;
    const int tile = blockIdx.x, tx = tile % tiles_x, ty = tile / tiles_x;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int ly = tid >> 3, lx = (tid & 7) * 2;
    const int i0 = tx * 16 + lx, j = ty * 16 + ly;
    const bool in0 = i0 < width && j < height, in1 = i0 + 1 < width && j < height;
    const uint32_t start = __ldg(tile_start + tile), end = __ldg(tile_start + tile + 1);
    const float pyf = (float)j + 0.5f;
    const float2 px = make_float2((float)i0 + 0.5f, (float)(i0 + 1) + 0.5f);
    const uint32_t pb0 = (1u << lx) | (1u << (16 + ly)), pb1 = (2u << lx) | (1u << (16 + ly));
    const uint32_t wrows = 0xFu << (16 + 4 * warp);  // this warp's 4 rows in the y-mask
    float2 T = make_float2(1.0f, 1.0f), Cr = make_float2(0.f, 0.f), Cg = Cr, Cb = Cr;
    bool done0 = !in0, done1 = !in1;
    uint32_t n_eval = 0, n_blend = 0;
    const uint32_t first = ok ? start : end;
    float4 r0, r1, r2;
    stage_load(entries, rec0, rec1, rec2, first + tid, end, r0, r1, r2);
    stage_store(sb[0], tid, first + tid, end, tx, ty, r0, r1, r2);
    __syncthreads();
    int buf = 0;
    for (uint32_t base = first; base < end; base += kBlendThreads) {
        const uint32_t nxt = base + kBlendThreads;
        stage_load(entries, rec0, rec1, rec2, nxt + tid, end, r0, r1, r2);  // prefetch the next batch
        const BlendBatch &B = sb[buf];
        if (!(done0 && done1)) {
            const int cnt = (int)min((uint32_t)kBlendThreads, end - base);
            for (int q = 0; q < cnt; ++q) {
                const float2 dq = B.d[q];
                const uint32_t m = __float_as_uint(dq.y);
                if ((m & wrows) == 0) continue;  // warp-uniform: no row of this warp in the AABB
                const float4 a = B.a[q];
                const float4 c = B.c[q];
                // pinned e2 chain: dy terms once per row, dx terms per pixel
                const float dy = __fsub_rn(pyf, a.y);
                const float t1 = __fmul_rn(a.w, dy);
                const float t3 = __fmul_rn(c.x, dy);
                const float t4 = __fmaf_rn(t3, dy, c.y);
                const float2 dx = sub2(px, make_float2(a.x, a.x));
                const float2 t2 = fma2(make_float2(a.z, a.z), dx, make_float2(t1, t1));
                const float2 e2 = fma2(dx, t2, make_float2(t4, t4));
                const bool box0 = (m & pb0) == pb0 && !done0, box1 = (m & pb1) == pb1 && !done1;
                const bool v0 = box0 && e2.x >= 0.0f, v1 = box1 && e2.y >= 0.0f;
                if (kCount) n_eval += (uint32_t)box0 + (uint32_t)box1;
                if (!(v0 || v1)) continue;
                const float a0 = v0 ? fminf(0.99f, ex2_approx(e2.x) * (1.0f / 255.0f)) : 0.0f;
                const float a1 = v1 ? fminf(0.99f, ex2_approx(e2.y) * (1.0f / 255.0f)) : 0.0f;
                float w0 = a0 * T.x, w1 = a1 * T.y;
                const bool s0 = v0 && (T.x - w0) < 1e-4f, s1 = v1 && (T.y - w1) < 1e-4f;
                w0 = s0 ? 0.0f : w0;
                w1 = s1 ? 0.0f : w1;
                done0 |= s0;
                done1 |= s1;
                if (kCount) n_blend += (uint32_t)(v0 && !s0) + (uint32_t)(v1 && !s1);
                const float2 w = make_float2(w0, w1);
                T = sub2(T, w);
                Cr = fma2(make_float2(c.z, c.z), w, Cr);
                Cg = fma2(make_float2(c.w, c.w), w, Cg);
                Cb = fma2(make_float2(dq.x, dq.x), w, Cb);
                if (done0 && done1) break;
            }
        }
        stage_store(sb[buf ^ 1], tid, nxt + tid, end, tx, ty, r0, r1, r2);
        buf ^= 1;
        if (__syncthreads_count(done0 && done1) == kBlendThreads) break;
    }
    if (kCount) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            n_eval += __shfl_xor_sync(0xffffffffu, n_eval, o);
            n_blend += __shfl_xor_sync(0xffffffffu, n_blend, o);
        }
        if ((tid & 31) == 0 && n_eval) {
            atomicAdd(&ctr->n_eval, (unsigned long long)n_eval);
            atomicAdd(&ctr->n_blend, (unsigned long long)n_blend);
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(&ctr->blend_ticket, 1u) == gridDim.x - 1;
        __syncthreads();
        if (s_last && tid == 0 && stats != nullptr) {
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
    const size_t hw = (size_t)width * height, p = (size_t)j * width + i0;
    if (in0) {
        out_rgb[p] = fmaf(T.x, bg0, Cr.x);
        out_rgb[hw + p] = fmaf(T.x, bg1, Cg.x);
        out_rgb[2 * hw + p] = fmaf(T.x, bg2, Cb.x);
        if (out_T) out_T[p] = T.x;
    }
    if (in1) {
        out_rgb[p + 1] = fmaf(T.y, bg0, Cr.y);
        out_rgb[hw + p + 1] = fmaf(T.y, bg1, Cg.y);
        out_rgb[2 * hw + p + 1] = fmaf(T.y, bg2, Cb.y);
        if (out_T) out_T[p + 1] = T.y;
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
    uint2 *rect = reinterpret_cast<uint2 *>(ws + L.rect);
    uint2 *rect_sorted = reinterpret_cast<uint2 *>(ws + L.rect_sorted);
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
        k_preprocess<<<L.n_parts, kPreBlock, 0, st>>>(sc, mask_l, mask_r, cam, t, ctr, lb, rec0, rec1, rec2, depth,
                                                      rect);
    if (ev && (e = cudaEventRecord(ev[1], st)) != cudaSuccess) return e;
    for (int pass = 0; pass < 4; ++pass) {
        const uint32_t *kin = pass == 0 ? depth : keys[(pass - 1) & 1];
        const uint32_t *vin = pass == 0 ? nullptr : vals[(pass - 1) & 1];
        uint32_t *h = shist + (size_t)pass * L.p_sort * 256;
        k_sort_upsweep<<<L.p_sort, kSortThreads, 0, st>>>(kin, ctr, pass, h);
        k_sort_downsweep<<<L.p_sort, kSortThreads, 0, st>>>(kin, vin, pass == 3 ? nullptr : keys[pass & 1],
                                                             vals[pass & 1], ctr, pass, h, rect,
                                                             pass == 3 ? rect_sorted : nullptr);
    }
    const uint32_t *order = vals[1];
    if (ev && (e = cudaEventRecord(ev[2], st)) != cudaSuccess) return e;
    const size_t cnt_smem = sizeof(int) * (size_t)(L.tiles_x + 1) * (L.tiles_y + 1);
    k_bin_count<<<L.p_bin, 256, cnt_smem, st>>>(rect_sorted, ctr, L.tiles_x, L.tiles_y, bhist);
    k_bin_colscan<<<(L.n_tiles + 31) / 32, 1024, 0, st>>>(bhist, L.p_bin, L.n_tiles, ttot, tstart, ctr, L.max_entries);
    const size_t scat_smem = (size_t)L.n_tiles * 4 + (size_t)L.bin_warps * L.n_tiles * 2;
    k_bin_scatter<<<L.p_bin, 32 * L.bin_warps, scat_smem, st>>>(order, rect_sorted, ctr, L.tiles_x, L.n_tiles, bhist,
                                                                 tstart, entries);
    if (ev && (e = cudaEventRecord(ev[3], st)) != cudaSuccess) return e;
    if (stats != nullptr)
        k_blend<true><<<L.n_tiles, kBlendThreads, 0, st>>>(tstart, entries, rec0, rec1, rec2, ctr, L.tiles_x, L.width,
                                                           L.height, cam.bg[0], cam.bg[1], cam.bg[2], out_rgb, out_T,
                                                           stats);
    else
        k_blend<false><<<L.n_tiles, kBlendThreads, 0, st>>>(tstart, entries, rec0, rec1, rec2, ctr, L.tiles_x, L.width,
                                                            L.height, cam.bg[0], cam.bg[1], cam.bg[2], out_rgb, out_T,
                                                            nullptr);
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
