// render.cu -- the per-frame hot path of fdgs_render.
//
//   k_cull           rows 1-2 + temporal cull: active mask OR,
//                    binary64 p_t >= 1/255 test (Eq. 3); survivor
//                    bits and per-partition counts -> k_count_scan ->
//                    k_cull_emit (survivors compacted in index order)
//   k_slice          rows 3-4 on the survivors: Eq. 1 slice, EWA
//                    projection + SH3 colour, the aabb_redundant bit;
//                    visible counts -> k_count_scan -> k_vis_emit
//   k_sort_*         row 5a: stable onesweep LSD radix sort (4 x 8-bit) of the
//                    fp32 depth keys -> canonical (depth, index) order (P:126
//                    "sorted by their depth", reading R8)
//   k_bin_count..    row 5b: tile cover per (Gaussian, tile row) (band_tiles),
//   k_row_scatter    per-tile counts, a stable 8-bit row partition of the row
//                    items, per-row warp-ordered scatter into the tile lists
//   k_blend_wi       row 6: per-tile front-to-back Eq. 2, four
//                    independent warps per tile, each staging and compositing
//                    its own record lists, U = T/255 carried, one stop test per
//                    pair of records (the timed kernel)
//   k_blend_ws       row 6: the counting / contribution-recording variant
//                    (producer warp + 4 consumer warps, visits every record)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <new>
#include <type_traits>
#include <vector>

#include "fdgs_internal.h"

namespace fdgs {

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) { return *(const volatile uint32_t *)p; }
__device__ __forceinline__ void st_volatile(uint32_t *p, uint32_t v) { *(volatile uint32_t *)p = v; }
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}


// ---------------------------------------------------------------- rows 1-4
// Uniform-work passes instead of one fused kernel whose blocks waited on their
// few survivor warps (ncu at C4: 59% of cycles stalled at the barriers), and
// no in-kernel look-back (blocks waiting on predecessors):
//   k_cull + k_count_scan + k_cull_emit   rows 1-2 + the temporal cull of row
//            3: one thread per Gaussian, mask bit (OR of the two key-frame
//            rows) then the pinned binary64 temporal test; survivor bits and
//            counts, scanned, emitted in ascending index order -> surv[];
//   k_slice + k_count_scan + k_vis_emit   rows 3-4 on the dense survivor list:
//            Eq. 1 slice, support and near culls, EWA projection, cover cull,
//            SH colour; records at the survivor slot, the visible slots
//            compacted in order (vis[], and their depth keys for the sort).
constexpr int kCullItems = 4 * kPreBlock;   // Gaussians per k_cull partition
constexpr int kSliceItems = 2 * kPreBlock;  // survivors per k_slice partition

// k_cull runs as three non-blocking passes (a decoupled look-back here left
// 53% of the warps waiting at the block barrier at C4): the survivor bits and
// per-partition counts, a one-block scan of the counts, then the ordered
// emission of the survivor indices.
__global__ void __launch_bounds__(kPreBlock) k_cull(SceneDev sc, const uint32_t *__restrict__ mask_l,
                                                    const uint32_t *__restrict__ mask_r, float t, Counters *ctr,
                                                    uint32_t *__restrict__ bits, uint32_t *__restrict__ cnt) {
    constexpr int R = kCullItems / kPreBlock;
    __shared__ uint32_t s_act, s_n;
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t part = blockIdx.x;
    // the scene's Gaussians: n, or a device count (a working set compacted on the
    // device); bits and counts are written for the whole capacity n
    const int n = sc.d_n ? min((int)__ldg(sc.d_n), sc.n) : sc.n;
    if (tid == 0) s_act = s_n = 0;
    __syncthreads();
    uint32_t nact = 0, nsurv = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = (int)part * kCullItems + r * kPreBlock + tid;
        bool act = false, keep = false;
        if (i < n) {
            uint32_t w = 0xffffffffu;
            if (mask_l != nullptr) {
                w = __ldg(mask_l + (i >> 5));
                if (mask_r != nullptr) w |= __ldg(mask_r + (i >> 5));
            }
            act = (w >> (i & 31)) & 1u;
            if (act) keep = temporal_pass(sc.ld_mean(i), sc.ld_scale(i), sc.ld_rot_l(i), sc.ld_rot_r(i), t);
        }
        nact += __popc(__ballot_sync(0xffffffffu, act));
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        nsurv += __popc(bal);
        if (lane == 0 && i - lane < sc.n) bits[i >> 5] = bal;
    }
    if (lane == 0) {
        if (nact) atomicAdd(&s_act, nact);
        if (nsurv) atomicAdd(&s_n, nsurv);
    }
    __syncthreads();
    if (tid == 0) {
        cnt[part] = s_n;
        if (s_act) atomicAdd(&ctr->n_act, s_act);
    }
}

// One block: exclusive scan of per-partition counts (in place), the total to
// *total.  parts = parts_ub, or ceil(*items / per_part) when items != NULL (the
// item count is only known on the device).
__global__ void __launch_bounds__(1024) k_count_scan(uint32_t *__restrict__ cnt, int parts_ub,
                                                     const uint32_t *items, int per_part, uint32_t *total) {
    __shared__ uint32_t s_w[32];
    __shared__ uint32_t s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int parts = items ? min(parts_ub, (int)((*items + per_part - 1) / per_part)) : parts_ub;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int c0 = 0; c0 < parts; c0 += 1024) {
        const int i = c0 + tid;
        const uint32_t x = i < parts ? cnt[i] : 0u;
        uint32_t inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) s_w[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const uint32_t wv = s_w[lane];
            uint32_t wi = wv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            s_w[lane] = wi - wv;
        }
        __syncthreads();
        const uint32_t carry = s_carry;
        if (i < parts) cnt[i] = carry + s_w[warp] + inc - x;
        __syncthreads();
        if (tid == 1023) s_carry = carry + s_w[31] + inc;
        __syncthreads();
    }
    if (tid == 0) *total = s_carry;
}

// Ordered emission: partition p's survivors go to [base_p, base_p + count).
__global__ void __launch_bounds__(kPreBlock) k_cull_emit(const uint32_t *__restrict__ bits,
                                                         const uint32_t *__restrict__ base, int n,
                                                         uint32_t *__restrict__ surv) {
    constexpr int WORDS = kCullItems / 32;  // 32 bit-words per partition
    __shared__ uint32_t s_off[WORDS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t part = blockIdx.x;
    const int nw = (n + 31) / 32;
    if (warp == 0) {
        const int wi = (int)part * WORDS + lane;
        const uint32_t c = wi < nw ? __popc(__ldg(bits + wi)) : 0u;
        uint32_t inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        s_off[lane] = __ldg(base + part) + inc - c;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < WORDS / (kPreBlock / 32); ++k) {
        const int w = warp * (WORDS / (kPreBlock / 32)) + k;  // word of this partition
        const int wi = (int)part * WORDS + w;
        if (wi >= nw) break;
        const uint32_t word = __ldg(bits + wi);
        if ((word >> lane) & 1u) surv[s_off[w] + __popc(word & lanemask_lt())] = (uint32_t)(wi * 32 + lane);
    }
}

// Grid-stride over partitions of kSliceItems survivors.  Records of visible
// Gaussians are written at their survivor slot (sparse); the visibility bits
// and per-partition counts feed k_count_scan + k_vis_emit, which compact the
// slots in order without any block waiting on another.
#ifndef FDGS_SLICE_MINB
#define FDGS_SLICE_MINB 3
#endif

// Is the pixel-AABB test redundant for this record?  True if every pixel centre
// of the image whose pinned fp32 e2 chain (DESIGN.md §3 step 10) can reach
// e2 >= 0 lies inside the AABB.  The chain has 7 roundings, each <= 2^-24 of a
// term bounded by |A'|dx^2 + |B'||dx dy| + |C'|dy^2 + |Q2|, so fp32 e2 <= the
// exact quadratic with A', C' scaled by (1 - d), |B'| by (1 + d), Q2 raised by
// d|Q2|, d = 2^-19 (> 9 x 2^-24 with slack); that quadratic's superlevel set
// {>= 0} lies in the box u +- dxm, v +- dym (dxm^2 = -4C''Q''/K'',
// K'' = 4A''C'' - B''^2, for either sign of B''), evaluated in binary64 and
// widened by 2^-30.  The blend then skips the per-pixel AABB test for lists of
// such records (bit 31 of rec1.w; results identical by construction).
__device__ __forceinline__ bool aabb_redundant(const Proj &pj, int W, int H) {
    constexpr double d = 0x1p-19, s = 1.0 + 0x1p-30;
    const double A = (double)pj.Ap * (1.0 - d), C = (double)pj.Cp * (1.0 - d);
    const double B = fabs((double)pj.Bp) * (1.0 + d), Q = (double)pj.Q2 + d * fabs((double)pj.Q2);
    if (Q < 0.0) return true;  // no pixel reaches e2 >= 0
    const double K = 4.0 * A * C - B * B;
    if (!(K > 0.0) || !(A < 0.0) || !(C < 0.0)) return false;
    const double dxm = sqrt((-4.0 * C * Q) / K) * s + 0x1p-30, dym = sqrt((-4.0 * A * Q) / K) * s + 0x1p-30;
    const double u = pj.u, v = pj.v;
    const double cx0 = fmax(ceil(u - dxm - 0.5), 0.0), cx1 = fmin(floor(u + dxm - 0.5), W - 1.0);
    const double cy0 = fmax(ceil(v - dym - 0.5), 0.0), cy1 = fmin(floor(v + dym - 0.5), H - 1.0);
    if (cx0 > cx1 || cy0 > cy1) return true;
    return cx0 >= pj.px0 && cx1 <= pj.px1 && cy0 >= pj.py0 && cy1 <= pj.py1;
}
__global__ void __launch_bounds__(kPreBlock, FDGS_SLICE_MINB) k_slice(SceneDev sc, CamDev cam, float t, Counters *ctr,
                                                     const uint32_t *__restrict__ surv, float4 *__restrict__ rec0,
                                                     float4 *__restrict__ rec1, float4 *__restrict__ rec2,
                                                     uint32_t *__restrict__ depth, uint2 *__restrict__ rect,
                                                     uint32_t *__restrict__ vbits, uint32_t *__restrict__ vcnt) {
    constexpr int R = kSliceItems / kPreBlock;
    __shared__ uint32_t s_n;
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t ns = ctr->n_surv;
    const uint32_t parts = (ns + kSliceItems - 1) / kSliceItems;
    for (uint32_t part = blockIdx.x; part < parts; part += gridDim.x) {
        if (tid == 0) s_n = 0;
        __syncthreads();
        uint32_t nv = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t sidx = part * kSliceItems + r * kPreBlock + tid;
            bool vis = false;
            if (sidx < ns) {
                const int i = (int)__ldg(surv + sidx);
                Slice sl;
                Proj pj;
                int st = slice_gaussian(sc.ld_mean(i), sc.ld_scale(i), sc.ld_rot_l(i), sc.ld_rot_r(i), __ldg(sc.L + i),
                                        t, sl);
                if (st == kNear) st = project_gaussian(sl, cam, pj);
                vis = st == kVisible;
                if (vis) {
                    float rgb[3];
                    const float mx = (float)sl.mu3[0], my = (float)sl.mu3[1], mz = (float)sl.mu3[2];
                    // dense SH, or the VQ codebook entry of the Gaussian (Ours-PP decode)
                    const size_t row = sc.sh_index ? (size_t)__ldg(sc.sh_index + i) : (size_t)i;
                    sh_color(sc.sh + row * 12, mx - cam.campos[0], my - cam.campos[1], mz - cam.campos[2], rgb);
                    const uint32_t ax = pj.px0 | (pj.px1 << 16), ay = pj.py0 | (pj.py1 << 16);
                    rec0[sidx] = make_float4(pj.u, pj.v, pj.Ap, pj.Bp);
                    const uint32_t inside = aabb_redundant(pj, cam.width, cam.height) ? 0x80000000u : 0u;
                    rec1[sidx] = make_float4(pj.Cp, pj.Q2, __uint_as_float(ax), __uint_as_float(ay | inside));
                    rec2[sidx] = make_float4(rgb[0], rgb[1], rgb[2], __uint_as_float(sc.orig(i)));
                    depth[sidx] = pj.depth_bits;
                    rect[sidx] = make_uint2(ax, ay);
                }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, vis);
            nv += __popc(bal);
            if (lane == 0 && sidx - lane < ns) vbits[sidx >> 5] = bal;
        }
        if (lane == 0 && nv) atomicAdd(&s_n, nv);
        __syncthreads();
        if (tid == 0) vcnt[part] = s_n;
    }
}

// Ordered compaction of the visible survivor slots: vis[pos] = slot and the
// depth key beside it (the depth sort's input), pos = partition base + rank.
__global__ void __launch_bounds__(kPreBlock) k_vis_emit(const uint32_t *__restrict__ vbits,
                                                        const uint32_t *__restrict__ base, const Counters *ctr,
                                                        const uint32_t *__restrict__ depth, uint32_t *__restrict__ vis,
                                                        uint32_t *__restrict__ keys) {
    constexpr int WORDS = kSliceItems / 32;  // 16 bit-words per partition
    __shared__ uint32_t s_off[WORDS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t ns = ctr->n_surv;
    const uint32_t parts = (ns + kSliceItems - 1) / kSliceItems;
    const int nw = (int)((ns + 31) / 32);
    for (uint32_t part = blockIdx.x; part < parts; part += gridDim.x) {
        if (warp == 0) {
            const int wi = (int)part * WORDS + lane;
            const uint32_t c = (lane < WORDS && wi < nw) ? __popc(__ldg(vbits + wi)) : 0u;
            uint32_t inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane < WORDS) s_off[lane] = __ldg(base + part) + inc - c;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < WORDS / (kPreBlock / 32); ++k) {
            const int w = warp * (WORDS / (kPreBlock / 32)) + k;
            const int wi = (int)part * WORDS + w;
            if (wi < nw) {
                const uint32_t word = __ldg(vbits + wi);
                if ((word >> lane) & 1u) {
                    const uint32_t slot = (uint32_t)(wi * 32 + lane), pos = s_off[w] + __popc(word & lanemask_lt());
                    vis[pos] = slot;
                    keys[pos] = __ldg(depth + slot);
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- rows 5a/5b
// Both sorts are stable LSD radix passes in onesweep form: partitions taken in
// ticket order, within-warp ranks by match_any, per-warp digit counters,
// per-digit decoupled look-back across partitions.  Look-back status words
// are 64-bit {epoch:32 | flag:2 | count:30}; the epoch (bumped once per frame)
// retires the previous frame's words, so no per-frame zeroing is needed.
constexpr int kSortThreads = 256;
#ifndef FDGS_LB_WIN
#define FDGS_LB_WIN 8
#endif
constexpr int kLbWin = FDGS_LB_WIN;  // predecessors read per look-back round trip
constexpr uint64_t kStA = 1ull << 30, kStP = 2ull << 30;

__device__ __forceinline__ uint64_t ld_volatile64(const uint64_t *p) { return *(const volatile uint64_t *)p; }
__device__ __forceinline__ void st_volatile64(uint64_t *p, uint64_t v) { *(volatile uint64_t *)p = v; }

__device__ __forceinline__ void part_range(uint32_t n, int parts, int b, uint32_t &lo, uint32_t &hi) {
    const uint32_t chunk = (n + parts - 1) / parts;
    lo = min((uint32_t)b * chunk, n);
    hi = min(lo + chunk, n);
}

// One stable pass over n = *n_ptr keys (digit = (key >> shift) & (2^BITS-1)).
//   gbase  : exclusive global base of every digit
//   status : [parts][2^BITS] look-back words (epoch-tagged)
//   vals_in NULL = identity values; keys_out NULL = do not write keys;
//   rect_in/rect_out: optional payload gathered through the value (row 5b input).
// The partition is reordered by digit in shared memory first, so the global
// stores are contiguous runs per digit (coalesced) instead of 4-byte scatters.
template <int BITS, int ITEMS>
__global__ void __launch_bounds__(kSortThreads) k_onesweep(const uint32_t *__restrict__ keys_in,
                                                           const uint32_t *__restrict__ vals_in,
                                                           uint32_t *__restrict__ keys_out,
                                                           uint32_t *__restrict__ vals_out, const uint32_t *n_ptr,
                                                           const uint32_t *epoch_ptr, uint32_t *ticket, int shift,
                                                           const uint32_t *__restrict__ gbase, uint64_t *status,
                                                           const uint2 *__restrict__ rect_in,
                                                           uint2 *__restrict__ rect_out) {
    constexpr int NW = kSortThreads / 32;
    constexpr int D = 1 << BITS;
    constexpr int TILE = kSortThreads * ITEMS;
    constexpr uint32_t MASK = D - 1;
    __shared__ uint32_t s_w[NW][D];
    __shared__ uint32_t s_lbase[D];   // block-local exclusive base of each digit
    __shared__ uint32_t s_gofs[D];    // global position of the digit's first key in this partition
    __shared__ uint32_t s_key[TILE], s_val[TILE];
    __shared__ uint32_t s_part;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n = *n_ptr;
    const uint64_t epoch = (uint64_t)*epoch_ptr << 32;
    const uint32_t parts = (n + TILE - 1) / TILE;
    while (true) {  // persistent: partitions are taken in ticket order
    if (tid == 0) s_part = atomicAdd(ticket, 1u);
    for (int k = lane; k < D; k += 32) s_w[warp][k] = 0;
    __syncthreads();
    const uint32_t part = s_part;
    if (part >= parts) return;
    uint32_t key[ITEMS], val[ITEMS], dig[ITEMS], rk[ITEMS];
    const uint32_t base = part * TILE + warp * (32 * ITEMS);
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const uint32_t i = base + k * 32 + lane;
        const bool valid = i < n;
        key[k] = valid ? __ldg(keys_in + i) : 0u;
        val[k] = valid ? (vals_in ? __ldg(vals_in + i) : i) : 0u;
        dig[k] = valid ? (key[k] >> shift) & MASK : (uint32_t)D;
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const uint32_t peers = __match_any_sync(0xffffffffu, dig[k]);
        const bool leader = (__ffs(peers) - 1) == lane;
        if (dig[k] < (uint32_t)D) rk[k] = s_w[warp][dig[k]] + __popc(peers & lanemask_lt());
        __syncwarp();
        if (leader && dig[k] < (uint32_t)D) s_w[warp][dig[k]] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit: prefix over warps, block total, block-local base (scan over
    // digits), then the look-back for the global offset
    uint32_t tot_d[(D + kSortThreads - 1) / kSortThreads];
#pragma unroll
    for (int c = 0; c * kSortThreads < D; ++c) {
        const int d = c * kSortThreads + tid;
        uint32_t tot = 0;
        if (d < D) {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const uint32_t x = s_w[w][d];
                s_w[w][d] = tot;
                tot += x;
            }
            s_lbase[d] = tot;
        }
        tot_d[c] = tot;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the digit totals (D <= 256)
        uint32_t run = 0;
        for (int c0 = 0; c0 < D; c0 += 32) {
            const uint32_t x = c0 + lane < D ? s_lbase[c0 + lane] : 0u;
            uint32_t inc = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (c0 + lane < D) s_lbase[c0 + lane] = run + inc - x;
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c * kSortThreads < D; ++c) {
        const int d = c * kSortThreads + tid;
        if (d >= D) continue;
        const uint32_t tot = tot_d[c];
        uint64_t *st = status + (size_t)part * D + d;
        uint32_t excl = 0;
        if (part == 0) {
            st_volatile64(st, epoch | kStP | tot);
        } else {
            st_volatile64(st, epoch | kStA | tot);
            // windowed look-back: kLbWin predecessors per round trip, nearest first
            int q = (int)part - 1;
            bool found = false;
            while (!found) {
                uint64_t w[kLbWin];
#pragma unroll
                for (int k = 0; k < kLbWin; ++k)
                    w[k] = q - k >= 0 ? ld_volatile64(status + (size_t)(q - k) * D + d) : (epoch | kStP);
                int k = 0;
                for (; k < kLbWin; ++k) {
                    const uint64_t sv = w[k];
                    if ((sv & 0xffffffff00000000ull) != epoch || (sv & (3ull << 30)) == 0) break;
                    excl += (uint32_t)(sv & kValMask);
                    if ((sv & (3ull << 30)) == kStP) {
                        found = true;
                        break;
                    }
                }
                q -= k;  // resume at the first unpublished predecessor
            }
            st_volatile64(st, epoch | kStP | (excl + tot));
        }
        s_gofs[d] = __ldg(gbase + d) + excl;
    }
    // local reorder by digit (stable), then contiguous global runs
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        if (dig[k] < (uint32_t)D) {
            const uint32_t li = s_lbase[dig[k]] + s_w[warp][dig[k]] + rk[k];
            s_key[li] = key[k];
            s_val[li] = val[k];
        }
    }
    __syncthreads();
    const uint32_t cnt = min((uint32_t)TILE, n - part * TILE);
    for (uint32_t li = tid; li < cnt; li += kSortThreads) {
        const uint32_t kk = s_key[li], vv = s_val[li];
        const uint32_t d = (kk >> shift) & MASK;
        const uint32_t pos = s_gofs[d] + (li - s_lbase[d]);
        if (keys_out) keys_out[pos] = kk;
        vals_out[pos] = vv;
        if (rect_out) rect_out[pos] = __ldg(rect_in + vv);
    }
    __syncthreads();
    }
}

// Row 5a prologue: digit histograms of the four 8-bit depth passes in one
// read of the keys; the last block turns them into exclusive bases.  Block 0
// also bumps the per-frame look-back epoch.
__global__ void __launch_bounds__(kSortThreads) k_sort_hist(const uint32_t *__restrict__ keys, Counters *ctr,
                                                            uint32_t *__restrict__ ghist, uint32_t *epoch) {
    __shared__ uint32_t h[4][256];
    __shared__ uint32_t s_scan[256];
    __shared__ bool s_last;
    const int tid = threadIdx.x;
    const uint32_t n = ctr->n_vis;
    if (blockIdx.x == 0 && tid == 0) *epoch = *epoch + 1;
#pragma unroll
    for (int p = 0; p < 4; ++p) h[p][tid] = 0;
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + tid; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = __ldg(keys + i);
#pragma unroll
        for (int p = 0; p < 4; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1u);
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < 4; ++p)
        if (h[p][tid]) atomicAdd(&ghist[p * 256 + tid], h[p][tid]);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&ctr->sort_ticket[0], 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int p = 0; p < 4; ++p) {
        const uint32_t c = __ldcg(&ghist[p * 256 + tid]);
        s_scan[tid] = c;
        __syncthreads();
        for (int off = 1; off < 256; off <<= 1) {
            const uint32_t v = tid >= off ? s_scan[tid - off] : 0;
            __syncthreads();
            s_scan[tid] += v;
            __syncthreads();
        }
        ghist[p * 256 + tid] = s_scan[tid] - c;
        __syncthreads();
    }
}

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

// Row 5b (1/6): tile rows per Gaussian (ny of its pixel AABB) in canonical
// order -> their exclusive scan = row-item offsets, and the first Gaussian of
// every row-item chunk.  Three non-blocking passes: k_bin_count (per partition
// of kScanNT Gaussians: the ny total, the band constants of the tile cover and
// the per-tile-row item counts), k_count_scan over the partitions, then
// k_bin_offsets (block scan + partition base).
#ifndef FDGS_ITEM_ILP
#define FDGS_ITEM_ILP 2
#endif
constexpr int kItemIlp = FDGS_ITEM_ILP;  // k_row_items / k_row_count: row items in flight per thread
constexpr int kScanNT = 256;     // threads (= items) per scan partition
constexpr int kItemTile = kScanNT;  // row items per chunk / partition
__global__ void __launch_bounds__(kScanNT) k_bin_count(const uint2 *__restrict__ rects,
                                                       const uint32_t *__restrict__ order,
                                                       const float4 *__restrict__ rec0,
                                                       const float4 *__restrict__ rec1, const Counters *ctrc,
                                                       BandConsts *__restrict__ bconst, int *__restrict__ rowdiff,
                                                       int tiles_y, uint32_t *__restrict__ pcnt) {
    __shared__ int s_rdiff[kMaxTilesY + 1];
    __shared__ uint32_t s_tot;
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t n = ctrc->n_vis;
    const uint32_t parts = (n + kScanNT - 1) / kScanNT;
    for (uint32_t part = blockIdx.x; part < parts; part += gridDim.x) {
        for (int k = tid; k <= tiles_y; k += blockDim.x) s_rdiff[k] = 0;
        if (tid == 0) s_tot = 0;
        __syncthreads();
        const uint32_t i = part * kScanNT + tid;
        uint32_t c = 0;
        if (i < n) {
            const uint2 rc = __ldg(rects + i);
            const TileRect tr = tile_rect(rc);
            c = (uint32_t)tr.ny;
            atomicAdd(&s_rdiff[tr.ty0], 1);  // row-item counts per tile row (1D diff), block-aggregated
            atomicAdd(&s_rdiff[tr.ty0 + tr.ny], -1);
            const uint32_t v = __ldg(order + i);
            const float4 a = __ldg(rec0 + v), b = __ldg(rec1 + v);
            bconst[i] = band_consts(a.x, a.y, a.z, a.w, b.x, b.y, rc.x & 0xffff, rc.x >> 16, rc.y & 0xffff,
                                    rc.y >> 16);
        }
        uint32_t w = c;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (lane == 0 && w) atomicAdd(&s_tot, w);
        __syncthreads();
        for (int k = tid; k <= tiles_y; k += blockDim.x)
            if (s_rdiff[k]) atomicAdd(&rowdiff[k], s_rdiff[k]);
        if (tid == 0) pcnt[part] = s_tot;
        __syncthreads();
    }
}

// Row 5b (1b/6): per partition, the block scan of ny plus the partition's base
// -> the item offset o of Gaussian i; its row items o .. o+ny-1 are expanded
// here (row key ty and owner i), so k_row_items needs no search.
__global__ void __launch_bounds__(kScanNT) k_bin_offsets(const uint2 *__restrict__ rects, const Counters *ctrc,
                                                         const uint32_t *__restrict__ pbase,
                                                         uint32_t *__restrict__ item_key,
                                                         uint32_t *__restrict__ item_owner, uint32_t item_cap) {
    __shared__ uint32_t s_w[kScanNT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n = ctrc->n_vis;
    const uint32_t parts = (n + kScanNT - 1) / kScanNT;
    for (uint32_t part = blockIdx.x; part < parts; part += gridDim.x) {
        const uint32_t i = part * kScanNT + tid;
        const uint32_t c = i < n ? (uint32_t)tile_rect(__ldg(rects + i)).ny : 0u;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_w[warp] = incl;
        __syncthreads();
        uint32_t wbase = __ldg(pbase + part);
        for (int k = 0; k < warp; ++k) wbase += s_w[k];
        if (i < n) {  // expand: row items o .. o+c-1 of Gaussian i (rows ty0 ..), within the capacity
            const uint32_t o = wbase + incl - c;
            const int ty0 = tile_rect(__ldg(rects + i)).ty0;
            for (uint32_t k = 0; k < c && o + k < item_cap; ++k) {
                item_key[o + k] = (uint32_t)(ty0 + (int)k);
                item_owner[o + k] = i;
            }
        }
        __syncthreads();
    }
}

// Row 5b (2/6): one thread per row item (Gaussian r, tile row ty): its tile
// cover [txa, txb] (band_tiles, binary64 pinned), the row key for the stable
// row partition, and the per-row difference array of the per-tile counts.
// Items are in canonical order (Gaussian-major, rows ascending).
__global__ void __launch_bounds__(kScanNT) k_row_items(const uint2 *__restrict__ rects,
                                                       const uint32_t *__restrict__ order,
                                                       const float4 *__restrict__ rec0,
                                                       const float4 *__restrict__ rec1,
                                                       const BandConsts *__restrict__ bconst, const Counters *ctrc,
                                                       const uint32_t *n_items_ptr,
                                                       const uint32_t *__restrict__ item_key,
                                                       uint32_t *__restrict__ item_pack, uint32_t *__restrict__ item_v,
                                                       uint32_t item_cap) {
    const uint32_t ni = *n_items_ptr;
    // the row partition (next launches) processes n_items_part items: n_items
    // when they fit the workspace, else none (the frame is then OVERFLOW and
    // nothing writes past the item / look-back buffers sized by the capacity)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        Counters *c = const_cast<Counters *>(ctrc);
        c->n_items_part = ni <= item_cap ? ni : 0u;
        if (ni > item_cap) c->status = FDGS_ERR_OVERFLOW;
    }
    if (ni > item_cap) return;  // more row items than the workspace holds
    // kItemIlp items per thread and iteration, their three levels of dependent
    // loads (item -> Gaussian -> record) issued together: the kernel is bound
    // by the latency of those gathers, not by the band arithmetic
    constexpr int U = kItemIlp;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < ni; i0 += U * stride) {
        uint32_t r[U], v[U];
        int ty[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = i0 + u * stride < ni ? i0 + u * stride : i0;  // past the end: this thread's own first item again, not stored
            r[u] = __ldg(item_v + i);  // owning Gaussian (canonical rank), from k_bin_offsets
            ty[u] = (int)__ldg(item_key + i);
        }
        uint2 rc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            rc[u] = __ldg(rects + r[u]);
            v[u] = __ldg(order + r[u]);
        }
        float4 a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a[u] = __ldg(rec0 + v[u]);
            b[u] = __ldg(rec1 + v[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = i0 + u * stride;
            if (i >= ni) break;
            const int px0 = rc[u].x & 0xffff, px1 = rc[u].x >> 16, py0 = rc[u].y & 0xffff, py1 = rc[u].y >> 16;
            int txa, txb;
            uint32_t pack = 0u;  // empty row: txb + 1 <= txa
            if (band_tiles(bconst[r[u]], a[u].x, a[u].y, a[u].z, a[u].w, b[u].x, px0, px1, py0, py1, ty[u], txa, txb))
                pack = (uint32_t)txa | ((uint32_t)(txb + 1) << 16);
            item_pack[i] = pack;
            item_v[i] = v[u];  // the owner index is replaced by the record slot
        }
    }
}

// Row 5b (3/6), one warp: prefix of the row-item difference array ->
// row_start[0..tiles_y] and the exclusive digit bases of the row partition
// passes (digit ty & 255, then ty >> 8).
__global__ void k_row_scan(const int *__restrict__ rowdiff, int tiles_y, uint32_t *__restrict__ row_start,
                           uint32_t *__restrict__ rbase) {
    __shared__ uint32_t s_rows[kMaxTilesY + 1];
    const int lane = threadIdx.x;  // one warp
    // items per row = prefix of the difference array; row starts = prefix of the items
    int run = 0;
    uint32_t start = 0;
    for (int y0 = 0; y0 < tiles_y; y0 += 32) {
        const int y = y0 + lane;
        int d = y < tiles_y ? __ldcg(rowdiff + y) : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, d, o);
            if (lane >= o) d += t;
        }
        const uint32_t items = (uint32_t)(run + d);
        uint32_t inc = y < tiles_y ? items : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (y < tiles_y) {
            s_rows[y] = items;
            row_start[y] = start + inc - items;
        }
        run += __shfl_sync(0xffffffffu, d, 31);
        start += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) row_start[tiles_y] = start;
    __syncwarp();
    // digit bases of the row partition: pass 0 digit = ty & 255, pass 1 digit = ty >> 8
    uint32_t hi1 = 0;
    for (int y = lane; y < min(tiles_y, 256); y += 32) hi1 += s_rows[y];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hi1 += __shfl_xor_sync(0xffffffffu, hi1, o);
    uint32_t acc = 0;
    for (int d0 = 0; d0 < 256; d0 += 32) {
        const int d = d0 + lane;
        const uint32_t c = (d < tiles_y ? s_rows[d] : 0u) + (d + 256 < tiles_y ? s_rows[d + 256] : 0u);
        uint32_t inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        rbase[d] = acc + inc - c;
        acc += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
        rbase[256] = 0;
        rbase[257] = hi1;
    }
}

// Row 5b (5/6), one block: per-tile entry counts (summed over the row
// segments by k_row_count) -> tile_start[0..T] and E (capacity check before
// the scatter writes any entry).
__global__ void __launch_bounds__(1024) k_tile_scan(const uint32_t *__restrict__ tile_cnt, int tiles_x, int tiles_y,
                                                    uint32_t *__restrict__ tile_start, Counters *ctr,
                                                    int64_t max_entries) {
    __shared__ uint32_t s_sum[1024];
    const int tid = threadIdx.x;
    const int T = tiles_x * tiles_y;
    const int chunk = (T + 1023) / 1024;
    const int k0 = min(tid * chunk, T), k1 = min(k0 + chunk, T);
    auto count = [&](int k) { return __ldcg(tile_cnt + k); };
    uint32_t local = 0;
    for (int k = k0; k < k1; ++k) local += count(k);
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
        run += count(k);
    }
    if (tid == 1023) {
        const uint32_t E = s_sum[1023];
        tile_start[T] = E;
        ctr->n_entries = E;
        if ((int64_t)E > max_entries) ctr->status = FDGS_ERR_OVERFLOW;
        else if (ctr->status == FDGS_OK) ctr->n_sort_entries = E;
    }
}

// Row 5b (5/6 and 6/6): per tile row, the stable scatter of its row items'
// entries into the row's tiles.  The row's items (canonical order after the
// stable row partition) are split into kRowSeg segments, one block each, and
// each warp walks a contiguous run of them: 32 (item, tile) entries per round
// in canonical order, ranked within the round by match_any on the tile, with
// warp-private per-tile counters carrying the count across rounds.
#ifndef FDGS_ROW_WARPS
#define FDGS_ROW_WARPS 2
#endif
constexpr int kRowWarps = FDGS_ROW_WARPS;

template <bool kWrite>
__device__ __forceinline__ void row_walk(uint32_t w0, uint32_t w1, int lane, const uint32_t *__restrict__ sorted,
                                         const uint32_t *__restrict__ item_pack,
                                         const uint32_t *__restrict__ item_v, uint32_t *cnt, const uint32_t *base,
                                         uint32_t *__restrict__ entries, uint8_t *s_own) {
    for (uint32_t r0 = w0; r0 < w1; r0 += 32) {
        const uint32_t r = r0 + lane;
        int c = 0, txa = 0;
        uint32_t v = 0;
        if (r < w1) {
            const uint32_t it = __ldg(sorted + r);
            const uint32_t pk = __ldg(item_pack + it);
            txa = (int)(pk & 0xffffu);
            c = max((int)(pk >> 16) - txa, 0);
            if (kWrite) v = __ldg(item_v + it);
        }
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int e0 = 0; e0 < total; e0 += 32) {
            const int e = e0 + lane;
            // owning item of entry e: every item with entries in [e0, e0 + 32)
            // marks the window slot where its run starts; the owner of slot
            // e - e0 is the run starting at the highest mark <= it
            const int ex = incl - c;
            const bool owns = c > 0 && ex < e0 + 32 && incl > e0;
            const int slot = max(ex, e0) - e0;
            const uint32_t marks = __reduce_or_sync(0xffffffffu, owns ? 1u << slot : 0u);
            if (owns) s_own[slot] = (uint8_t)lane;
            __syncwarp();
            const int j = s_own[31 - __clz(marks & ((2u << lane) - 1u))];
            const int exj = __shfl_sync(0xffffffffu, incl - c, j);
            const int jx = __shfl_sync(0xffffffffu, txa, j);
            const uint32_t vj = __shfl_sync(0xffffffffu, v, j);
            const bool valid = e < total;
            const uint32_t tx = valid ? (uint32_t)(jx + (e - exj)) : 0xffffffffu;
            const uint32_t peers = __match_any_sync(0xffffffffu, tx);
            const bool leader = (__ffs(peers) - 1) == lane;
            if (kWrite && valid) entries[base[tx] + cnt[tx] + __popc(peers & lanemask_lt())] = vj;
            __syncwarp();
            if (valid && leader) cnt[tx] += __popc(peers);
            __syncwarp();
        }
    }
}

__device__ __forceinline__ void row_seg_range(const uint32_t *row_start, int ty, int seg, uint32_t &lo,
                                              uint32_t &hi) {
    const uint32_t a = __ldg(row_start + ty), b = __ldg(row_start + ty + 1);
    const uint32_t per = (b - a + kRowSeg - 1) / kRowSeg;
    lo = min(a + seg * per, b);
    hi = min(lo + per, b);
}

// Row 5b (5/6) per (row, segment): the segment's entry count per tile ->
// hist[ty][seg][tx], from a shared-memory difference array over the row's
// tiles (2 shared atomics per row item)
#ifndef FDGS_ROWCNT_THREADS
#define FDGS_ROWCNT_THREADS 256
#endif
__global__ void __launch_bounds__(FDGS_ROWCNT_THREADS) k_row_count(const uint32_t *__restrict__ sorted,
                                                   const uint32_t *__restrict__ item_pack,
                                                   const uint32_t *__restrict__ row_start, int tiles_x,
                                                   uint32_t *__restrict__ hist, uint32_t *__restrict__ tile_cnt,
                                                   const Counters *ctrc) {
    extern __shared__ int s_d[];  // [tiles_x + 1]
    const int ty = blockIdx.x / kRowSeg, seg = blockIdx.x % kRowSeg;
    const int tid = threadIdx.x;
    if (ctrc->status != FDGS_OK) return;
    for (int k = tid; k <= tiles_x; k += blockDim.x) s_d[k] = 0;
    __syncthreads();
    uint32_t lo, hi;
    row_seg_range(row_start, ty, seg, lo, hi);
    constexpr int U = kItemIlp;  // items in flight per thread (their two dependent loads issued together)
    for (uint32_t r0 = lo + tid; r0 < hi; r0 += U * blockDim.x) {
        uint32_t it[U], pk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) it[u] = __ldg(sorted + min(r0 + u * blockDim.x, hi - 1));
#pragma unroll
        for (int u = 0; u < U; ++u) pk[u] = __ldg(item_pack + it[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int txa = (int)(pk[u] & 0xffffu), txe = (int)(pk[u] >> 16);
            if (r0 + u * blockDim.x < hi && txe > txa) {
                atomicAdd(&s_d[txa], 1);
                atomicAdd(&s_d[txe], -1);
            }
        }
    }
    __syncthreads();
    if (tid < 32) {  // prefix over the row's tiles, one warp
        int run = 0;
        for (int x0 = 0; x0 < tiles_x; x0 += 32) {
            const int x = x0 + tid;
            int val = x < tiles_x ? s_d[x] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, val, o);
                if (tid >= o) val += t;
            }
            if (x < tiles_x) {
                hist[((size_t)ty * kRowSeg + seg) * tiles_x + x] = (uint32_t)(run + val);
                if (run + val) atomicAdd(&tile_cnt[ty * tiles_x + x], (uint32_t)(run + val));  // per-tile total
            }
            run += __shfl_sync(0xffffffffu, val, 31);
        }
    }
}

// Row 5b (6/6) per (row, segment): global base of every tile (tile_start +
// earlier segments + earlier warps), then the warp-ordered scatter of entries
__global__ void __launch_bounds__(32 * kRowWarps) k_row_scatter(const uint32_t *__restrict__ sorted,
                                                                const uint32_t *__restrict__ item_pack,
                                                                const uint32_t *__restrict__ item_v,
                                                                const uint32_t *__restrict__ row_start, int tiles_x,
                                                                const uint32_t *__restrict__ hist,
                                                                const uint32_t *__restrict__ tile_start,
                                                                uint32_t *__restrict__ entries, const Counters *ctrc) {
    extern __shared__ uint32_t s_mem[];  // [kRowWarps][tiles_x] counters, then [tiles_x] base
    uint32_t *s_cnt = s_mem, *s_base = s_mem + kRowWarps * tiles_x;
    const int ty = blockIdx.x / kRowSeg, seg = blockIdx.x % kRowSeg;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (ctrc->status != FDGS_OK) return;
    for (int k = tid; k < kRowWarps * tiles_x; k += blockDim.x) s_cnt[k] = 0;
    __syncthreads();
    uint32_t lo, hi;
    row_seg_range(row_start, ty, seg, lo, hi);
    const uint32_t per = (hi - lo + kRowWarps - 1) / kRowWarps;
    const uint32_t w0 = min(lo + warp * per, hi), w1 = min(w0 + per, hi);
    uint32_t *my = s_cnt + warp * tiles_x;
    // per-warp tile counts: difference array over the warp's items (2 shared
    // atomics per item), then a per-warp prefix over the row's tiles
    int *md = reinterpret_cast<int *>(my);
    for (uint32_t r = w0 + lane; r < w1; r += 32) {
        const uint32_t pk = __ldg(item_pack + __ldg(sorted + r));
        const int txa = (int)(pk & 0xffffu), txe = (int)(pk >> 16);
        if (txe > txa) {
            atomicAdd(&md[txa], 1);
            if (txe < tiles_x) atomicAdd(&md[txe], -1);
        }
    }
    __syncwarp();
    {
        int run = 0;
        for (int x0 = 0; x0 < tiles_x; x0 += 32) {
            const int x = x0 + lane;
            int val = x < tiles_x ? md[x] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, val, o);
                if (lane >= o) val += t;
            }
            if (x < tiles_x) md[x] = run + val;
            run += __shfl_sync(0xffffffffu, val, 31);
        }
    }
    __syncthreads();
    for (int x = tid; x < tiles_x; x += blockDim.x) {
        uint32_t b = __ldg(tile_start + ty * tiles_x + x);
        for (int sg = 0; sg < seg; ++sg) b += __ldg(hist + ((size_t)ty * kRowSeg + sg) * tiles_x + x);
        s_base[x] = b;
        uint32_t run = 0;
        for (int w = 0; w < kRowWarps; ++w) {
            const uint32_t c = s_cnt[w * tiles_x + x];
            s_cnt[w * tiles_x + x] = run;
            run += c;
        }
    }
    __syncthreads();
    __shared__ uint8_t s_own[kRowWarps][32];  // run-start owner per window slot (row_walk)
    row_walk<true>(w0, w1, lane, sorted, item_pack, item_v, my, s_base, entries, s_own[warp]);
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

// Stage one splat record for the tile.  Besides the pixel-AABB mask (the
// per-pixel decision), a refined row mask culls whole warps: row r is kept only
// if the ellipse {e2 >= -margin} reaches the row's segment of pixel centres
// (the concave quadratic's maximum over the segment, at the clamped argmax).
// This is pure culling: the margin (1e-3 relative to the quadratic's
// magnitude, + 1e-3) exceeds the rounding of both this test and the pinned
// fp32 e2 chain, so no pixel with e2 >= 0 is dropped.
__device__ __forceinline__ void stage_fields(int tx, int ty, const float4 &r0, const float4 &r1, const float4 &r2,
                                             float4 &oa, float4 &oc, float4 &od) {
    const uint32_t ax = __float_as_uint(r1.z), ay = __float_as_uint(r1.w);
    const int x0 = max((int)(ax & 0xffff) - tx * 16, 0), x1 = min((int)(ax >> 16) - tx * 16, 15);
    const int y0 = max((int)(ay & 0xffff) - ty * 16, 0), y1 = min((int)((ay >> 16) & 0x7fffu) - ty * 16, 15);
    const uint32_t xm = ((2u << x1) - 1u) & ~((1u << x0) - 1u);
    const uint32_t ym = ((2u << y1) - 1u) & ~((1u << y0) - 1u);
    uint32_t yr = 0;
    const float u = r0.x, v = r0.y, Ap = r0.z, Bp = r0.w, Cp = r1.x, Q2 = r1.y;
    const float dxl = (float)(tx * 16 + x0) + 0.5f - u, dxr = (float)(tx * 16 + x1) + 0.5f - u;
    const float dxm = fmaxf(fabsf(dxl), fabsf(dxr));
    const float hA = -0.5f / Ap;  // A' < 0
    for (int r = y0; r <= y1; ++r) {
        const float dy = (float)(ty * 16 + r) + 0.5f - v;
        const float dx = fminf(fmaxf(Bp * dy * hA, dxl), dxr);
        const float f = fmaf(dx, fmaf(Ap, dx, Bp * dy), fmaf(Cp * dy, dy, Q2));
        const float mag = fabsf(Ap) * dxm * dxm + fabsf(Bp) * dxm * fabsf(dy) + fabsf(Cp) * dy * dy;
        if (f >= -(1e-3f * mag + 1e-3f)) yr |= 1u << r;
    }
    oa = r0;
    oc = make_float4(r1.x, r1.y, r2.x, r2.y);
    od = make_float4(r2.z, __uint_as_float(~(xm | (ym << 16))), __uint_as_float(yr << 16), r2.w);  // .w: gid bits
}

__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    float2 d;
    asm("mul.rn.f32x2 %0, %1, %2;"
        : "=l"(*reinterpret_cast<unsigned long long *>(&d))
        : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)));
    return d;
}


// Warp-specialised blend: one producer warp stages records 32 at a time into
// a ring of kWsBuf shared-memory batches (gathers + the row-culling mask), four
// consumer warps composite them.  Full/empty mbarriers replace block-wide
// barriers, so consumer warps drift independently; a consumer whose pixels
// have all terminated keeps releasing batches without computing, and the
// producer stops once all four are done.  Pixel mapping and arithmetic are
// those of k_blend_wi; this kernel visits every record of the tile (for the
// Eq. 2 work counters) and records contributions (fdgs_stv_score).
constexpr int kWsBuf = 6;
// fl(x * kInv255) is monotone in x and equals 0.99f exactly for one float,
// kAlphaPre = 252.44998f (0x437c7332), so min(0.99f, fl(x * kInv255)) ==
// fl(min(x, kAlphaPre) * kInv255) for every x >= 0 (checked exhaustively
// over [128, 256) by tests/test_host_logic.py).
constexpr float kInv255 = 1.0f / 255.0f;
constexpr float kAlphaPre = 0x1.f8e664p+7f;  // 252.44998f
constexpr int kWsThreads = 160;
struct WsBatch {
    float4 a[32], c[32], d[32];
};

__device__ __forceinline__ void mb_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mb_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t addr = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}

// kContrib (Sec. 4.2.1 spatial score): additionally records, per
// Gaussian, the sum over the tile's pixels of its blending weight
// w = alpha_i prod_{j<i}(1 - alpha_j) -- exactly the weight the composite
// uses.  Weights are rounded to fixed point (2^-24, error <= 2^-25 per pixel)
// and summed as integers: each consumer warp reduces its 64 pixels with
// REDUX into its own shared slot, the producer adds the four slots of a
// released batch and issues one 64-bit global atomic per (tile, Gaussian), so
// the per-Gaussian totals are independent of scheduling (deterministic).
constexpr float kContribScale = 16777216.0f;  // 2^24
template <bool kCount, bool kContrib = false>
__global__ void __launch_bounds__(kWsThreads) k_blend_ws(const uint32_t *__restrict__ tile_start,
                                                         const uint32_t *__restrict__ entries,
                                                         const float4 *__restrict__ rec0,
                                                         const float4 *__restrict__ rec1,
                                                         const float4 *__restrict__ rec2, Counters *ctr, int tiles_x,
                                                         int width, int height, float bg0, float bg1, float bg2,
                                                         float *__restrict__ out_rgb, float *__restrict__ out_T,
                                                         fdgs_frame_stats *stats,
                                                         unsigned long long *__restrict__ contrib = nullptr,
                                                         uint32_t *stv_info = nullptr) {
    __shared__ WsBatch sb[kWsBuf];
    __shared__ uint32_t s_n[kWsBuf];
    __shared__ uint32_t s_rel[kWsBuf][4];  // per consumer warp: records whose ellipse reaches its rows
    __shared__ uint32_t s_acc[kContrib ? kWsBuf : 1][4][32];
    __shared__ __align__(8) uint64_t full[kWsBuf], empty[kWsBuf];
    __shared__ uint32_t s_done;
    __shared__ bool s_last;
    const bool ok = ctr->status == FDGS_OK;
    const int tile = blockIdx.x, tx = tile % tiles_x, ty = tile / tiles_x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t start = __ldg(tile_start + tile), end = __ldg(tile_start + tile + 1);
    if (tid == 0) {
        for (int b = 0; b < kWsBuf; ++b) {
            mb_init(&full[b], 1);
            mb_init(&empty[b], 4);
        }
        s_done = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t first = ok ? start : end;
    if (warp == 4) {  // ------------------------------------------------ producer
        // kContrib: flush the four consumer sums of a released batch slot
        auto flush = [&](int b) {
            if (lane < (int)s_n[b]) {
                const unsigned long long tot = (unsigned long long)s_acc[b][0][lane] + s_acc[b][1][lane] +
                                               s_acc[b][2][lane] + s_acc[b][3][lane];
                if (tot) atomicAdd(contrib + __float_as_uint(sb[b].d[lane].w), tot);
            }
        };
        if (kContrib && tid == 128 && stv_info != nullptr) {  // frame status / entry count for the caller
            if (!ok) atomicMax(&stv_info[0], ctr->status);
            atomicMax(&stv_info[1], ctr->n_entries);
        }
        uint32_t k = 0;
        for (uint32_t base = first;; base += 32, ++k) {
            const int b = (int)(k % kWsBuf);
            if (k >= kWsBuf) {
                mb_wait(&empty[b], ((k / kWsBuf) - 1) & 1);
                if (kContrib) flush(b);
            }
            const bool stop = base >= end || *(volatile uint32_t *)&s_done == 4;
            const uint32_t n = stop ? 0u : min(32u, end - base);
            uint32_t rows = 0;
            if (lane < (int)n) {
                const uint32_t v = __ldg(entries + base + lane);
                const float4 r0 = __ldg(rec0 + v), r1 = __ldg(rec1 + v), r2 = __ldg(rec2 + v);
                float4 oa, oc, od;
                stage_fields(tx, ty, r0, r1, r2, oa, oc, od);
                sb[b].a[lane] = oa;
                sb[b].c[lane] = oc;
                sb[b].d[lane] = od;
                rows = __float_as_uint(od.z);
                if (kContrib) s_acc[b][0][lane] = s_acc[b][1][lane] = s_acc[b][2][lane] = s_acc[b][3][lane] = 0u;
            }
#pragma unroll
            for (int w = 0; w < 4; ++w) {  // record lists per consumer warp (rows 4w..4w+3)
                const uint32_t rel = __ballot_sync(0xffffffffu, (rows >> (16 + 4 * w)) & 0xFu);
                if (lane == w) s_rel[b][w] = rel;
            }
            if (lane == 0) s_n[b] = n;
            __syncwarp();
            if (lane == 0) mb_arrive(&full[b]);
            if (n == 0) {
                if (kContrib)  // batches still in flight: wait for their release, then flush
                    for (uint32_t kk = k >= kWsBuf - 1 ? k - (kWsBuf - 1) : 0; kk < k; ++kk) {
                        mb_wait(&empty[kk % kWsBuf], (kk / kWsBuf) & 1);
                        flush((int)(kk % kWsBuf));
                    }
                break;
            }
        }
    } else {  // --------------------------------------------------------- consumers
        const int ly = tid >> 3, lx = (tid & 7) * 2;
        const int i0 = tx * 16 + lx, j = ty * 16 + ly;
        const bool in0 = i0 < width && j < height, in1 = i0 + 1 < width && j < height;
        float pyf = (float)j + 0.5f;
        float2 px = make_float2((float)i0 + 0.5f, (float)(i0 + 1) + 0.5f);
        const uint32_t pb0 = (1u << lx) | (1u << (16 + ly)), pb1 = (2u << lx) | (1u << (16 + ly));
        const float kInf = __int_as_float(0x7f800000);
        float2 thr = make_float2(in0 ? 0.0f : kInf, in1 ? 0.0f : kInf);
        float2 T = make_float2(1.0f, 1.0f), Cr = make_float2(0.f, 0.f), Cg = Cr, Cb = Cr;
        uint32_t n_eval = 0, n_blend = 0;
        bool wdone = false;
        for (uint32_t k = 0;; ++k) {
            const int b = (int)(k % kWsBuf);
            mb_wait(&full[b], (k / kWsBuf) & 1);
            const int cnt = (int)s_n[b];
            if (cnt == 0) break;
            if (!wdone) {
                const WsBatch &B = sb[b];
                const uint32_t rel = s_rel[b][warp];
                // kCount visits every record (its Eq. 2 work count includes the pairs of
                // records whose ellipse misses this warp's rows); otherwise only the
                // records of this warp's list
                for (uint32_t it = kCount ? (cnt == 32 ? ~0u : (1u << cnt) - 1u) : rel; it != 0u; it &= it - 1u) {
                    const int q = __ffs(it) - 1;
                    const float4 dq = B.d[q];
                    const uint32_t m = __float_as_uint(dq.y);
                    if (kCount) {
                        n_eval += (uint32_t)((m & pb0) == 0u && thr.x == 0.0f) +
                                  (uint32_t)((m & pb1) == 0u && thr.y == 0.0f);
                        if (((rel >> q) & 1u) == 0u) continue;
                    }
                    const float4 a = B.a[q];
                    const float4 c = B.c[q];
                    // keep the pixel centres live in registers (the compiler otherwise
                    // rematerialises them from the indices in every iteration)
                    asm volatile("" : "+f"(pyf), "+f"(px.x), "+f"(px.y));
                    const float dy = __fsub_rn(pyf, a.y);
                    const float t1 = __fmul_rn(a.w, dy);
                    const float t3 = __fmul_rn(c.x, dy);
                    const float t4 = __fmaf_rn(t3, dy, c.y);
                    const float2 dx = sub2(px, make_float2(a.x, a.x));
                    const float2 t2 = fma2(make_float2(a.z, a.z), dx, make_float2(t1, t1));
                    const float2 e2 = fma2(dx, t2, make_float2(t4, t4));
                    const bool v0 = (m & pb0) == 0u && e2.x >= thr.x, v1 = (m & pb1) == 0u && e2.y >= thr.y;
                    // branch-free body (a skip costs more issue slots than the ~10% of
                    // records with no eligible lane save); kContrib skips warp-uniformly
                    // since its REDUX needs the whole warp
                    if (kContrib && !__any_sync(0xffffffffu, v0 || v1)) continue;
                    // alpha = min(0.99, 2^e2 * (1/255)) computed as min(2^e2, kAlphaPre) * (1/255)
                    // (one packed multiply; bit-identical, see kAlphaPre)
                    const float m0 = v0 ? fminf(ex2_approx(e2.x), kAlphaPre) : 0.0f;
                    const float m1 = v1 ? fminf(ex2_approx(e2.y), kAlphaPre) : 0.0f;
                    float2 w = mul2(mul2(make_float2(m0, m1), make_float2(kInv255, kInv255)), T);
                    const float2 test = sub2(T, w);
                    const bool s0 = v0 && test.x < 1e-4f, s1 = v1 && test.y < 1e-4f;
                    w.x = s0 ? 0.0f : w.x;
                    w.y = s1 ? 0.0f : w.y;
                    thr.x = s0 ? kInf : thr.x;
                    thr.y = s1 ? kInf : thr.y;
                    if (kCount) n_blend += (uint32_t)(v0 && !s0) + (uint32_t)(v1 && !s1);
                    T = sub2(T, w);
                    Cr = fma2(make_float2(c.z, c.z), w, Cr);
                    Cg = fma2(make_float2(c.w, c.w), w, Cg);
                    Cb = fma2(make_float2(dq.x, dq.x), w, Cb);
                    if (kContrib) {  // S^S term alpha_i prod_{j<i}(1 - alpha_j) of P:251, this warp's 64 pixels
                        const uint32_t f = __float2uint_rn(w.x * kContribScale) + __float2uint_rn(w.y * kContribScale);
                        const uint32_t sum = __reduce_add_sync(0xffffffffu, f);
                        if (lane == 0) s_acc[b][warp][q] = sum;
                    }
                }
                wdone = __all_sync(0xffffffffu, thr.x == kInf && thr.y == kInf);
                if (wdone && lane == 0) atomicAdd(&s_done, 1u);
            }
            __syncwarp();
            if (lane == 0) mb_arrive(&empty[b]);
        }
        if (kCount) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                n_eval += __shfl_xor_sync(0xffffffffu, n_eval, o);
                n_blend += __shfl_xor_sync(0xffffffffu, n_blend, o);
            }
            if (lane == 0 && n_eval) {
                atomicAdd(&ctr->n_eval, (unsigned long long)n_eval);
                atomicAdd(&ctr->n_blend, (unsigned long long)n_blend);
            }
        }
        if (ok && out_rgb != nullptr) {
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
    }
    if (kCount) {
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
}

// Per-warp record lists of the timed blend (k_blend_wi): for each record of
// the tile whose quadratic reaches one of the warp's four rows (per-row
// maximum over the tile's pixel-centre columns, with a margin), the common
// 16 bytes {u, A', r, g} and, per row of the warp, {b, ~AABB mask, t1, t4}:
// the row terms of the pinned e2 chain (dy, t1 = B' dy, t3 = C' dy,
// t4 = fma(t3, dy, Q2)), evaluated once per (record, row).
//
// Footprint of consumer warp w in the tile: 4 rows x 16 columns (a strip).
constexpr int kWlRows = 4, kWlCols = 16;
__host__ __device__ constexpr int wl_row0(int w) { return 4 * w; }
__host__ __device__ constexpr int wl_col0(int w) { return 0; }

// Two 16-byte loads per record for a consumer thread: the common part and its
// row's part (colour b and the mask repeated per row).
struct WlEntry {
    float4 a;            // u, A', r, g
    float4 t[kWlRows];   // per row of the warp: b, ~AABB mask bits, t1, t4
};
static_assert(sizeof(WlEntry) == 16 + 16 * kWlRows, "WlEntry layout");

#ifndef FDGS_WL_UNROLL
#define FDGS_WL_UNROLL 4
#endif
constexpr int kWlUnroll = FDGS_WL_UNROLL;
constexpr float kStopU = 1e-4f / 255.0f;  // the stop threshold 1e-4 on T, on U = T / 255
// Stage one record for warp strip `warp` (rows 4w..4w+3) of tile (tx, ty)
// (k_blend_wi): the complemented pixel-AABB mask mb, the pinned e2 row terms
// {b, mb, t1, t4} of the strip's rows (DESIGN.md §3 step 10), and whether the
// record reaches the strip.  Reach: for some row of the strip inside the
// AABB, the maximum over the tile ∩ AABB pixel-centre columns of the row's
// quadratic x (A' x + t1) + t4 (the consumer's own chain, at the stationary
// point clamped to the columns) is >= -margin, margin = 1e-3 |quadratic| +
// 1e-3 over the tile ∩ AABB -- well above the rounding of this test and of the
// pinned fp32 chain, so no pixel with e2 >= 0 is dropped (pure culling;
// brute-force soundness test: tests/test_gpu_fullsize.py).  Explicit IEEE
// intrinsics throughout, so every inlined copy takes the same decisions
// (fdgs_debug_strip_reach replays it).
template <int ROWS>
__device__ __forceinline__ bool strip_stage(const float4 &r0, const float4 &r1, float b, int tx, int ty, int row0,
                                            const float (&rowc)[ROWS], uint32_t &mb, float (&t1s)[ROWS],
                                            float (&t4s)[ROWS]) {
    const float u = r0.x, v = r0.y, Ap = r0.z, Bp = r0.w, Cp = r1.x, Q2 = r1.y;
    const uint32_t ax = __float_as_uint(r1.z), ay = __float_as_uint(r1.w);
    const int x0 = max((int)(ax & 0xffff) - tx * 16, 0), x1 = min((int)(ax >> 16) - tx * 16, 15);
    const int y0 = max((int)(ay & 0xffff) - ty * 16, 0);
    const int y1 = x0 > x1 ? -1 : min((int)((ay >> 16) & 0x7fffu) - ty * 16, 15);
    const uint32_t xm = ((2u << x1) - 1u) & ~((1u << x0) - 1u);
    const uint32_t ym = ((2u << y1) - 1u) & ~((1u << y0) - 1u);
    mb = ~(xm | (ym << 16));
    const float xl = __fsub_rn((float)(tx * 16 + x0) + 0.5f, u);
    const float xr = __fsub_rn((float)(tx * 16 + x1) + 0.5f, u);
    const float yl = __fsub_rn((float)(ty * 16 + y0) + 0.5f, v), yr = __fsub_rn((float)(ty * 16 + y1) + 0.5f, v);
    const float X = fmaxf(fabsf(xl), fabsf(xr)), Y = fmaxf(fabsf(yl), fabsf(yr));
    const float mag = __fmaf_rn(__fmul_rn(fabsf(Ap), X), X,
                                __fmaf_rn(__fmul_rn(fabsf(Bp), X), Y, __fmul_rn(__fmul_rn(fabsf(Cp), Y), Y)));
    const float marg = -__fmaf_rn(1e-3f, mag, 1e-3f);
    const float hA = __fdividef(-0.5f, Ap);  // stationary point only
    bool rw = false;
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {  // pinned e2 chain, row terms (DESIGN.md step 10)
        const int row = row0 + r;
        const float dy = __fsub_rn(rowc[r], v);  // rowc[r] = pixel-centre y of the strip's row r
        const float t1 = __fmul_rn(Bp, dy);
        const float t3 = __fmul_rn(Cp, dy);
        const float t4 = __fmaf_rn(t3, dy, Q2);
        const float xs = fminf(fmaxf(__fmul_rn(t1, hA), xl), xr);
        rw |= row >= y0 && row <= y1 && __fmaf_rn(xs, __fmaf_rn(Ap, xs, t1), t4) >= marg;
        t1s[r] = t1;
        t4s[r] = t4;
    }
    (void)b;
    return rw;
}

constexpr int kBlendRows = kWlRows;  // strip height of the timed blend (k_blend_wi)

// Tests: the strip-reach decisions of every entry of the frame last rendered
// in the workspace (bit w of out[k]: entry k is staged for warp strip w).
__global__ void __launch_bounds__(128) k_debug_strip_reach(const uint32_t *__restrict__ tile_start,
                                                           const uint32_t *__restrict__ entries,
                                                           const float4 *__restrict__ rec0,
                                                           const float4 *__restrict__ rec1, const Counters *ctr,
                                                           int tiles_x, uint8_t *__restrict__ out) {
    if (ctr->status != FDGS_OK) return;
    const int tile = blockIdx.x, tx = tile % tiles_x, ty = tile / tiles_x;
    const uint32_t start = tile_start[tile], end = tile_start[tile + 1];
    for (uint32_t k = start + threadIdx.x; k < end; k += blockDim.x) {
        const uint32_t v = entries[k];
        const float4 r0 = rec0[v], r1 = rec1[v];
        uint32_t bits = 0, mb;
        constexpr int R = kBlendRows;  // strip height of the timed blend
        float t1s[R], t4s[R];
        for (int w = 0; w < 16 / R; ++w) {
            float rowc[R];
            for (int r = 0; r < R; ++r) rowc[r] = (float)(ty * 16 + R * w + r) + 0.5f;
            if (strip_stage<R>(r0, r1, 0.0f, tx, ty, R * w, rowc, mb, t1s, t4s)) bits |= ((1u << (R / 4)) - 1u) << (w * R / 4);
        }
        out[k] = (uint8_t)bits;
    }
}

cudaError_t launch_debug_strip_reach(char *ws, const RenderLayout &L, uint8_t *out, cudaStream_t st) {
    k_debug_strip_reach<<<L.n_tiles, 128, 0, st>>>(reinterpret_cast<const uint32_t *>(ws + L.tile_start),
                                                   reinterpret_cast<const uint32_t *>(ws + L.entries),
                                                   reinterpret_cast<const float4 *>(ws + L.rec0),
                                                   reinterpret_cast<const float4 *>(ws + L.rec1),
                                                   reinterpret_cast<const Counters *>(ws + L.counters), L.tiles_x,
                                                   out);
    return cudaGetLastError();
}

// Warp-independent blend (the timed kernel): no producer warp and no barriers
// between warps.  Each of the 4 warps of a tile block stages its own batches of
// 32 records (one per lane: the gather, the AABB mask, the per-row reach test
// and the pinned row terms of its 4-row strip) into a private shared list,
// then composites it; the next batch's records are gathered into registers
// while the current list is composited.
#ifndef FDGS_WI_MINB
#define FDGS_WI_MINB 8
#endif
#ifndef FDGS_WI_PAIR_UNROLL
#define FDGS_WI_PAIR_UNROLL 4
#endif
constexpr int kWiPairUnroll = FDGS_WI_PAIR_UNROLL;

constexpr int kWiThreads = 128;
__global__ void __launch_bounds__(kWiThreads, FDGS_WI_MINB) k_blend_wi(const uint32_t *__restrict__ tile_start,
                                                         const uint32_t *__restrict__ entries,
                                                         const float4 *__restrict__ rec0,
                                                         const float4 *__restrict__ rec1,
                                                         const float4 *__restrict__ rec2, const Counters *ctr,
                                                         int tiles_x, int width, int height, float bg0, float bg1,
                                                         float bg2, float *__restrict__ out_rgb,
                                                         float *__restrict__ out_T) {
    __shared__ WlEntry s_list[4][32];
    const bool ok = ctr->status == FDGS_OK;
    const int tile = blockIdx.x, tx = tile % tiles_x, ty = tile / tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t start = __ldg(tile_start + tile), end = ok ? __ldg(tile_start + tile + 1) : start;
    // consumer geometry: 2 horizontally adjacent pixels per thread
    const int rr = lane / (kWlCols / 2), ly = wl_row0(warp) + rr, lx = wl_col0(warp) + (lane % (kWlCols / 2)) * 2;
    const int i0 = tx * 16 + lx, j = ty * 16 + ly;
    const bool in0 = i0 < width && j < height, in1 = i0 + 1 < width && j < height;
    float2 px = make_float2((float)i0 + 0.5f, (float)(i0 + 1) + 0.5f);
    const uint32_t pb0 = (1u << lx) | (1u << (16 + ly)), pb1 = (2u << lx) | (1u << (16 + ly));
    const float kInf = __int_as_float(0x7f800000);
    float2 thr = make_float2(in0 ? 0.0f : kInf, in1 ? 0.0f : kInf);
    float2 T = make_float2(kInv255, kInv255), Cr = make_float2(0.f, 0.f), Cg = Cr, Cb = Cr;
    // footprint bits of this warp in the complemented AABB mask
    const uint32_t foot = 0xffffu | (((1u << kWlRows) - 1u) << (16 + wl_row0(warp)));
    auto step = [&](int q, auto kAabb) {
        const float4 a = s_list[warp][q].a;
        const float4 rt = s_list[warp][q].t[rr];
        asm volatile("" : "+f"(px.x), "+f"(px.y));
        const float2 dx = sub2(px, make_float2(a.x, a.x));
        const float2 t2 = fma2(make_float2(a.y, a.y), dx, make_float2(rt.z, rt.z));
        const float2 e2 = fma2(dx, t2, make_float2(rt.w, rt.w));
        bool v0 = e2.x >= thr.x, v1 = e2.y >= thr.y;
        if constexpr (decltype(kAabb)::value) {
            const uint32_t m = __float_as_uint(rt.y);
            v0 = v0 && (m & pb0) == 0u;
            v1 = v1 && (m & pb1) == 0u;
        }
        const float m0 = v0 ? fminf(ex2_approx(e2.x), kAlphaPre) : 0.0f;
        const float m1 = v1 ? fminf(ex2_approx(e2.y), kAlphaPre) : 0.0f;
        const float2 w = mul2(make_float2(m0, m1), T);
        const float2 Tprev = T;
        T = fma2(make_float2(-kInv255, -kInv255), w, T);
        Cr = fma2(make_float2(a.z, a.z), w, Cr);
        Cg = fma2(make_float2(a.w, a.w), w, Cg);
        Cb = fma2(make_float2(rt.x, rt.x), w, Cb);
        const bool s0 = T.x < kStopU, s1 = T.y < kStopU;
        if (__builtin_expect(s0 || s1, 0)) {
            if (s0) {
                Cr.x = fmaf(-a.z, w.x, Cr.x);
                Cg.x = fmaf(-a.w, w.x, Cg.x);
                Cb.x = fmaf(-rt.x, w.x, Cb.x);
                T.x = Tprev.x;
                thr.x = kInf;
            }
            if (s1) {
                Cr.y = fmaf(-a.z, w.y, Cr.y);
                Cg.y = fmaf(-a.w, w.y, Cg.y);
                Cb.y = fmaf(-rt.x, w.y, Cb.y);
                T.y = Tprev.y;
                thr.y = kInf;
            }
        }
    };
    // Two records, one stop test: U after both is checked; a
    // pixel that fell below the threshold is rolled back to the record that
    // crossed it (U restored to before that record, the colour steps of the
    // crossing record and of any later one subtracted, colours reloaded from
    // the list).  Same stop decisions as the per-record test.
    auto blend1 = [&](const float4 &a, const float4 &rt, auto kAabb, float2 &w) {
        asm volatile("" : "+f"(px.x), "+f"(px.y));
        const float2 dx = sub2(px, make_float2(a.x, a.x));
        const float2 t2 = fma2(make_float2(a.y, a.y), dx, make_float2(rt.z, rt.z));
        const float2 e2 = fma2(dx, t2, make_float2(rt.w, rt.w));
        bool v0 = e2.x >= thr.x, v1 = e2.y >= thr.y;
        if constexpr (decltype(kAabb)::value) {
            const uint32_t m = __float_as_uint(rt.y);
            v0 = v0 && (m & pb0) == 0u;
            v1 = v1 && (m & pb1) == 0u;
        }
        const float m0 = v0 ? fminf(ex2_approx(e2.x), kAlphaPre) : 0.0f;
        const float m1 = v1 ? fminf(ex2_approx(e2.y), kAlphaPre) : 0.0f;
        w = mul2(make_float2(m0, m1), T);
        T = fma2(make_float2(-kInv255, -kInv255), w, T);
        Cr = fma2(make_float2(a.z, a.z), w, Cr);
        Cg = fma2(make_float2(a.w, a.w), w, Cg);
        Cb = fma2(make_float2(rt.x, rt.x), w, Cb);
    };
    auto step2 = [&](int q, auto kAabb) {
        const float2 T0 = T;
        float2 w1, w2;
        blend1(s_list[warp][q].a, s_list[warp][q].t[rr], kAabb, w1);
        const float2 T1 = T;
        blend1(s_list[warp][q + 1].a, s_list[warp][q + 1].t[rr], kAabb, w2);
        // a warp vote: the branch is uniform (no reconvergence barrier per pair)
        if (__builtin_expect(__any_sync(0xffffffffu, fminf(T.x, T.y) < kStopU), 0)) {
            const float4 a1 = s_list[warp][q].a, r1 = s_list[warp][q].t[rr];
            const float4 a2 = s_list[warp][q + 1].a, r2 = s_list[warp][q + 1].t[rr];
            auto undo = [&](float &cr, float &cg, float &cb, float &t, float &th, float t0, float t1, float x1,
                            float x2) {
                if (!(t < kStopU)) return;
                cr = fmaf(-a2.z, x2, cr);  // the second record's step, always
                cg = fmaf(-a2.w, x2, cg);
                cb = fmaf(-r2.x, x2, cb);
                t = t1;
                if (t1 < kStopU) {  // the first record crossed
                    cr = fmaf(-a1.z, x1, cr);
                    cg = fmaf(-a1.w, x1, cg);
                    cb = fmaf(-r1.x, x1, cb);
                    t = t0;
                }
                th = __int_as_float(0x7f800000);
            };
            undo(Cr.x, Cg.x, Cb.x, T.x, thr.x, T0.x, T1.x, w1.x, w2.x);
            undo(Cr.y, Cg.y, Cb.y, T.y, thr.y, T0.y, T1.y, w1.y, w2.y);
        }
    };
    // pixel-centre y of this warp's strip rows (per-warp constants)
    float rowc[kWlRows];
#pragma unroll
    for (int r = 0; r < kWlRows; ++r) rowc[r] = (float)(ty * 16 + wl_row0(warp) + r) + 0.5f;
    // gather a batch (warp-uniform bs < end): lanes past the tile's last entry
    // re-load that entry (valid memory, culled by lane < n below) -- no zeroing
    auto fetch = [&](uint32_t bs, float4 &a0, float4 &a1, float4 &a2) {
        const uint32_t v = __ldg(entries + min(bs + lane, end - 1));
        a0 = __ldg(rec0 + v);
        a1 = __ldg(rec1 + v);
        a2 = __ldg(rec2 + v);
    };
    bool wdone = __all_sync(0xffffffffu, thr.x == kInf && thr.y == kInf);
    float4 r0, r1, r2;
    if (start < end) fetch(start, r0, r1, r2);
    for (uint32_t base = start; base < end && !wdone; base += 32) {
        const int n = (int)min(32u, end - base);
        // ---- stage this warp's list of the batch
        const bool redundant = (__float_as_uint(r1.w) & 0x80000000u) != 0u;
        uint32_t mb = 0;
        float t1s[kWlRows], t4s[kWlRows];
        const bool rw = strip_stage<kWlRows>(r0, r1, r2.z, tx, ty, wl_row0(warp), rowc, mb, t1s, t4s);
        const float u = r0.x, Ap = r0.z;
        const bool reach = lane < n && rw;
        const uint32_t bal = __ballot_sync(0xffffffffu, reach);
        const bool masked = __any_sync(0xffffffffu, reach && !redundant && (mb & foot) != 0u);
        __syncwarp();  // the previous list has been read
        if (reach) {
            WlEntry &E = s_list[warp][__popc(bal & lanemask_lt())];
            E.a = make_float4(u, Ap, r2.x, r2.y);
#pragma unroll
            for (int r = 0; r < kWlRows; ++r) E.t[r] = make_float4(r2.z, __uint_as_float(mb), t1s[r], t4s[r]);
        }
        // ---- gather the next batch while this one is composited
        if (base + 32 < end) fetch(base + 32, r0, r1, r2);
        __syncwarp();
        const int cnt = __popc(bal);
        if (masked) {
#pragma unroll kWlUnroll
            for (int q = 0; q < cnt; ++q) step(q, std::true_type{});
        } else {
            int q = 0;
#pragma unroll kWiPairUnroll
            for (; q + 1 < cnt; q += 2) step2(q, std::false_type{});
            if (q < cnt) step(q, std::false_type{});
        }
        wdone = __all_sync(0xffffffffu, thr.x == kInf && thr.y == kInf);
    }
    T = mul2(T, make_float2(255.0f, 255.0f));
    if (ok && out_rgb != nullptr) {
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
}


// ---------------------------------------------------------------- launcher
// Grid shapes of the front end (compile-time; DESIGN.md "Thin front-end
// kernels"): persistent onesweep grids on FDGS_PGRID blocks per SM divided by
// FDGS_PGRID_DIV, the binning kernels on FDGS_BIN_GRID / FDGS_ITEM_GRID blocks
// per SM.  The library reads no environment variables.
#ifndef FDGS_PGRID
#define FDGS_PGRID 1
#endif
#ifndef FDGS_PGRID_DIV
#define FDGS_PGRID_DIV 2
#endif
#ifndef FDGS_BIN_GRID
#define FDGS_BIN_GRID 2
#endif
#ifndef FDGS_ITEM_GRID
#define FDGS_ITEM_GRID 2
#endif
static_assert(FDGS_PGRID >= 1 && FDGS_PGRID_DIV >= 1 && FDGS_BIN_GRID >= 1 && FDGS_ITEM_GRID >= 1, "grid shapes");
__global__ void __launch_bounds__(256) k_zero(uint4 *__restrict__ p, size_t n16) {
    for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n16; i += (size_t)gridDim.x * 256)
        p[i] = make_uint4(0u, 0u, 0u, 0u);
}
static int sort_grid(int p_sort) { return std::max(1, FDGS_PGRID * p_sort / FDGS_PGRID_DIV); }

static void launch_timed_blend(const uint32_t *tstart, const uint32_t *entries, const float4 *rec0,
                               const float4 *rec1, const float4 *rec2, const Counters *ctr, const RenderLayout &L,
                               const CamDev &cam, float *out_rgb, float *out_T, cudaStream_t st) {
    k_blend_wi<<<L.n_tiles, kWiThreads, 0, st>>>(tstart, entries, rec0, rec1, rec2, ctr, L.tiles_x, L.width,
                                                 L.height, cam.bg[0], cam.bg[1], cam.bg[2], out_rgb, out_T);
}

cudaError_t launch_render(const SceneDev &sc, const uint32_t *mask_l, const uint32_t *mask_r, const CamDev &cam,
                          float t, float *out_rgb, float *out_T, char *ws, const RenderLayout &L,
                          fdgs_frame_stats *stats, cudaStream_t st, cudaEvent_t const *ev, cudaStream_t blend_st,
                          cudaEvent_t split_ev, unsigned long long *contrib, uint32_t *stv_info, bool front_only) {
    Counters *ctr = reinterpret_cast<Counters *>(ws + L.counters);
    float4 *rec0 = reinterpret_cast<float4 *>(ws + L.rec0);
    float4 *rec1 = reinterpret_cast<float4 *>(ws + L.rec1);
    float4 *rec2 = reinterpret_cast<float4 *>(ws + L.rec2);
    uint32_t *depth = reinterpret_cast<uint32_t *>(ws + L.depth);
    uint2 *rect = reinterpret_cast<uint2 *>(ws + L.rect);
    uint2 *rect_sorted = reinterpret_cast<uint2 *>(ws + L.rect_sorted);
    uint32_t *keys[2] = {reinterpret_cast<uint32_t *>(ws + L.keys0), reinterpret_cast<uint32_t *>(ws + L.keys1)};
    uint32_t *vals[2] = {reinterpret_cast<uint32_t *>(ws + L.vals0), reinterpret_cast<uint32_t *>(ws + L.vals1)};
    uint32_t *tstart = reinterpret_cast<uint32_t *>(ws + L.tile_start);
    uint32_t *entries = reinterpret_cast<uint32_t *>(ws + L.entries);
    uint32_t *surv = reinterpret_cast<uint32_t *>(ws + L.surv);
    uint32_t *vis = reinterpret_cast<uint32_t *>(ws + L.vis);

    cudaError_t e = cudaSuccess;
    // stage events; captured (front_only) as event-record nodes of the graph
    auto rec = [&](int k) {
        return front_only ? cudaEventRecordWithFlags(ev[k], st, cudaEventRecordExternal) : cudaEventRecord(ev[k], st);
    };
    if (ev && (e = rec(0)) != cudaSuccess) return e;
    {
        // counters, digit bases, histograms: a kernel, not a memset (a memset
        // node in a captured graph adds a copy-engine hop to every frame)
        {
            const size_t n16 = (L.zero_end - L.counters) / 16;  // ~30 KB at C3; one block per 64 KB
            k_zero<<<(int)std::min<size_t>(std::max<size_t>(1, n16 / 4096), 148), 256, 0, st>>>(
                reinterpret_cast<uint4 *>(ws + L.counters), n16);
        }
        if (sc.n > 0) {
            uint32_t *cbits = reinterpret_cast<uint32_t *>(ws + L.surv_bits);
            uint32_t *ccnt = reinterpret_cast<uint32_t *>(ws + L.cull_cnt);
            k_cull<<<L.cull_parts, kPreBlock, 0, st>>>(sc, mask_l, mask_r, t, ctr, cbits, ccnt);
            k_count_scan<<<1, 1024, 0, st>>>(ccnt, L.cull_parts, nullptr, kCullItems, &ctr->n_surv);
            k_cull_emit<<<L.cull_parts, kPreBlock, 0, st>>>(cbits, ccnt, sc.n, surv);
            uint32_t *vbits = reinterpret_cast<uint32_t *>(ws + L.vis_bits);
            uint32_t *vcnt = reinterpret_cast<uint32_t *>(ws + L.vis_cnt);
            k_slice<<<L.slice_grid, kPreBlock, 0, st>>>(sc, cam, t, ctr, surv, rec0, rec1, rec2, depth, rect, vbits,
                                                        vcnt);
            k_count_scan<<<1, 1024, 0, st>>>(vcnt, L.n_parts, &ctr->n_surv, kSliceItems, &ctr->n_vis);
            k_vis_emit<<<L.slice_grid, kPreBlock, 0, st>>>(vbits, vcnt, ctr, depth, vis, keys[1]);
        }
        if (ev && (e = rec(1)) != cudaSuccess) return e;
        uint32_t *gbase = reinterpret_cast<uint32_t *>(ws + L.sort_gbase);  // [4][256] depth digit bases
        uint32_t *epoch = reinterpret_cast<uint32_t *>(ws + L.epoch);
        uint64_t *sstat = reinterpret_cast<uint64_t *>(ws + L.sort_status);
        k_sort_hist<<<L.p_sort, kSortThreads, 0, st>>>(keys[1], ctr, gbase, epoch);
        static_assert(kDepthTile == kSortThreads * kDepthItems, "depth-sort partition = status-table stride");
        for (int pass = 0; pass < 4; ++pass) {
            // pass 0 reads the compacted keys (keys[1]) and the visible survivor slots
            const uint32_t *kin = pass == 0 ? keys[1] : keys[(pass - 1) & 1];
            const uint32_t *vin = pass == 0 ? vis : vals[(pass - 1) & 1];
            k_onesweep<8, kDepthItems><<<std::min(L.sort_parts, sort_grid(L.p_sort)), kSortThreads, 0, st>>>(
                kin, vin, pass == 3 ? nullptr : keys[pass & 1], vals[pass & 1], &ctr->n_vis, epoch,
                &ctr->sort_ticket[1 + pass], 8 * pass, gbase + 256 * pass,
                sstat + (size_t)pass * L.sort_parts * 256, rect, pass == 3 ? rect_sorted : nullptr);
        }
        const uint32_t *order = vals[1];
        if (ev && (e = rec(2)) != cudaSuccess) return e;
        int *rowdiff = reinterpret_cast<int *>(ws + L.row_diff);
        uint32_t *rbase = reinterpret_cast<uint32_t *>(ws + L.tile_gbase);  // [0..255] pass 0, [256..511] pass 1
        uint32_t *row_start = reinterpret_cast<uint32_t *>(ws + L.row_start);
        uint32_t *ikey[2] = {reinterpret_cast<uint32_t *>(ws + L.ekey0), reinterpret_cast<uint32_t *>(ws + L.ekey1)};
        uint32_t *ival[2] = {reinterpret_cast<uint32_t *>(ws + L.eval0), reinterpret_cast<uint32_t *>(ws + L.eval1)};
        uint32_t *ipack = reinterpret_cast<uint32_t *>(ws + L.item_pack);
        uint32_t *iv = reinterpret_cast<uint32_t *>(ws + L.item_v);
        uint32_t *rhist = reinterpret_cast<uint32_t *>(ws + L.row_hist);
        uint64_t *tstat = reinterpret_cast<uint64_t *>(ws + L.tile_status);
        BandConsts *bconst = reinterpret_cast<BandConsts *>(ws + L.band_consts);
        const uint32_t item_chunks = (uint32_t)std::max<int64_t>(1, (L.max_entries + kItemTile - 1) / kItemTile);
        {
            uint32_t *pcnt = reinterpret_cast<uint32_t *>(ws + L.bin_cnt);  // items per k_bin_count partition
            const int bparts = std::max(1, (L.n + kScanNT - 1) / kScanNT);
            const int bgrid = std::min(bparts, FDGS_BIN_GRID * L.p_sort);
            k_bin_count<<<bgrid, kScanNT, 0, st>>>(rect_sorted, order, rec0, rec1, ctr, bconst, rowdiff, L.tiles_y,
                                                   pcnt);
            k_count_scan<<<1, 1024, 0, st>>>(pcnt, bparts, &ctr->n_vis, kScanNT, &ctr->n_items);
            k_bin_offsets<<<bgrid, kScanNT, 0, st>>>(rect_sorted, ctr, pcnt, ikey[0], iv, (uint32_t)L.max_entries);
        }
        k_row_items<<<(int)std::min<uint32_t>(item_chunks, FDGS_ITEM_GRID * L.p_sort), kScanNT, 0, st>>>(
            rect_sorted, order, rec0, rec1, bconst, ctr, &ctr->n_items, ikey[0], ipack, iv, (uint32_t)L.max_entries);
        k_row_scan<<<1, 32, 0, st>>>(rowdiff, L.tiles_y, row_start, rbase);
        // stable partition of the row items by tile row (canonical order kept within a row)
        const int rgrid = std::min((int)item_chunks, sort_grid(L.p_sort));
        const uint32_t *sorted_items = ival[0];
        // one pass when the rows fit its digit (6/7/8 bits: the digit width
        // follows tiles_y, so the per-digit scans and look-backs cover only
        // digits that can occur; C3/C4's 64 rows take 64 digits, not 256)
        auto row_pass0 = [&](auto bits) {
            k_onesweep<decltype(bits)::value, kTileSortItems><<<rgrid, kSortThreads, 0, st>>>(
                ikey[0], nullptr, L.tiles_y > 256 ? ikey[1] : nullptr, ival[0], &ctr->n_items_part, epoch,
                &ctr->tile_ticket[0], 0, rbase, tstat, nullptr, nullptr);
        };
        if (L.tiles_y <= 64) row_pass0(std::integral_constant<int, 6>{});
        else if (L.tiles_y <= 128) row_pass0(std::integral_constant<int, 7>{});
        else row_pass0(std::integral_constant<int, 8>{});
        if (L.tiles_y > 256) {
            k_onesweep<8, kTileSortItems><<<rgrid, kSortThreads, 0, st>>>(ikey[1], ival[0], nullptr, ival[1], &ctr->n_items_part, epoch,
                                                           &ctr->tile_ticket[1], 8, rbase + 256,
                                                           tstat + (size_t)L.tile_parts * 256, nullptr, nullptr);
            sorted_items = ival[1];
        }
        const int nrb = L.tiles_y * kRowSeg;
        const size_t cnt_smem = sizeof(uint32_t) * (size_t)kRowWarps * L.tiles_x;
        uint32_t *tcnt = reinterpret_cast<uint32_t *>(ws + L.tile_cnt);  // per-tile totals (zeroed per frame)
        k_row_count<<<nrb, FDGS_ROWCNT_THREADS, sizeof(int) * (L.tiles_x + 1), st>>>(sorted_items, ipack, row_start, L.tiles_x, rhist,
                                                                      tcnt, ctr);
        k_tile_scan<<<1, 1024, 0, st>>>(tcnt, L.tiles_x, L.tiles_y, tstart, ctr, L.max_entries);
        k_row_scatter<<<nrb, 32 * kRowWarps, cnt_smem + sizeof(uint32_t) * L.tiles_x, st>>>(
            sorted_items, ipack, iv, row_start, L.tiles_x, rhist, tstart, entries, ctr);
    }
    if (front_only) return cudaGetLastError();  // graph capture of the front end
    // the blend may run on its own (lower-priority) stream, ordered after the front end
    cudaStream_t bst = st;
    if (blend_st != nullptr) {
        if ((e = cudaEventRecord(split_ev, st)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(blend_st, split_ev, 0)) != cudaSuccess) return e;
        bst = blend_st;
    }
    if (ev && (e = cudaEventRecord(ev[3], bst)) != cudaSuccess) return e;
    if (contrib != nullptr) {  // spatial-score recording (fdgs_stv_score)
        k_blend_ws<false, true><<<L.n_tiles, kWsThreads, 0, bst>>>(tstart, entries, rec0, rec1, rec2, ctr, L.tiles_x,
                                                                   L.width, L.height, cam.bg[0], cam.bg[1], cam.bg[2],
                                                                   out_rgb, out_T, nullptr, contrib, stv_info);
    } else if (stats != nullptr) {  // Eq. 2 work counters (visits every record)
        k_blend_ws<true><<<L.n_tiles, kWsThreads, 0, bst>>>(tstart, entries, rec0, rec1, rec2, ctr, L.tiles_x, L.width,
                                                            L.height, cam.bg[0], cam.bg[1], cam.bg[2], out_rgb, out_T,
                                                            stats);
    } else {  // the timed blend
        launch_timed_blend(tstart, entries, rec0, rec1, rec2, ctr, L, cam, out_rgb, out_T, bst);
    }
    if (ev && (e = cudaEventRecord(ev[4], bst)) != cudaSuccess) return e;
    return cudaGetLastError();
}

// Opt-in to large dynamic shared memory once per process.
__host__ cudaError_t render_set_smem_attrs() {
    cudaError_t e = cudaFuncSetAttribute(k_row_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_row_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    return e;
}

}  // namespace fdgs

// ---------------------------------------------------------------- CUDA graph
// One captured frame (launch_render with the blend on a second captured
// stream) per workspace layout.  Per frame only the four kernel nodes whose
// arguments change are re-parameterised (cull: scene, masks, t; cull emission:
// n; slice: scene, camera, t; blend: background, outputs) and the graph is
// launched: one host call instead of ~21 launches.  Front-end nodes run at the
// device's greatest stream priority, the blend at the least (as
// fdgs_render_split), so frames of different workspaces interleave.
namespace fdgs {

struct RenderGraphImpl {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t n_cull = nullptr, n_emit = nullptr, n_slice = nullptr;
    cudaKernelNodeParams p_cull{}, p_emit{}, p_slice{};
    // stage events 0-2 (front-end start, after preprocess, after the depth
    // sort) as event-record nodes, re-pointed per launch at the caller's events
    cudaEvent_t ph[3] = {nullptr, nullptr, nullptr};  // the nodes' events when the launch passes none
    cudaGraphNode_t n_ev[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t cur_ev[3] = {nullptr, nullptr, nullptr};
    RenderLayout L{};
    char *ws = nullptr;
};

cudaError_t render_graph_build(RenderGraphImpl &g, const SceneDev &sc, const CamDev &cam, char *ws,
                               const RenderLayout &L) {
    g.L = L;
    g.ws = ws;
    // the front end only: the blend is launched directly after the graph (on
    // the caller's blend stream), so it keeps the stream-priority split
    cudaStream_t s1 = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    for (int k = 0; k < 3 && e == cudaSuccess; ++k) e = cudaEventCreate(&g.ph[k]);
    for (int k = 0; k < 3; ++k) g.cur_ev[k] = g.ph[k];
    cudaEvent_t evs[5] = {g.ph[0], g.ph[1], g.ph[2], nullptr, nullptr};
    if (e == cudaSuccess) e = cudaStreamBeginCapture(s1, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        cudaError_t le = launch_render(sc, nullptr, nullptr, cam, 0.0f, nullptr, nullptr, ws, L, nullptr, s1, evs,
                                       nullptr, nullptr, nullptr, nullptr, true);
        cudaError_t ee = cudaStreamEndCapture(s1, &g.graph);
        e = le != cudaSuccess ? le : ee;
    }
    if (e == cudaSuccess) {
        size_t nn = 0;
        e = cudaGraphGetNodes(g.graph, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        if (e == cudaSuccess) e = cudaGraphGetNodes(g.graph, nodes.data(), &nn);
        int least = 0, greatest = 0;
        if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
        for (size_t k = 0; e == cudaSuccess && k < nn; ++k) {
            cudaGraphNodeType ty;
            if ((e = cudaGraphNodeGetType(nodes[k], &ty)) != cudaSuccess) break;
            if (ty == cudaGraphNodeTypeEventRecord) {
                cudaEvent_t x = nullptr;
                if ((e = cudaGraphEventRecordNodeGetEvent(nodes[k], &x)) != cudaSuccess) break;
                for (int j = 0; j < 3; ++j)
                    if (x == g.ph[j]) g.n_ev[j] = nodes[k];
                continue;
            }
            if (ty != cudaGraphNodeTypeKernel) continue;
            cudaKernelNodeParams p{};
            if ((e = cudaGraphKernelNodeGetParams(nodes[k], &p)) != cudaSuccess) break;
            cudaKernelNodeAttrValue pr{};
            pr.priority = greatest;
            e = cudaGraphKernelNodeSetAttribute(nodes[k], cudaKernelNodeAttributePriority, &pr);
            if (p.func == (void *)k_cull) g.n_cull = nodes[k], g.p_cull = p;
            else if (p.func == (void *)k_cull_emit) g.n_emit = nodes[k], g.p_emit = p;
            else if (p.func == (void *)k_slice) g.n_slice = nodes[k], g.p_slice = p;
        }
        // an empty layout (n = 0) captures no cull / slice nodes (launch_render skips them)
        const bool cull_nodes = g.n_cull && g.n_emit && g.n_slice;
        if (e == cudaSuccess && ((L.n > 0 && !cull_nodes) || !g.n_ev[0] || !g.n_ev[1] || !g.n_ev[2]))
            e = cudaErrorInvalidValue;
    }
    // front-end nodes at the device's greatest priority, whatever the launching stream's
    if (e == cudaSuccess) e = cudaGraphInstantiateWithFlags(&g.exec, g.graph, cudaGraphInstantiateFlagUseNodePriority);
    if (s1) cudaStreamDestroy(s1);
    return e;
}

cudaError_t render_graph_launch(RenderGraphImpl &g, const SceneDev &sc, const uint32_t *mask_l,
                                const uint32_t *mask_r, const CamDev &cam, float t, float *out_rgb, float *out_T,
                                cudaStream_t st, cudaStream_t blend_st, cudaEvent_t split_ev,
                                cudaEvent_t const *ev) {
    const RenderLayout &L = g.L;
    char *ws = g.ws;
    Counters *ctr = reinterpret_cast<Counters *>(ws + L.counters);
    uint32_t *cbits = reinterpret_cast<uint32_t *>(ws + L.surv_bits);
    uint32_t *ccnt = reinterpret_cast<uint32_t *>(ws + L.cull_cnt);
    uint32_t *surv = reinterpret_cast<uint32_t *>(ws + L.surv);
    float4 *rec0 = reinterpret_cast<float4 *>(ws + L.rec0);
    float4 *rec1 = reinterpret_cast<float4 *>(ws + L.rec1);
    float4 *rec2 = reinterpret_cast<float4 *>(ws + L.rec2);
    uint32_t *depth = reinterpret_cast<uint32_t *>(ws + L.depth);
    uint2 *rect = reinterpret_cast<uint2 *>(ws + L.rect);
    uint32_t *vbits = reinterpret_cast<uint32_t *>(ws + L.vis_bits);
    uint32_t *vcnt = reinterpret_cast<uint32_t *>(ws + L.vis_cnt);
    uint32_t *tstart = reinterpret_cast<uint32_t *>(ws + L.tile_start);
    uint32_t *entries = reinterpret_cast<uint32_t *>(ws + L.entries);
    // k_cull(sc, mask_l, mask_r, t, ctr, bits, cnt)
    const Counters *cctr = ctr;
    void *a_cull[] = {(void *)&sc, (void *)&mask_l, (void *)&mask_r, (void *)&t, (void *)&ctr, (void *)&cbits,
                      (void *)&ccnt};
    cudaKernelNodeParams p = g.p_cull;
    p.kernelParams = a_cull;
    p.extra = nullptr;
    cudaError_t e = g.n_cull ? cudaGraphExecKernelNodeSetParams(g.exec, g.n_cull, &p) : cudaSuccess;
    // k_cull_emit(bits, base, n, surv)
    const uint32_t *cbits_c = cbits, *ccnt_c = ccnt;
    int n = sc.n;
    void *a_emit[] = {(void *)&cbits_c, (void *)&ccnt_c, (void *)&n, (void *)&surv};
    p = g.p_emit;
    p.kernelParams = a_emit;
    p.extra = nullptr;
    if (e == cudaSuccess && g.n_emit) e = cudaGraphExecKernelNodeSetParams(g.exec, g.n_emit, &p);
    // k_slice(sc, cam, t, ctr, surv, rec0, rec1, rec2, depth, rect, vbits, vcnt)
    const uint32_t *surv_c = surv;
    void *a_slice[] = {(void *)&sc,   (void *)&cam,  (void *)&t,     (void *)&ctr,   (void *)&surv_c, (void *)&rec0,
                       (void *)&rec1, (void *)&rec2, (void *)&depth, (void *)&rect, (void *)&vbits,  (void *)&vcnt};
    p = g.p_slice;
    p.kernelParams = a_slice;
    p.extra = nullptr;
    if (e == cudaSuccess && g.n_slice) e = cudaGraphExecKernelNodeSetParams(g.exec, g.n_slice, &p);
    for (int k = 0; k < 3 && e == cudaSuccess; ++k) {  // the stage events of this frame (or the placeholders)
        cudaEvent_t want = ev ? ev[k] : g.ph[k];
        if (want != g.cur_ev[k] && (e = cudaGraphExecEventRecordNodeSetEvent(g.exec, g.n_ev[k], want)) == cudaSuccess)
            g.cur_ev[k] = want;
    }
    if (e == cudaSuccess) e = cudaGraphLaunch(g.exec, st);
    if (e != cudaSuccess) return e;
    // the timed blend, launched directly (on the blend stream when given)
    cudaStream_t bst = st;
    if (blend_st != nullptr) {
        if ((e = cudaEventRecord(split_ev, st)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(blend_st, split_ev, 0)) != cudaSuccess) return e;
        bst = blend_st;
    }
    if (ev && (e = cudaEventRecord(ev[3], bst)) != cudaSuccess) return e;
    launch_timed_blend(tstart, entries, rec0, rec1, rec2, cctr, L, cam, out_rgb, out_T, bst);
    if (ev && (e = cudaEventRecord(ev[4], bst)) != cudaSuccess) return e;
    return cudaGetLastError();
}

void render_graph_free(RenderGraphImpl &g) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    for (auto &x : g.ph) {
        if (x) cudaEventDestroy(x);
        x = nullptr;
    }
    g.exec = nullptr;
    g.graph = nullptr;
}
RenderGraphImpl *render_graph_new() { return new (std::nothrow) RenderGraphImpl(); }
void render_graph_delete(RenderGraphImpl *g) {
    if (g) {
        render_graph_free(*g);
        delete g;
    }
}
const RenderLayout &render_graph_layout(const RenderGraphImpl &g) { return g.L; }

}  // namespace fdgs
