// stv.cu -- spatial-temporal variation score of Sec. 4.2.1,
// the pruning criterion that produces the scene the
// render path then draws.
//
//   S^S_i(t)  = sum over all views and pixels of alpha_i prod_{j<i}(1-alpha_j)
//               (P:249-253): recorded by the contribution variant of the
//               render blend (render.cu k_blend_ws<.., kContrib>), one frame
//               per (view, t), accumulated per Gaussian in 2^-24 fixed point
//   p2_i(t)   = ((t-mu_t)^2/Sigma_t^2 - 1/Sigma_t) p_i(t)
//   S^TV_i(t) = 1 / (0.5 tanh|p2_i(t)| + 0.5)
//   gamma_i   = min(V_i / V_p, 1), V_i = s_x s_y s_z s_t (binary32, left to
//               right), V_p the nearest-rank percentile of V ("normalized
//               following LightGaussian"; reading R20)
//   S_i       = sum_t S^TV_i(t) gamma_i S^S_i(t)   (combine 0, time-aligned, R20)
//             = gamma_i (sum_t S^TV_i(t)) (sum_t S^S_i(t))   (combine 1, the
//               literal product of the two sums of P:264-272)
//
//   k_stv_init / k_vol_hist / k_vol_pick : exact nearest-rank selection of
//       V_p by a 4 x 8-bit MSD radix select over the fp32 bits of V (all V > 0,
//       so bit order = value order)
//   k_stv_accum : per t, fold the recorded S^S with S^TV and gamma
#include <algorithm>
#include <cmath>
#include <vector>

#include "fdgs_internal.h"

namespace fdgs {

__device__ __forceinline__ float volume4(float4 s) {
    float v = __fmul_rn(s.x, s.y);
    v = __fmul_rn(v, s.z);
    return __fmul_rn(v, s.w);
}

__global__ void k_stv_init(StvState *st, uint32_t rank) {
    const int t = threadIdx.x;
    st->hist[t] = 0;
    if (t == 0) {
        st->info[0] = st->info[1] = 0;
        st->prefix = 0;
        st->rank = rank;
    }
}

// Histogram of digit (bits >> shift) & 255 over the volumes whose higher digits
// equal the selected prefix.
__global__ void __launch_bounds__(256) k_vol_hist(SceneDev sc, StvState *st, int shift) {
    const int n = sc.n;
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t hi = shift >= 24 ? 0u : ~0u << (shift + 8);
    const uint32_t prefix = st->prefix;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t bits = __float_as_uint(volume4(sc.ld_scale(i)));
        if (((bits ^ prefix) & hi) == 0) atomicAdd(&h[(bits >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&st->hist[threadIdx.x], h[threadIdx.x]);
}

// Pick the digit holding the remaining rank; clear the histogram for the next pass.
__global__ void k_vol_pick(StvState *st, int shift) {
    __shared__ uint32_t h[256];
    const int t = threadIdx.x;
    h[t] = st->hist[t];
    st->hist[t] = 0;
    __syncthreads();
    if (t == 0) {
        uint32_t cum = 0, rank = st->rank;
        for (int d = 0; d < 256; ++d) {
            if (rank < cum + h[d]) {
                st->prefix |= (uint32_t)d << shift;
                st->rank = rank - cum;
                break;
            }
            cum += h[d];
        }
    }
}

// One t: S^S_i(t) from the fixed-point recorder (then cleared for the next t),
// S^TV_i(t) in binary64, folded into the running sums.
// Per-t terms by variant (score ablations of P:636-669): the temporal factor
// T(t) (gamma applied at the end, it is constant in t) and the spatial S(t):
//   0 full T = S^TV(p2), S = S^S     1 S^S only T = 1 (no gamma), S = S^S
//   2 S^T only T = S^TV(p2), S = 1   3 T = S^TV(p1) = 1/(0.5 tanh|p1| + 0.5), S = S^S
//   4 T = Sigma_t, S = S^S
__global__ void __launch_bounds__(256) k_stv_accum(SceneDev sc, float t, unsigned long long *__restrict__ contrib,
                                                   const StvState *st, double *__restrict__ acc_a,
                                                   double *__restrict__ acc_b, double *__restrict__ acc_c,
                                                   bool first, bool last, int mode, int variant,
                                                   float *__restrict__ out_score, float *__restrict__ out_spatial,
                                                   float *__restrict__ out_gamma) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= sc.n) return;
    const double ss = (double)contrib[i] * 0x1p-24;
    contrib[i] = 0ull;
    const float4 mean = sc.ld_mean(i), s = sc.ld_scale(i);
    const double sig = sigma44(s, sc.ld_rot_l(i), sc.ld_rot_r(i));
    const double dt = (double)t - (double)mean.w;
    const double p = exp(-(dt * dt) / (2.0 * sig));
    double Tt, St = ss;
    if (variant == 3) {
        const double p1 = -(dt / sig) * p;
        Tt = 1.0 / (0.5 * tanh(fabs(p1)) + 0.5);
    } else if (variant == 4) {
        Tt = sig;
    } else if (variant == 1) {
        Tt = 1.0;
    } else {
        const double p2 = ((dt * dt) / (sig * sig) - 1.0 / sig) * p;
        Tt = 1.0 / (0.5 * tanh(fabs(p2)) + 0.5);
    }
    if (variant == 2) St = 1.0;
    double a = first ? 0.0 : acc_a[i], b = first ? 0.0 : acc_b[i], c = first ? 0.0 : acc_c[i];
    a += Tt * St;  // time-aligned
    b += Tt;       // sum_t T
    c += St;       // sum_t S
    if (out_spatial) out_spatial[i] = (float)ss;
    if (!last) {
        acc_a[i] = a;
        acc_b[i] = b;
        acc_c[i] = c;
        return;
    }
    const double vp = (double)__uint_as_float(st->prefix);
    const double g = fmin((double)volume4(s) / vp, 1.0);
    const double gg = variant == 1 ? 1.0 : g;
    out_score[i] = (float)(mode == 0 ? a * gg : gg * b * c);
    if (out_gamma) out_gamma[i] = (float)g;
}

// n_ts == 0: the sums over t are empty (score 0); gamma does not depend on t.
__global__ void __launch_bounds__(256) k_stv_empty(SceneDev sc, const StvState *st, float *__restrict__ out_score,
                                                   float *__restrict__ out_gamma) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= sc.n) return;
    out_score[i] = 0.0f;
    if (out_gamma) out_gamma[i] = (float)fmin((double)volume4(sc.ld_scale(i)) / (double)__uint_as_float(st->prefix), 1.0);
}

// m_{i,j} of P:282 read literally: bit i |= (view's weight sum of i > threshold);
// the recorder is cleared for the next view.
__global__ void __launch_bounds__(256) k_contrib_mask(unsigned long long *__restrict__ contrib, int n,
                                                      unsigned long long thr_fixed, uint32_t *__restrict__ mask) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool set = false;
    if (i < n) {
        set = contrib[i] > thr_fixed;
        contrib[i] = 0ull;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, set);
    if ((threadIdx.x & 31) == 0 && i < n && word) mask[i >> 5] |= word;
}

// ---- pruning selection: keep the `keep` highest scores, equal
// scores ranked by ascending index (reading R23).
//
// key = the score's bits remapped so that ascending key = descending score
// (-0 folded onto +0, so equal values have equal keys).  A 4 x 8-bit MSD radix
// select finds T = the key of rank keep-1 and the remaining rank r within T's
// equal range; then per 1024-element chunk the count of keys == T, a one-block
// scan of the counts, and the emission: bit i = key_i < T, or key_i == T and
// i is among the first r+1 indices holding T.
constexpr int kPruneChunk = 1024;

__device__ __forceinline__ uint32_t prune_key(float s) {
    uint32_t b = __float_as_uint(s);
    if ((b << 1) == 0u) b = 0u;
    const uint32_t ord = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // ascending in value
    return ~ord;
}

__global__ void __launch_bounds__(256) k_prune_hist(const float *__restrict__ score, int n, StvState *st,
                                                    int shift) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t hi = shift >= 24 ? 0u : ~0u << (shift + 8);
    const uint32_t prefix = st->prefix;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = prune_key(__ldg(score + i));
        if (((k ^ prefix) & hi) == 0) atomicAdd(&h[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&st->hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_prune_count(const float *__restrict__ score, int n, const StvState *st,
                                                     uint32_t *__restrict__ cnt) {
    __shared__ uint32_t s_n;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const uint32_t T = st->prefix;
    uint32_t c = 0;
    for (int r = 0; r < kPruneChunk / 256; ++r) {
        const int i = blockIdx.x * kPruneChunk + r * 256 + threadIdx.x;
        c += __popc(__ballot_sync(0xffffffffu, i < n && prune_key(__ldg(score + i)) == T));
    }
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_n, c);
    __syncthreads();
    if (threadIdx.x == 0) cnt[blockIdx.x] = s_n;
}

// all: keep >= n (every bit below n set, T unused).
__global__ void __launch_bounds__(256) k_prune_emit(const float *__restrict__ score, int n, const StvState *st,
                                                    const uint32_t *__restrict__ base, bool all,
                                                    uint32_t *__restrict__ mask) {
    __shared__ uint32_t s_w[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t T = all ? 0u : st->prefix;
    const uint32_t r = all ? 0u : st->rank;  // T-valued elements kept: the first r + 1
    uint32_t carry = all ? 0u : base[blockIdx.x];
    for (int k = 0; k < kPruneChunk / 256; ++k) {
        const int i = blockIdx.x * kPruneChunk + k * 256 + tid;
        const uint32_t key = i < n ? prune_key(__ldg(score + i)) : 0xffffffffu;
        const bool eq = i < n && key == T;
        const uint32_t be = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) s_w[warp] = __popc(be);
        __syncthreads();
        uint32_t before = carry, tot = 0;
        for (int w = 0; w < 8; ++w) {
            if (w < warp) before += s_w[w];
            tot += s_w[w];
        }
        __syncthreads();
        const uint32_t pos = before + __popc(be & ((1u << lane) - 1u));  // rank among T-valued, by index
        const bool set = i < n && (all || key < T || (eq && pos <= r));
        const uint32_t word = __ballot_sync(0xffffffffu, set);
        if (lane == 0 && i < n) mask[i >> 5] = word;
        carry += tot;
    }
}

size_t prune_workspace_bytes(int32_t n) {
    const size_t chunks = (size_t)(std::max(n, 0) + kPruneChunk - 1) / kPruneChunk;
    return ((sizeof(StvState) + 255) & ~size_t(255)) + ((4 * std::max<size_t>(chunks, 1) + 255) & ~size_t(255));
}

cudaError_t launch_prune_mask(const float *score, int n, int64_t keep, uint32_t *mask, char *ws, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    if (keep <= 0) return cudaMemsetAsync(mask, 0, 4 * (size_t)((n + 31) / 32), st);
    StvState *state = reinterpret_cast<StvState *>(ws);
    uint32_t *cnt = reinterpret_cast<uint32_t *>(ws + ((sizeof(StvState) + 255) & ~size_t(255)));
    const int chunks = (n + kPruneChunk - 1) / kPruneChunk;
    if (keep >= n) {
        k_prune_emit<<<chunks, 256, 0, st>>>(score, n, state, cnt, true, mask);
        return cudaGetLastError();
    }
    k_stv_init<<<1, 256, 0, st>>>(state, (uint32_t)(keep - 1));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int hgrid = std::max(1, std::min((n + 255) / 256, 4 * sms));
    for (int shift = 24; shift >= 0; shift -= 8) {
        k_prune_hist<<<hgrid, 256, 0, st>>>(score, n, state, shift);
        k_vol_pick<<<1, 256, 0, st>>>(state, shift);
    }
    k_prune_count<<<chunks, 256, 0, st>>>(score, n, state, cnt);
    k_count_scan<<<1, 1024, 0, st>>>(cnt, chunks, nullptr, 0, &state->info[0]);
    k_prune_emit<<<chunks, 256, 0, st>>>(score, n, state, cnt, false, mask);
    return cudaGetLastError();
}

StvLayout stv_layout(int32_t n, const fdgs_camera *cams, int32_t n_cams, int64_t max_entries) {
    StvLayout L{};
    const size_t nn = (size_t)std::max(n, 1);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    L.state = 0;
    L.contrib = al(sizeof(StvState));
    L.acc_a = L.contrib + al(8 * nn);
    L.acc_b = L.acc_a + al(8 * nn);
    L.acc_c = L.acc_b + al(8 * nn);
    L.render = L.acc_c + al(8 * nn);
    size_t rb = 0;
    for (int c = 0; c < n_cams; ++c)
        rb = std::max(rb, render_layout(n, cams[c].width, cams[c].height, max_entries).total);
    L.total = L.render + rb;
    return L;
}

cudaError_t launch_stv(const SceneDev &sc, const CamDev *cams, const fdgs_camera *hcams, int n_cams, const float *ts,
                       int n_ts, uint32_t rank, int mode, int variant, int64_t max_entries, char *ws,
                       const StvLayout &SL, float *out_score, float *out_spatial, float *out_gamma,
                       cudaStream_t st) {
    StvState *state = reinterpret_cast<StvState *>(ws + SL.state);
    auto *contrib = reinterpret_cast<unsigned long long *>(ws + SL.contrib);
    double *acc[3] = {reinterpret_cast<double *>(ws + SL.acc_a), reinterpret_cast<double *>(ws + SL.acc_b),
                      reinterpret_cast<double *>(ws + SL.acc_c)};
    char *rws = ws + SL.render;
    const int n = sc.n;
    cudaError_t e = cudaSuccess;
    k_stv_init<<<1, 256, 0, st>>>(state, rank);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int hgrid = std::max(1, std::min((n + 255) / 256, 4 * sms));
    for (int shift = 24; shift >= 0; shift -= 8) {
        k_vol_hist<<<hgrid, 256, 0, st>>>(sc, state, shift);
        k_vol_pick<<<1, 256, 0, st>>>(state, shift);
    }
    if (n_ts == 0) {
        k_stv_empty<<<(n + 255) / 256, 256, 0, st>>>(sc, state, out_score, out_gamma);
        return cudaGetLastError();
    }
    if ((e = cudaMemsetAsync(contrib, 0, 8 * (size_t)n, st)) != cudaSuccess) return e;
    int pw = -1, ph = -1;
    for (int k = 0; k < n_ts; ++k) {
        for (int c = 0; c < n_cams; ++c) {
            const RenderLayout L = render_layout(n, hcams[c].width, hcams[c].height, max_entries);
            if (hcams[c].width != pw || hcams[c].height != ph) {
                // epoch-tagged look-back tables sit at size-dependent offsets: restart them
                if ((e = cudaMemsetAsync(rws, 0, L.total, st)) != cudaSuccess) return e;
                pw = hcams[c].width;
                ph = hcams[c].height;
            }
            e = launch_render(sc, nullptr, nullptr, cams[c], ts[k], nullptr, nullptr, rws, L, nullptr, st, nullptr,
                              nullptr, nullptr, contrib, state->info);
            if (e != cudaSuccess) return e;
        }
        k_stv_accum<<<(n + 255) / 256, 256, 0, st>>>(sc, ts[k], contrib, state, acc[0], acc[1], acc[2], k == 0,
                                                     k == n_ts - 1, mode, variant, out_score,
                                                     out_spatial ? out_spatial + (size_t)k * n : nullptr, out_gamma);
    }
    return cudaGetLastError();
}

cudaError_t launch_keyframe_contrib(const SceneDev &sc, const CamDev *cams, const fdgs_camera *hcams, int n_cams,
                                    float t_key, unsigned long long thr_fixed, int64_t max_entries, char *ws,
                                    const StvLayout &SL, uint32_t *out_mask, cudaStream_t st) {
    StvState *state = reinterpret_cast<StvState *>(ws + SL.state);
    auto *contrib = reinterpret_cast<unsigned long long *>(ws + SL.contrib);
    char *rws = ws + SL.render;
    const int n = sc.n;
    cudaError_t e;
    k_stv_init<<<1, 256, 0, st>>>(state, 0u);
    if ((e = cudaMemsetAsync(contrib, 0, 8 * (size_t)n, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(out_mask, 0, 4 * (size_t)((n + 31) / 32), st)) != cudaSuccess) return e;
    int pw = -1, ph = -1;
    for (int c = 0; c < n_cams; ++c) {
        const RenderLayout L = render_layout(n, hcams[c].width, hcams[c].height, max_entries);
        if (hcams[c].width != pw || hcams[c].height != ph) {
            if ((e = cudaMemsetAsync(rws, 0, L.total, st)) != cudaSuccess) return e;
            pw = hcams[c].width;
            ph = hcams[c].height;
        }
        e = launch_render(sc, nullptr, nullptr, cams[c], t_key, nullptr, nullptr, rws, L, nullptr, st, nullptr,
                          nullptr, nullptr, contrib, state->info);
        if (e != cudaSuccess) return e;
        k_contrib_mask<<<(n + 255) / 256, 256, 0, st>>>(contrib, n, thr_fixed, out_mask);
    }
    return cudaGetLastError();
}

}  // namespace fdgs
