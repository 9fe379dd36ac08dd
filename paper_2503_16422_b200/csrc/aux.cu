// aux.cu -- key-frame masks, mask OR / compaction,
// scene validation and the derived L_i = ln(255 sigma_i) field.
#include <algorithm>

#include "fdgs_internal.h"

namespace fdgs {

// ------------------------------------------------------------ key-frame mask
// One thread per Gaussian: slice once at t_key, project into every camera,
// visible = temporal & support & near & cover culls (the render decision
// path, reading R3); warp ballot -> one uint32 word per warp, no atomics.
__global__ void __launch_bounds__(256) k_keyframe(SceneDev sc, const CamDev *__restrict__ cams, int n_cams, float t,
                                                  uint32_t *__restrict__ out) {
    extern __shared__ CamDev s_cams[];
    for (int c = threadIdx.x; c < n_cams; c += blockDim.x) s_cams[c] = cams[c];
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool vis = false;
    if (i < sc.n) {
        Slice sl;
        const int st = slice_gaussian(sc.ld_mean(i), sc.ld_scale(i), sc.ld_rot_l(i),
                                      sc.ld_rot_r(i), __ldg(sc.L + i), t, sl);
        if (st == kNear) {
            for (int c = 0; c < n_cams && !vis; ++c) {
                Proj pj;
                vis = project_gaussian(sl, s_cams[c], pj) == kVisible;
            }
        }
    }
    const uint32_t word = __ballot_sync(0xffffffffu, vis);
    if ((threadIdx.x & 31) == 0 && i < sc.n) out[i >> 5] = word;
}

cudaError_t launch_keyframe(const SceneDev &sc, const CamDev *d_cams, int n_cams, float t, uint32_t *out,
                            cudaStream_t st) {
    if (sc.n == 0) return cudaSuccess;
    const size_t smem = sizeof(CamDev) * (size_t)n_cams;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_keyframe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k_keyframe<<<(sc.n + 255) / 256, 256, smem, st>>>(sc, d_cams, n_cams, t, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------ mask OR
// Each thread ORs 4 consecutive words (one 16-byte vector when aligned).
__global__ void k_mask_or(const uint32_t *__restrict__ a, const uint32_t *__restrict__ b, int nw,
                          uint32_t *__restrict__ o, bool vec) {
    const int w0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (w0 >= nw) return;
    if (vec && w0 + 4 <= nw) {
        const uint4 x = __ldg(reinterpret_cast<const uint4 *>(a + w0)), y = __ldg(reinterpret_cast<const uint4 *>(b + w0));
        *reinterpret_cast<uint4 *>(o + w0) = make_uint4(x.x | y.x, x.y | y.y, x.z | y.z, x.w | y.w);
        return;
    }
    for (int w = w0; w < min(w0 + 4, nw); ++w) o[w] = __ldg(a + w) | __ldg(b + w);
}

cudaError_t launch_mask_or(const uint32_t *a, const uint32_t *b, int n, uint32_t *out, cudaStream_t st) {
    const int nw = (n + 31) / 32;
    if (nw == 0) return cudaSuccess;
    const bool vec = ((uintptr_t)a % 16 == 0) && ((uintptr_t)b % 16 == 0) && ((uintptr_t)out % 16 == 0);
    const int threads = 256, per_block = 4 * threads;
    k_mask_or<<<(nw + per_block - 1) / per_block, threads, 0, st>>>(a, b, nw, out, vec);
    return cudaGetLastError();
}

// ------------------------------------------------------------ compaction
// 256 Gaussians (8 words) per block; warp ballot is free (one word per lane
// group), block scan of popcounts, decoupled look-back across blocks.
__device__ __forceinline__ uint32_t ldv(const uint32_t *p) { return *(const volatile uint32_t *)p; }
__device__ __forceinline__ void stv(uint32_t *p, uint32_t v) { *(volatile uint32_t *)p = v; }

__global__ void __launch_bounds__(256) k_mask_compact(const uint32_t *__restrict__ a, const uint32_t *__restrict__ b,
                                                      int n, int32_t *__restrict__ idx, uint32_t *__restrict__ count,
                                                      uint32_t *ticket_status) {
    __shared__ uint32_t s_part, s_w[8], s_excl;
    uint32_t *ticket = ticket_status;
    uint32_t *status = ticket_status + 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_part = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t part = s_part;
    const int i = (int)part * 256 + tid;
    bool set = false;
    if (i < n) {
        uint32_t w = __ldg(a + (i >> 5));
        if (b) w |= __ldg(b + (i >> 5));
        set = (w >> (i & 31)) & 1u;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, set);
    if (lane == 0) s_w[warp] = __popc(bal);
    __syncthreads();
    if (tid == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < 8; ++w) {
            const uint32_t c = s_w[w];
            s_w[w] = tot;
            tot += c;
        }
        uint32_t excl = 0;
        if (part == 0) {
            stv(&status[0], kFlagP | tot);
        } else {
            stv(&status[part], kFlagA | tot);
            int j = (int)part - 1;
            while (true) {
                const uint32_t s = ldv(&status[j]);
                const uint32_t f = s & ~kValMask;
                if (f == 0) continue;
                excl += s & kValMask;
                if (f == kFlagP) break;
                --j;
            }
            stv(&status[part], kFlagP | (excl + tot));
        }
        s_excl = excl;
        if (part == gridDim.x - 1) *count = excl + tot;
    }
    __syncthreads();
    if (set) {
        uint32_t lt;
        asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
        idx[s_excl + s_w[warp] + __popc(bal & lt)] = i;
    }
}

cudaError_t launch_mask_compact(const uint32_t *a, const uint32_t *b, int n, int32_t *idx, uint32_t *count,
                                uint32_t *ws, cudaStream_t st) {
    const int parts = (n + 255) / 256;
    cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(uint32_t) * (32 + (size_t)parts), st);
    if (e != cudaSuccess) return e;
    if (parts == 0) return cudaMemsetAsync(count, 0, sizeof(uint32_t), st);
    k_mask_compact<<<parts, 256, 0, st>>>(a, b, n, idx, count, ws);
    return cudaGetLastError();
}

// ------------------------------------------------------------ validation
// SPEC invariants and the degenerate-Sigma_t guard.
__global__ void k_validate(SceneDev sc, unsigned long long *first_bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= sc.n) return;
    const float4 ql = sc.ld_rot_l(i), qr = sc.ld_rot_r(i), s = sc.ld_scale(i);
    const float op = sc.opacity[i];
    const double nl = sqrt((double)ql.x * ql.x + (double)ql.y * ql.y + (double)ql.z * ql.z + (double)ql.w * ql.w);
    const double nr = sqrt((double)qr.x * qr.x + (double)qr.y * qr.y + (double)qr.z * qr.z + (double)qr.w * qr.w);
    bool bad = !(fabs(nl - 1.0) <= 1e-6) || !(fabs(nr - 1.0) <= 1e-6);
    bad |= !(s.x > 0.f && s.y > 0.f && s.z > 0.f && s.w > 0.f);
    bad |= !(op > 0.f && op <= 1.f);
    bad |= !isfinite(sc.L[i]);
    if (sc.sh_index != nullptr) bad |= (int)sc.sh_index[i] >= sc.sh_k;
    if (!bad) {
        // Sigma_44 = sum_j (R4[3][j] s_j)^2 > 1e-12
        const double a = ql.x, b = ql.y, c = ql.z, d = ql.w, p = qr.x, q = qr.y, r = qr.z, w = qr.w;
        const double Rm[4][4] = {{p, -q, -r, -w}, {q, p, w, -r}, {r, -w, p, q}, {w, r, -q, p}};
        const double L3[4] = {d, -c, b, a};
        const double s4[4] = {s.x, s.y, s.z, s.w};
        double s44 = 0.0;
        for (int j = 0; j < 4; ++j) {
            double acc = 0.0;
            for (int k = 0; k < 4; ++k) acc += L3[k] * Rm[k][j];
            const double m = acc * s4[j];
            s44 += m * m;
        }
        bad |= !(s44 > 1e-12);
    }
    if (bad) atomicMin(first_bad, (unsigned long long)i);
}

cudaError_t launch_validate(const SceneDev &sc, unsigned long long *d_first_bad, cudaStream_t st) {
    if (sc.n == 0) return cudaSuccess;
    k_validate<<<(sc.n + 255) / 256, 256, 0, st>>>(sc, d_first_bad);
    return cudaGetLastError();
}

__global__ void k_log255(const float *__restrict__ op, int n, float *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __double2float_rn(log(255.0 * (double)op[i]));
}

cudaError_t launch_log255(const float *op, int n, float *out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_log255<<<(n + 255) / 256, 256, 0, st>>>(op, n, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------ working set
// Gather of the compacted working set: one thread per active Gaussian (the
// ascending index list of k_mask_compact), a 64-byte parameter record, the
// opacity terms and the SH record (or VQ index).
__global__ void __launch_bounds__(256) k_scene_gather(SceneDev sc, const int32_t *__restrict__ idx,
                                                      const uint32_t *__restrict__ count, float4 *__restrict__ params,
                                                      float *__restrict__ opacity, float *__restrict__ L,
                                                      float4 *__restrict__ sh, uint16_t *__restrict__ sh_index,
                                                      uint32_t *__restrict__ gid) {
    const uint32_t m = *count;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const int i = __ldg(idx + j);
        params[4 * (size_t)j + 0] = sc.ld_mean(i);
        params[4 * (size_t)j + 1] = sc.ld_scale(i);
        params[4 * (size_t)j + 2] = sc.ld_rot_l(i);
        params[4 * (size_t)j + 3] = sc.ld_rot_r(i);
        opacity[j] = __ldg(sc.opacity + i);
        L[j] = __ldg(sc.L + i);
        if (sh_index) {
            sh_index[j] = __ldg(sc.sh_index + i);
        } else {
#pragma unroll
            for (int k = 0; k < 12; ++k) sh[12 * (size_t)j + k] = __ldg(sc.sh + 12 * (size_t)i + k);
        }
        gid[j] = (uint32_t)i;
    }
}

cudaError_t launch_scene_compact(const SceneDev &sc, const uint32_t *mask_l, const uint32_t *mask_r, float4 *params,
                                 float *opacity, float *L, float4 *sh, uint16_t *sh_index, uint32_t *gid,
                                 uint32_t *count, uint32_t *ws, cudaStream_t st) {
    if (sc.n == 0) return cudaMemsetAsync(count, 0, sizeof(uint32_t), st);
    int32_t *idx = reinterpret_cast<int32_t *>(ws);
    uint32_t *cws = ws + (size_t)sc.n;
    cudaError_t e = launch_mask_compact(mask_l, mask_r, sc.n, idx, count, cws, st);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    k_scene_gather<<<std::min((sc.n + 255) / 256, 8 * sms), 256, 0, st>>>(sc, idx, count, params, opacity, L, sh,
                                                                          sh_index, gid);
    return cudaGetLastError();
}

}  // namespace fdgs
