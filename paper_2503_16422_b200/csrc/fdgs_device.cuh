// fdgs_device.cuh -- device-side decision path of the render hot path.
//
// Slice (Eq. 1) + temporal marginal (Eq. 3) + EWA
// projection to a 2D conic (P:139 Sigma_2D).  Every operation that DECIDES
// something (a cull, the pixel AABB, the depth key, the fp32 record fields)
// is an explicit IEEE binary64 intrinsic (__dmul_rn, __fma_rn, ...), in the
// order listed in DESIGN.md "Decision path", so the compiler can neither
// contract nor reorder it.  The render kernel and the key-frame mask kernel
// both call these functions, which is what makes a key-frame mask sound
// (reading R3).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fdgs {

// Pinned constants.
constexpr double kKT = 0x1.62a40fda3e3ccp+3;      // 2 ln 255
constexpr double kLog2e = 0x1.71547652b82fep+0;   // log2(e)
constexpr double kCH = -0x1.71547652b82fep-1;     // -log2(e)/2
constexpr double kC1 = -0x1.71547652b82fep+0;     // -log2(e)
constexpr double kDilation = 0.3;
constexpr double kJClamp = 1.3;
constexpr double kMarginMul = 1.0 + 0x1p-10;
constexpr double kMarginAdd = 0x1p-4;
constexpr double kLim = 0x1p30;

enum Stage : int { kTemporal = 0, kSupport = 1, kNear = 2, kCover = 3, kVisible = 4 };

// Camera with the per-view constants of the decision path, built on the host.
struct CamDev {
    double R[9];
    double T[3];
    double fx, fy, cx, cy;
    double limx, limy;     // 1.3 * (W / (2 fx)), 1.3 * (H / (2 fy))
    double z_near;
    float campos[3];       // camera centre -R^T T (value path: SH direction)
    float bg[3];
    int32_t width, height;
};

struct Slice {
    double mu3[3];
    double cov3[6];        // xx xy xz yy yz zz
    double Q;              // ln(255 sigma p_t)
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Row r of R4 = L(q_l) R(q_r), pinned fma chain over k = 0..3.
__device__ __forceinline__ void rotor_row(const double Lr[4], const double Rm[4][4], double out[4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        double acc = dmul(Lr[0], Rm[0][j]);
        acc = dfma(Lr[1], Rm[1][j], acc);
        acc = dfma(Lr[2], Rm[2][j], acc);
        acc = dfma(Lr[3], Rm[3][j], acc);
        out[j] = acc;
    }
}

// The temporal cull alone (row 3 of R4, Sigma_44, dt^2 <= K_T Sigma_44): the
// same ops as the start of slice_gaussian, so both take the same decision.
__device__ __forceinline__ bool temporal_pass(float4 mean, float4 sc, float4 ql, float4 qr, float t_f) {
    const double a = ql.x, b = ql.y, c = ql.z, d = ql.w;
    const double p = qr.x, q = qr.y, r = qr.z, s = qr.w;
    const double Rm[4][4] = {{p, -q, -r, -s}, {q, p, s, -r}, {r, -s, p, q}, {s, r, -q, p}};
    const double s4[4] = {(double)sc.x, (double)sc.y, (double)sc.z, (double)sc.w};
    const double L3[4] = {d, -c, b, a};
    double row[4], m[4];
    rotor_row(L3, Rm, row);
#pragma unroll
    for (int j = 0; j < 4; ++j) m[j] = dmul(row[j], s4[j]);
    double s44 = dmul(m[0], m[0]);
    s44 = dfma(m[1], m[1], s44);
    s44 = dfma(m[2], m[2], s44);
    s44 = dfma(m[3], m[3], s44);
    const double dt = dsub((double)t_f, (double)mean.w);
    return dmul(dt, dt) <= dmul(kKT, s44);
}

// Sigma_44 = (R4 S S^T R4^T)_44 alone (row 3 of R4), the same ops as the start
// of slice_gaussian.  Used by the temporal score (Sigma_t).
__device__ __forceinline__ double sigma44(float4 sc, float4 ql, float4 qr) {
    const double a = ql.x, b = ql.y, c = ql.z, d = ql.w;
    const double p = qr.x, q = qr.y, r = qr.z, s = qr.w;
    const double Rm[4][4] = {{p, -q, -r, -s}, {q, p, s, -r}, {r, -s, p, q}, {s, r, -q, p}};
    const double s4[4] = {(double)sc.x, (double)sc.y, (double)sc.z, (double)sc.w};
    const double L3[4] = {d, -c, b, a};
    double row[4], m[4];
    rotor_row(L3, Rm, row);
#pragma unroll
    for (int j = 0; j < 4; ++j) m[j] = dmul(row[j], s4[j]);
    double s44 = dmul(m[0], m[0]);
    s44 = dfma(m[1], m[1], s44);
    s44 = dfma(m[2], m[2], s44);
    return dfma(m[3], m[3], s44);
}

// Eq. 1 slice with the temporal (p_t >= 1/255) and support (sigma p_t >= 1/255)
// culls.  Returns the stage reached (kTemporal / kSupport on cull, else kNear
// meaning "continue to projection").
__device__ __forceinline__ int slice_gaussian(float4 mean, float4 sc, float4 ql, float4 qr, float L, float t_f,
                                              Slice &o) {
    const double a = ql.x, b = ql.y, c = ql.z, d = ql.w;
    const double p = qr.x, q = qr.y, r = qr.z, s = qr.w;
    const double Rm[4][4] = {{p, -q, -r, -s}, {q, p, s, -r}, {r, -s, p, q}, {s, r, -q, p}};
    const double s4[4] = {(double)sc.x, (double)sc.y, (double)sc.z, (double)sc.w};
    // row 3 first: it alone decides the temporal cull
    double m[4];
    {
        const double L3[4] = {d, -c, b, a};
        double row[4];
        rotor_row(L3, Rm, row);
#pragma unroll
        for (int j = 0; j < 4; ++j) m[j] = dmul(row[j], s4[j]);
    }
    double s44 = dmul(m[0], m[0]);
    s44 = dfma(m[1], m[1], s44);
    s44 = dfma(m[2], m[2], s44);
    s44 = dfma(m[3], m[3], s44);
    const double dt = dsub((double)t_f, (double)mean.w);
    const double dt2 = dmul(dt, dt);
    const double kts = dmul(kKT, s44);
    if (!(dt2 <= kts)) return kTemporal;
    const double r44 = ddiv(1.0, s44);
    double h = dmul(dt2, r44);
    h = dmul(h, 0.5);
    const double Q = dsub((double)L, h);
    o.Q = Q;
    if (!(Q >= 0.0)) return kSupport;
    const double Lrows[3][4] = {{a, -b, -c, -d}, {b, a, -d, c}, {c, d, a, -b}};
    const double mu[3] = {(double)mean.x, (double)mean.y, (double)mean.z};
    double Nm[3][4];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double row[4], M[4];
        rotor_row(Lrows[k], Rm, row);
#pragma unroll
        for (int j = 0; j < 4; ++j) M[j] = dmul(row[j], s4[j]);
        double cc = dmul(M[0], m[0]);
        cc = dfma(M[1], m[1], cc);
        cc = dfma(M[2], m[2], cc);
        cc = dfma(M[3], m[3], cc);
        const double v = dmul(cc, r44);
        o.mu3[k] = dfma(v, dt, mu[k]);
#pragma unroll
        for (int j = 0; j < 4; ++j) Nm[k][j] = dfma(-v, m[j], M[j]);
    }
    const int PK[6] = {0, 0, 0, 1, 1, 2}, PL[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int e = 0; e < 6; ++e) {
        const int k = PK[e], l = PL[e];
        double acc = dmul(Nm[k][0], Nm[l][0]);
        acc = dfma(Nm[k][1], Nm[l][1], acc);
        acc = dfma(Nm[k][2], Nm[l][2], acc);
        acc = dfma(Nm[k][3], Nm[l][3], acc);
        o.cov3[e] = acc;
    }
    return kNear;
}

struct Proj {
    int px0, px1, py0, py1;
    uint32_t depth_bits;
    float u, v, Ap, Bp, Cp, Q2;
};

// EWA projection + near / cover culls + pixel AABB + fp32 record fields.
__device__ __forceinline__ int project_gaussian(const Slice &sl, const CamDev &cam, Proj &o) {
    double pc[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        double acc = dmul(cam.R[3 * r + 0], sl.mu3[0]);
        acc = dfma(cam.R[3 * r + 1], sl.mu3[1], acc);
        acc = dfma(cam.R[3 * r + 2], sl.mu3[2], acc);
        pc[r] = dadd(acc, cam.T[r]);
    }
    const double z = pc[2];
    if (!(z > cam.z_near)) return kNear;
    const double rz = ddiv(1.0, z);
    const double xz = dmul(pc[0], rz), yz = dmul(pc[1], rz);
    const double cxz = fmin(fmax(xz, -cam.limx), cam.limx);
    const double cyz = fmin(fmax(yz, -cam.limy), cam.limy);
    const double j00 = dmul(cam.fx, rz), j11 = dmul(cam.fy, rz);
    const double j02 = -dmul(dmul(cam.fx, cxz), rz), j12 = -dmul(dmul(cam.fy, cyz), rz);
    double Tm[2][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        Tm[0][k] = dfma(j02, cam.R[6 + k], dmul(j00, cam.R[k]));
        Tm[1][k] = dfma(j12, cam.R[6 + k], dmul(j11, cam.R[3 + k]));
    }
    const double S3[3][3] = {{sl.cov3[0], sl.cov3[1], sl.cov3[2]},
                             {sl.cov3[1], sl.cov3[3], sl.cov3[4]},
                             {sl.cov3[2], sl.cov3[4], sl.cov3[5]}};
    double U[2][3];
#pragma unroll
    for (int aa = 0; aa < 2; ++aa)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double acc = dmul(Tm[aa][0], S3[0][k]);
            acc = dfma(Tm[aa][1], S3[1][k], acc);
            acc = dfma(Tm[aa][2], S3[2][k], acc);
            U[aa][k] = acc;
        }
    double a2 = dmul(U[0][0], Tm[0][0]);
    a2 = dfma(U[0][1], Tm[0][1], a2);
    a2 = dfma(U[0][2], Tm[0][2], a2);
    a2 = dadd(a2, kDilation);
    double b2 = dmul(U[0][0], Tm[1][0]);
    b2 = dfma(U[0][1], Tm[1][1], b2);
    b2 = dfma(U[0][2], Tm[1][2], b2);
    double c2 = dmul(U[1][0], Tm[1][0]);
    c2 = dfma(U[1][1], Tm[1][1], c2);
    c2 = dfma(U[1][2], Tm[1][2], c2);
    c2 = dadd(c2, kDilation);
    const double bb = dmul(b2, b2);
    const double det = dfma(a2, c2, -bb);
    const double rdet = ddiv(1.0, det);
    const double A = dmul(c2, rdet), B = -dmul(b2, rdet), C = dmul(a2, rdet);
    const double u = dfma(cam.fx, xz, cam.cx), v = dfma(cam.fy, yz, cam.cy);
    const double q2 = dmul(2.0, sl.Q);
    const double hx = dfma(__dsqrt_rn(dmul(q2, a2)), kMarginMul, kMarginAdd);
    const double hy = dfma(__dsqrt_rn(dmul(q2, c2)), kMarginMul, kMarginAdd);
    double ex0 = ceil(dsub(dsub(u, hx), 0.5)), ex1 = floor(dsub(dadd(u, hx), 0.5));
    double ey0 = ceil(dsub(dsub(v, hy), 0.5)), ey1 = floor(dsub(dadd(v, hy), 0.5));
    ex0 = fmin(fmax(ex0, -kLim), kLim);
    ex1 = fmin(fmax(ex1, -kLim), kLim);
    ey0 = fmin(fmax(ey0, -kLim), kLim);
    ey1 = fmin(fmax(ey1, -kLim), kLim);
    int px0 = (int)ex0, px1 = (int)ex1, py0 = (int)ey0, py1 = (int)ey1;
    px0 = max(px0, 0);
    py0 = max(py0, 0);
    px1 = min(px1, cam.width - 1);
    py1 = min(py1, cam.height - 1);
    o.px0 = px0; o.px1 = px1; o.py0 = py0; o.py1 = py1;
    o.depth_bits = __float_as_uint(__double2float_rn(z));
    o.u = __double2float_rn(u);
    o.v = __double2float_rn(v);
    o.Ap = __double2float_rn(dmul(kCH, A));
    o.Bp = __double2float_rn(dmul(kC1, B));
    o.Cp = __double2float_rn(dmul(kCH, C));
    o.Q2 = __double2float_rn(dmul(kLog2e, sl.Q));
    if (!(px0 <= px1 && py0 <= py1)) return kCover;
    return kVisible;
}

// Tile cover of a visible Gaussian, binary64 from
// the binary32 record fields, pinned op sequence (identical list in the
// oracle: or_band_consts / or_band_tiles).
struct BandConsts {
    double dxm, dym, dyr, i2a, Qm;
};

__device__ __forceinline__ BandConsts band_consts(float fu, float fv, float fA, float fB, float fC, float fQ,
                                                  int px0, int px1, int py0, int py1) {
    const double u = fu, v = fv, Ap = fA, Bp = fB, Cp = fC, Q2 = fQ;
    const double X = fmax(fabs(dsub(dadd((double)px0, 0.5), u)), fabs(dsub(dadd((double)px1, 0.5), u)));
    const double Y = fmax(fabs(dsub(dadd((double)py0, 0.5), v)), fabs(dsub(dadd((double)py1, 0.5), v)));
    double mag = dmul(fabs(Ap), X);
    mag = dmul(mag, X);
    double t = dmul(fabs(Bp), X);
    mag = dfma(t, Y, mag);
    t = dmul(fabs(Cp), Y);
    mag = dfma(t, Y, mag);
    const double m = dfma(mag, 0x1p-12, 0x1p-10);
    BandConsts c;
    c.Qm = dadd(Q2, m);
    double K = dmul(4.0, Ap);
    K = dmul(K, Cp);
    K = dfma(-Bp, Bp, K);
    c.dxm = __dsqrt_rn(ddiv(dmul(dmul(-4.0, Cp), c.Qm), K));
    c.dym = __dsqrt_rn(ddiv(dmul(dmul(-4.0, Ap), c.Qm), K));
    c.dyr = -ddiv(dmul(Bp, c.dxm), dmul(2.0, Cp));
    c.i2a = ddiv(0.5, Ap);
    return c;
}

__device__ __forceinline__ double band_root(const BandConsts &c, double Ap, double Bp, double Cp, double dy,
                                            bool plus) {
    const double b = dmul(Bp, dy);
    double cc = dmul(Cp, dy);
    cc = dfma(cc, dy, c.Qm);
    double D = dmul(b, b);
    D = dfma(dmul(-4.0, Ap), cc, D);
    D = D > 0.0 ? D : 0.0;
    return plus ? dmul(dadd(-b, __dsqrt_rn(D)), c.i2a) : dmul(dsub(-b, __dsqrt_rn(D)), c.i2a);
}

__device__ __forceinline__ bool band_tiles(const BandConsts &c, float fu, float fv, float fA, float fB, float fC,
                                           int px0, int px1, int py0, int py1, int ty, int &txa, int &txb) {
    const double u = fu, v = fv, Ap = fA, Bp = fB, Cp = fC;
    int ja = 16 * ty, jb = 16 * ty + 15;
    ja = max(ja, py0);
    jb = min(jb, py1);
    if (ja > jb) return false;
    const double dya = dsub(dadd((double)ja, 0.5), v), dyb = dsub(dadd((double)jb, 0.5), v);
    if (dyb < -c.dym || dya > c.dym) return false;
    const double dyr = c.dyr, dyl = -c.dyr;
    const double xr = (dyr >= dya && dyr <= dyb) ? c.dxm : band_root(c, Ap, Bp, Cp, dyr < dya ? dya : dyb, false);
    const double xl = (dyl >= dya && dyl <= dyb) ? -c.dxm : band_root(c, Ap, Bp, Cp, dyl < dya ? dya : dyb, true);
    double ca = ceil(dsub(dadd(u, xl), 0.5)), cb = floor(dsub(dadd(u, xr), 0.5));
    if (ca < (double)px0) ca = (double)px0;
    if (cb > (double)px1) cb = (double)px1;
    if (ca > cb) return false;
    txa = ((int)ca) >> 4;
    txb = ((int)cb) >> 4;
    return true;
}

// Degree-3 SH colour c_i(d), value path in fp32: rgb = max(0, sum + 0.5).
__device__ __forceinline__ void sh_color(const float4 *__restrict__ sh4, float dx, float dy, float dz, float out[3]) {
    const float inv = rsqrtf(dx * dx + dy * dy + dz * dz);
    const float x = dx * inv, y = dy * inv, z = dz * inv;
    float c[48];
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const float4 w = __ldg(sh4 + k);
        c[4 * k] = w.x; c[4 * k + 1] = w.y; c[4 * k + 2] = w.z; c[4 * k + 3] = w.w;
    }
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    float Y[16];
    Y[0] = 0.28209479177387814f;
    Y[1] = -0.4886025119029199f * y;
    Y[2] = 0.4886025119029199f * z;
    Y[3] = -0.4886025119029199f * x;
    Y[4] = 1.0925484305920792f * xy;
    Y[5] = -1.0925484305920792f * yz;
    Y[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    Y[7] = -1.0925484305920792f * xz;
    Y[8] = 0.5462742152960396f * (xx - yy);
    Y[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    Y[10] = 2.890611442640554f * xy * z;
    Y[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    Y[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    Y[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    Y[14] = 1.445305721320277f * z * (xx - yy);
    Y[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        float acc = 0.5f;
#pragma unroll
        for (int k = 0; k < 16; ++k) acc = fmaf(Y[k], c[3 * k + ch], acc);
        out[ch] = fmaxf(acc, 0.0f);
    }
}

}  // namespace fdgs
