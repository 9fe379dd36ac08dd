/*
 * fdgs_oracle.c -- CPU ORACLE for the 4DGS-1K render hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2503_16422_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant generator with the
 * CUDA path (paper_2503_16422_b200/csrc/).
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n):
 *   - Eq. 1: conditional 3D Gaussian mu_{xyz|t}, Sigma_{xyz|t}
 *     of each 4D Gaussian with Sigma = R S S^T R^T, R = L(q_l) R(q_r).
 *   - Eq. 3: alpha_i = p_i(t) p(u,v|t) sigma_i with the
 *     unnormalised temporal marginal p_i(t) = exp(-(t-mu_t)^2 / (2 Sigma_44))
 *     (reading R1) and the EWA-projected 2D Gaussian (reading R2).
 *   - Eq. 2: I(u,v,t) = sum_i c_i(d) alpha_i prod_{j<i}(1-alpha_j)
 *     over Gaussians sorted by depth, evaluated PER PIXEL (no tiles).
 *   - Sec. 4.2.2: key-frame visibility masks (union over views)
 *     and the active set of a frame = union of the two bracketing masks;
 *     the paper-literal masks from the Eq. 2 blending weights.
 *   - Sec. 4.2.1: the spatial-temporal variation score
 *     (spatial term from the blending weights, S^TV from p2 / p1, gamma, both
 *     combine readings, the ablation variants).
 *   - P:483 (Ours-PP): SH read through a vector-quantised codebook.
 *
 * Pinned by tests/test_oracle_pins.py, tests/test_oracle_projection_pins.py
 * (off-axis projection, SH basis vs scipy, view direction) and
 * tests/test_oracle_stv.py; tools/mutate_oracle.py checks every listed
 * mutant of this file fails one of them.  No function is parity-unpinned.
 *
 * Numeric paths:
 *   - every DECISION (temporal/support/near/cover culls, pixel AABB, depth key,
 *     the fp32 record fields) is a pinned sequence of IEEE binary64 ops on the
 *     fp32 inputs, followed by RN conversion to binary32.  It is written out
 *     below op by op; the CUDA side implements the same list independently.
 *   - the per-pixel eligibility e2 >= 0 is a pinned binary32 chain on the
 *     fp32 record fields (fmaf placement fixed).
 *   - every VALUE (alpha, colour, transmittance, output rgb) is binary64,
 *     from the literal formulas of Eq. 2/3 (alpha = sigma * p_t * exp(-power)).
 *   - the termination test T(1-alpha) < 1e-4 is a value-path decision; at a
 *     knife edge (|T(1-alpha)/1e-4 - 1| < 1e-3) both outcomes are recorded
 *     (reading R17, "two-branch termination").
 *
 * Build: gcc -O2 -std=c11 -fPIC -shared -fopenmp -ffp-contract=off
 *        -fno-fast-math -o liboracle.so fdgs_oracle.c -lm
 * (-ffp-contract=off: no silent fma contraction; x86-64 SSE: no excess
 * precision.  fma()/fmaf() from glibc are correctly rounded.)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- inputs */
typedef struct {
    int32_t n;
    const float *mean;            /* [n][4] x,y,z,t                         */
    const float *scale;           /* [n][4] linear std-devs                  */
    const float *rot_l;           /* [n][4] unit quaternion (w,x,y,z)        */
    const float *rot_r;           /* [n][4]                                  */
    const float *opacity;         /* [n]    sigma                            */
    const float *log255_opacity;  /* [n]    L = fp32(ln(255 sigma))          */
    const float *sh;              /* [n][16][3], or the VQ codebook [K][16][3] */
    const uint16_t *sh_index;     /* VQ ("vector quantization on SH"):
                                     Gaussian i uses codebook entry sh_index[i];
                                     NULL = dense SH                             */
} or_scene;

typedef struct {
    int32_t width, height;
    float fx, fy, cx, cy;
    float R[9];                   /* world->camera, row-major                */
    float T[3];
    float z_near;
    float bg[3];
} or_camera;

/* Pinned constants (DESIGN.md Appendix "constants"). */
#define OR_KT      0x1.62a40fda3e3ccp+3   /* 2 ln 255: p_t >= 1/255 <=> dt^2 <= KT*S44 */
#define OR_LOG2E   0x1.71547652b82fep+0   /* log2(e)                                  */
#define OR_CH     -0x1.71547652b82fep-1   /* -log2(e)/2                               */
#define OR_C1     -0x1.71547652b82fep+0   /* -log2(e)                                 */
#define OR_DIL     0.3                    /* low-pass dilation, px^2                   */
#define OR_JCLAMP  1.3                    /* Jacobian clamp, x half-FOV tangent        */
#define OR_MARGIN_MUL (1.0 + 0x1p-10)
#define OR_MARGIN_ADD 0x1p-4
#define OR_ALPHA_MAX 0.99
#define OR_T_STOP    1e-4
#define OR_KNIFE     1e-3

/* Stages of the decision path (first failing cull). */
enum { ST_TEMPORAL = 0, ST_SUPPORT = 1, ST_NEAR = 2, ST_COVER = 3, ST_VISIBLE = 4 };

typedef struct {
    int32_t stage;
    int32_t px0, px1, py0, py1;
    uint32_t depth_bits;
    float f32[6];          /* u, v, A', B', C', Q2 (binary32 record fields) */
    /* binary64 values */
    double mu3[3], cov3[6], s44, dt;
    double cam[3];
    double cov2[3];        /* a (xx, dilated), b (xy), c (yy, dilated) */
    double conic[3];       /* A, B, C : power = 0.5(A dx^2 + 2B dx dy + C dy^2) */
    double u, v, Q;
    double amp;            /* sigma * p_t(t) (Eq. 3), value path */
    double rgb[3];
} or_gauss;

/* ------------------------------------------------ Sec. 3: 4D rotation
 * R4 = L(q_l) R(q_r); rows of L(a,b,c,d): (a,-b,-c,-d), (b,a,-d,c), (c,d,a,-b),
 * (d,-c,b,a); rows of R(p,q,r,s): (p,-q,-r,-s), (q,p,s,-r), (r,-s,p,q),
 * (s,r,-q,p).  Pinned: R4[i][j] = fma(L[i][3],R[3][j], fma(L[i][2],R[2][j],
 * fma(L[i][1],R[1][j], L[i][0]*R[0][j]))).                                   */
void or_rotor4(const float *ql, const float *qr, double *R4)
{
    const double a = ql[0], b = ql[1], c = ql[2], d = ql[3];
    const double p = qr[0], q = qr[1], r = qr[2], s = qr[3];
    const double Lm[4][4] = {{a, -b, -c, -d}, {b, a, -d, c}, {c, d, a, -b}, {d, -c, b, a}};
    const double Rm[4][4] = {{p, -q, -r, -s}, {q, p, s, -r}, {r, -s, p, q}, {s, r, -q, p}};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double acc = Lm[i][0] * Rm[0][j];
            acc = fma(Lm[i][1], Rm[1][j], acc);
            acc = fma(Lm[i][2], Rm[2][j], acc);
            acc = fma(Lm[i][3], Rm[3][j], acc);
            R4[i * 4 + j] = acc;
        }
}

/* --------------------------------------------- SH degree 3 ("c_i(d)")
 * Real SH basis with the splatting-ecosystem signs (reading R9),
 * constants written as their closed forms; rgb = max(0, sum Y_k sh_k + 0.5). */
void or_sh_basis(const double *d, double *Y)
{
    const double PI = 3.14159265358979323846;
    const double x = d[0], y = d[1], z = d[2];
    const double xx = x * x, yy = y * y, zz = z * z;
    Y[0] = 0.5 * sqrt(1.0 / PI);
    const double k1 = sqrt(3.0 / (4.0 * PI));
    Y[1] = -k1 * y;
    Y[2] = k1 * z;
    Y[3] = -k1 * x;
    const double k2a = sqrt(15.0 / (4.0 * PI)), k2b = sqrt(5.0 / (16.0 * PI)), k2c = sqrt(15.0 / (16.0 * PI));
    Y[4] = k2a * x * y;
    Y[5] = -k2a * y * z;
    Y[6] = k2b * (2.0 * zz - xx - yy);
    Y[7] = -k2a * x * z;
    Y[8] = k2c * (xx - yy);
    const double k3a = sqrt(35.0 / (32.0 * PI)), k3b = sqrt(105.0 / (4.0 * PI)),
                 k3c = sqrt(21.0 / (32.0 * PI)), k3d = sqrt(7.0 / (16.0 * PI)),
                 k3e = sqrt(105.0 / (16.0 * PI));
    Y[9] = -k3a * y * (3.0 * xx - yy);
    Y[10] = k3b * x * y * z;
    Y[11] = -k3c * y * (4.0 * zz - xx - yy);
    Y[12] = k3d * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    Y[13] = -k3c * x * (4.0 * zz - xx - yy);
    Y[14] = k3e * z * (xx - yy);
    Y[15] = -k3a * x * (xx - 3.0 * yy);
}

static void or_sh_rgb(const float *sh, const double d[3], double out[3])
{
    double Y[16];
    or_sh_basis(d, Y);
    for (int ch = 0; ch < 3; ++ch) {
        double acc = 0.0;
        for (int k = 0; k < 16; ++k) acc += Y[k] * (double)sh[k * 3 + ch];
        acc += 0.5;
        out[ch] = acc > 0.0 ? acc : 0.0;
    }
}

/* ------------------------------------------------ per-Gaussian decision path
 * Follows Eq. 1 + Eq. 3 + EWA projection (P:139
 * Sigma_2D, reading R6/R7).  Every op is listed in DESIGN.md "Decision path". */
void or_gauss_eval(const or_scene *S, int i, const or_camera *cam, float t_f, or_gauss *g)
{
    memset(g, 0, sizeof *g);
    const float *mu = S->mean + 4 * (size_t)i;
    const float *sc = S->scale + 4 * (size_t)i;
    double R4[16];
    or_rotor4(S->rot_l + 4 * (size_t)i, S->rot_r + 4 * (size_t)i, R4);
    /* M = R4 diag(s) */
    double M[4][4];
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) M[r][c] = R4[r * 4 + c] * (double)sc[c];
    const double m0 = M[3][0], m1 = M[3][1], m2 = M[3][2], m3 = M[3][3];
    /* Sigma_44 = m.m */
    double s44 = m0 * m0;
    s44 = fma(m1, m1, s44);
    s44 = fma(m2, m2, s44);
    s44 = fma(m3, m3, s44);
    const double t = (double)t_f;
    const double dt = t - (double)mu[3];
    const double dt2 = dt * dt;
    g->s44 = s44;
    g->dt = dt;
    /* temporal cull: p_t >= 1/255 <=> dt^2 <= 2 ln255 * Sigma_44 */
    const double kts = OR_KT * s44;
    if (!(dt2 <= kts)) { g->stage = ST_TEMPORAL; return; }
    const double r44 = 1.0 / s44;
    /* Sigma_{k,4} = M_k . m ; v = Sigma_{1:3,4} / Sigma_44 ; mu3 = mu + v dt */
    double v[3], Nm[3][4];
    for (int k = 0; k < 3; ++k) {
        double c = M[k][0] * m0;
        c = fma(M[k][1], m1, c);
        c = fma(M[k][2], m2, c);
        c = fma(M[k][3], m3, c);
        v[k] = c * r44;
        g->mu3[k] = fma(v[k], dt, (double)mu[k]);
        for (int j = 0; j < 4; ++j) Nm[k][j] = fma(-v[k], M[3][j], M[k][j]);
    }
    /* Sigma3 = N N^T  (projector form of the Schur complement of Eq. 1) */
    static const int PK[6] = {0, 0, 0, 1, 1, 2}, PL[6] = {0, 1, 2, 1, 2, 2};
    for (int e = 0; e < 6; ++e) {
        const int k = PK[e], l = PL[e];
        double acc = Nm[k][0] * Nm[l][0];
        acc = fma(Nm[k][1], Nm[l][1], acc);
        acc = fma(Nm[k][2], Nm[l][2], acc);
        acc = fma(Nm[k][3], Nm[l][3], acc);
        g->cov3[e] = acc;
    }
    /* Q = L - dt^2/(2 Sigma_44) = ln(255 sigma p_t) ; support cull Q >= 0 */
    double h = dt2 * r44;
    h = h * 0.5;
    const double Q = (double)S->log255_opacity[i] - h;
    g->Q = Q;
    if (!(Q >= 0.0)) { g->stage = ST_SUPPORT; return; }
    /* camera transform */
    double Rc[3][3], Tc[3];
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) Rc[r][c] = (double)cam->R[r * 3 + c];
        Tc[r] = (double)cam->T[r];
    }
    double pc[3];
    for (int r = 0; r < 3; ++r) {
        double acc = Rc[r][0] * g->mu3[0];
        acc = fma(Rc[r][1], g->mu3[1], acc);
        acc = fma(Rc[r][2], g->mu3[2], acc);
        pc[r] = acc + Tc[r];
        g->cam[r] = pc[r];
    }
    const double z = pc[2];
    if (!(z > (double)cam->z_near)) { g->stage = ST_NEAR; return; }
    const double fx = cam->fx, fy = cam->fy, cx = cam->cx, cy = cam->cy;
    const double rz = 1.0 / z;
    const double xz = pc[0] * rz, yz = pc[1] * rz;
    const double limx = OR_JCLAMP * ((double)cam->width / (2.0 * fx));
    const double limy = OR_JCLAMP * ((double)cam->height / (2.0 * fy));
    const double cxz = fmin(fmax(xz, -limx), limx);
    const double cyz = fmin(fmax(yz, -limy), limy);
    const double j00 = fx * rz, j11 = fy * rz;
    const double j02 = -((fx * cxz) * rz), j12 = -((fy * cyz) * rz);
    /* Tm = J Rc (2x3) */
    double Tm[2][3];
    for (int k = 0; k < 3; ++k) {
        Tm[0][k] = fma(j02, Rc[2][k], j00 * Rc[0][k]);
        Tm[1][k] = fma(j12, Rc[2][k], j11 * Rc[1][k]);
    }
    /* U = Tm Sigma3 (2x3); Sigma2 = U Tm^T + 0.3 I */
    const double S3[3][3] = {{g->cov3[0], g->cov3[1], g->cov3[2]},
                             {g->cov3[1], g->cov3[3], g->cov3[4]},
                             {g->cov3[2], g->cov3[4], g->cov3[5]}};
    double U[2][3];
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k) {
            double acc = Tm[a][0] * S3[0][k];
            acc = fma(Tm[a][1], S3[1][k], acc);
            acc = fma(Tm[a][2], S3[2][k], acc);
            U[a][k] = acc;
        }
    double a2 = U[0][0] * Tm[0][0];
    a2 = fma(U[0][1], Tm[0][1], a2);
    a2 = fma(U[0][2], Tm[0][2], a2);
    a2 = a2 + OR_DIL;
    double b2 = U[0][0] * Tm[1][0];
    b2 = fma(U[0][1], Tm[1][1], b2);
    b2 = fma(U[0][2], Tm[1][2], b2);
    double c2 = U[1][0] * Tm[1][0];
    c2 = fma(U[1][1], Tm[1][1], c2);
    c2 = fma(U[1][2], Tm[1][2], c2);
    c2 = c2 + OR_DIL;
    g->cov2[0] = a2; g->cov2[1] = b2; g->cov2[2] = c2;
    const double bb = b2 * b2;
    const double det = fma(a2, c2, -bb);
    const double rdet = 1.0 / det;
    const double A = c2 * rdet, B = -(b2 * rdet), C = a2 * rdet;
    g->conic[0] = A; g->conic[1] = B; g->conic[2] = C;
    const double u = fma(fx, xz, cx), vv = fma(fy, yz, cy);
    g->u = u; g->v = vv;
    /* pixel AABB of {power <= Q}: |dx| <= sqrt(2 Q a2), with margin */
    const double q2 = 2.0 * Q;
    const double hx = fma(sqrt(q2 * a2), OR_MARGIN_MUL, OR_MARGIN_ADD);
    const double hy = fma(sqrt(q2 * c2), OR_MARGIN_MUL, OR_MARGIN_ADD);
    double ex0 = ceil((u - hx) - 0.5), ex1 = floor((u + hx) - 0.5);
    double ey0 = ceil((vv - hy) - 0.5), ey1 = floor((vv + hy) - 0.5);
    const double LIM = 0x1p30;
    ex0 = fmin(fmax(ex0, -LIM), LIM); ex1 = fmin(fmax(ex1, -LIM), LIM);
    ey0 = fmin(fmax(ey0, -LIM), LIM); ey1 = fmin(fmax(ey1, -LIM), LIM);
    int px0 = (int)ex0, px1 = (int)ex1, py0 = (int)ey0, py1 = (int)ey1;
    if (px0 < 0) px0 = 0;
    if (py0 < 0) py0 = 0;
    if (px1 > cam->width - 1) px1 = cam->width - 1;
    if (py1 > cam->height - 1) py1 = cam->height - 1;
    g->px0 = px0; g->px1 = px1; g->py0 = py0; g->py1 = py1;
    {
        float zf = (float)z;
        uint32_t bits;
        memcpy(&bits, &zf, 4);
        g->depth_bits = bits;
    }
    g->f32[0] = (float)u;
    g->f32[1] = (float)vv;
    g->f32[2] = (float)(OR_CH * A);
    g->f32[3] = (float)(OR_C1 * B);
    g->f32[4] = (float)(OR_CH * C);
    g->f32[5] = (float)(OR_LOG2E * Q);
    if (!(px0 <= px1 && py0 <= py1)) { g->stage = ST_COVER; return; }
    g->stage = ST_VISIBLE;
    /* value path: amp = sigma * p_t (Eq. 3), colour c_i(d) (Eq. 2) */
    g->amp = (double)S->opacity[i] * exp(-(dt * dt) / (2.0 * s44));
    double ccam[3], d[3];
    for (int k = 0; k < 3; ++k)
        ccam[k] = -(Rc[0][k] * Tc[0] + Rc[1][k] * Tc[1] + Rc[2][k] * Tc[2]);
    for (int k = 0; k < 3; ++k) d[k] = g->mu3[k] - ccam[k];
    const double nd = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int k = 0; k < 3; ++k) d[k] /= nd;
    or_sh_rgb(S->sh + 48 * (size_t)(S->sh_index ? S->sh_index[i] : i), d, g->rgb);
}

/* Exported: decision records for all Gaussians (mask not applied).
 * f64 layout per Gaussian (OR_REC64 doubles): mu3[3] cov3[6] s44 Q amp rgb[3]
 * cam[3] u v cov2[3] conic[3]. */
#define OR_REC64 26
void or_records(const or_scene *S, const or_camera *cam, float t,
                int32_t *stage, int32_t *rect4, uint32_t *depth_bits, float *f32x6,
                double *f64x26)
{
#pragma omp parallel for schedule(static)
    for (int i = 0; i < S->n; ++i) {
        or_gauss g;
        or_gauss_eval(S, i, cam, t, &g);
        stage[i] = g.stage;
        if (rect4) { rect4[4 * i] = g.px0; rect4[4 * i + 1] = g.px1; rect4[4 * i + 2] = g.py0; rect4[4 * i + 3] = g.py1; }
        if (depth_bits) depth_bits[i] = g.depth_bits;
        if (f32x6) memcpy(f32x6 + 6 * (size_t)i, g.f32, sizeof g.f32);
        if (f64x26) {
            double *o = f64x26 + OR_REC64 * (size_t)i;
            o[0] = g.mu3[0]; o[1] = g.mu3[1]; o[2] = g.mu3[2];
            memcpy(o + 3, g.cov3, 6 * sizeof(double));
            o[9] = g.s44; o[10] = g.Q; o[11] = g.amp;
            o[12] = g.rgb[0]; o[13] = g.rgb[1]; o[14] = g.rgb[2];
            o[15] = g.cam[0]; o[16] = g.cam[1]; o[17] = g.cam[2];
            o[18] = g.u; o[19] = g.v;
            o[20] = g.cov2[0]; o[21] = g.cov2[1]; o[22] = g.cov2[2];
            o[23] = g.conic[0]; o[24] = g.conic[1]; o[25] = g.conic[2];
        }
    }
}

/* ------------------------------------------------------- canonical order  */
typedef struct { uint32_t key; int32_t idx; } or_key;
static int or_key_cmp(const void *a, const void *b)
{
    const or_key *x = a, *y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

static inline int or_mask_bit(const uint32_t *mask, int i)
{
    return mask == NULL ? 1 : (int)((mask[i >> 5] >> (i & 31)) & 1u);
}

/* Evaluate all Gaussians; return visible (active & stage==VISIBLE) in canonical
 * order (ascending (depth bits, index); reading R8). */
static or_gauss *or_visible(const or_scene *S, const uint32_t *mask, const or_camera *cam,
                            float t, int *n_vis_out, int *n_act_out)
{
    or_gauss *all = (or_gauss *)malloc(sizeof(or_gauss) * (size_t)(S->n > 0 ? S->n : 1));
    int n_act = 0;
#pragma omp parallel for schedule(static) reduction(+ : n_act)
    for (int i = 0; i < S->n; ++i) {
        if (!or_mask_bit(mask, i)) { all[i].stage = -1; continue; }
        n_act += 1;
        or_gauss_eval(S, i, cam, t, &all[i]);
    }
    int nv = 0;
    for (int i = 0; i < S->n; ++i) nv += all[i].stage == ST_VISIBLE;
    or_key *keys = (or_key *)malloc(sizeof(or_key) * (size_t)(nv > 0 ? nv : 1));
    int k = 0;
    for (int i = 0; i < S->n; ++i)
        if (all[i].stage == ST_VISIBLE) { keys[k].key = all[i].depth_bits; keys[k].idx = i; ++k; }
    qsort(keys, (size_t)nv, sizeof(or_key), or_key_cmp);
    or_gauss *vis = (or_gauss *)malloc(sizeof(or_gauss) * (size_t)(nv > 0 ? nv : 1));
    int *ids = (int *)malloc(sizeof(int) * (size_t)(nv > 0 ? nv : 1));
    for (int j = 0; j < nv; ++j) { vis[j] = all[keys[j].idx]; ids[j] = keys[j].idx; }
    /* stash the Gaussian index in the (unused) stage field of the copy */
    for (int j = 0; j < nv; ++j) vis[j].stage = ids[j];
    free(ids);
    free(keys);
    free(all);
    *n_vis_out = nv;
    if (n_act_out) *n_act_out = n_act;
    return vis;
}

/* Exported: canonical visible order (Gaussian indices) + count. */
int or_canonical_order(const or_scene *S, const uint32_t *mask, const or_camera *cam, float t,
                       int32_t *out_ids, int32_t cap)
{
    int nv, na;
    or_gauss *vis = or_visible(S, mask, cam, t, &nv, &na);
    for (int j = 0; j < nv && j < cap; ++j) out_ids[j] = vis[j].stage;
    free(vis);
    return nv;
}

/* Tile cover of a visible Gaussian.  Per Gaussian,
 * in binary64 from the binary32 record fields: the margin m = 2^-12 (|A'|X^2 +
 * |B'|XY + |C'|Y^2) + 2^-10 over its pixel AABB (X, Y the largest |dx|, |dy|),
 * Qm = Q2 + m, K = 4A'C' - B'^2 > 0, the half extents dxm = sqrt(-4C'Qm/K),
 * dym = sqrt(-4A'Qm/K) of the m-inflated ellipse e2 >= -m, the dy of its
 * rightmost point dyr = -B'dxm/(2C') (leftmost: -dyr) and 1/(2A').
 * c[0..4] = dxm, dym, dyr, i2a, Qm. */
void or_band_consts(const float *f32, int px0, int px1, int py0, int py1, double *c)
{
    const double u = f32[0], v = f32[1], Ap = f32[2], Bp = f32[3], Cp = f32[4], Q2 = f32[5];
    const double X = fmax(fabs(((double)px0 + 0.5) - u), fabs(((double)px1 + 0.5) - u));
    const double Y = fmax(fabs(((double)py0 + 0.5) - v), fabs(((double)py1 + 0.5) - v));
    double mag = fabs(Ap) * X;
    mag = mag * X;
    double t = fabs(Bp) * X;
    mag = fma(t, Y, mag);
    t = fabs(Cp) * Y;
    mag = fma(t, Y, mag);
    const double m = fma(mag, 0x1p-12, 0x1p-10);
    const double Qm = Q2 + m;
    double K = 4.0 * Ap;
    K = K * Cp;
    K = fma(-Bp, Bp, K);                         /* 4A'C' - B'^2 > 0 */
    c[0] = sqrt(((-4.0 * Cp) * Qm) / K);
    c[1] = sqrt(((-4.0 * Ap) * Qm) / K);
    c[2] = -(Bp * c[0]) / (2.0 * Cp);
    c[3] = 0.5 / Ap;
    c[4] = Qm;
}

/* Tiles [*txa, *txb] of tile row ty reached by the m-inflated ellipse: the
 * band is empty iff it misses the y-range [-dym, dym]; else the x-extent over
 * the band is +-dxm where the extreme point's dy lies in the band, else the
 * root at the band edge nearest to it; pixel columns clamped to the AABB.
 * Returns 0 if no tile.  The margin exceeds the rounding of the pinned fp32
 * e2 chain, so every pixel with e2 >= 0 lies in a covered tile. */
static double or_band_root(const double *c, double Ap, double Bp, double Cp, double dy, double sgn)
{
    const double b = Bp * dy;
    double cc = Cp * dy;
    cc = fma(cc, dy, c[4]);
    double D = b * b;
    D = fma(-4.0 * Ap, cc, D);
    D = D > 0.0 ? D : 0.0;
    return sgn > 0.0 ? (-b + sqrt(D)) * c[3] : (-b - sqrt(D)) * c[3];
}

int or_band_tiles(const float *f32, int px0, int px1, int py0, int py1, const double *c, int ty, int *txa,
                  int *txb)
{
    const double u = f32[0], v = f32[1], Ap = f32[2], Bp = f32[3], Cp = f32[4];
    int ja = 16 * ty, jb = 16 * ty + 15;
    if (ja < py0) ja = py0;
    if (jb > py1) jb = py1;
    if (ja > jb) return 0;
    const double dya = ((double)ja + 0.5) - v, dyb = ((double)jb + 0.5) - v;
    if (dyb < -c[1] || dya > c[1]) return 0;       /* band misses the y-range */
    const double dyr = c[2], dyl = -c[2];
    const double xr = (dyr >= dya && dyr <= dyb) ? c[0] : or_band_root(c, Ap, Bp, Cp, dyr < dya ? dya : dyb, -1.0);
    const double xl = (dyl >= dya && dyl <= dyb) ? -c[0] : or_band_root(c, Ap, Bp, Cp, dyl < dya ? dya : dyb, 1.0);
    double ca = ceil((u + xl) - 0.5), cb = floor((u + xr) - 0.5);
    if (ca < (double)px0) ca = (double)px0;
    if (cb > (double)px1) cb = (double)px1;
    if (ca > cb) return 0;
    *txa = ((int)ca) >> 4;
    *txb = ((int)cb) >> 4;
    return 1;
}

/* Exported: per-tile lists (16x16 tiles, tile id = ty*ceil(W/16)+tx) in
 * canonical order: each visible Gaussian appended, in canonical order, to
 * every tile of its tile cover (or_band_tiles per tile row of its pixel
 * AABB).  ranges[2*tile] = [start, end). */
int64_t or_tile_lists(const or_scene *S, const uint32_t *mask, const or_camera *cam, float t,
                      int64_t *ranges, int32_t *ids, int64_t cap)
{
    int nv, na;
    or_gauss *vis = or_visible(S, mask, cam, t, &nv, &na);
    const int tw = (cam->width + 15) / 16, th = (cam->height + 15) / 16, nt = tw * th;
    int64_t *cnt = (int64_t *)calloc((size_t)nt, sizeof(int64_t));
    double *bc = (double *)malloc(sizeof(double) * 5 * (size_t)(nv > 0 ? nv : 1));
    for (int j = 0; j < nv; ++j) or_band_consts(vis[j].f32, vis[j].px0, vis[j].px1, vis[j].py0, vis[j].py1, bc + 5 * j);
    for (int j = 0; j < nv; ++j)
        for (int ty = vis[j].py0 / 16; ty <= vis[j].py1 / 16; ++ty) {
            int a, b;
            if (!or_band_tiles(vis[j].f32, vis[j].px0, vis[j].px1, vis[j].py0, vis[j].py1, bc + 5 * j, ty, &a, &b))
                continue;
            for (int tx = a; tx <= b; ++tx) cnt[ty * tw + tx]++;
        }
    int64_t total = 0;
    for (int k = 0; k < nt; ++k) { ranges[2 * k] = total; total += cnt[k]; ranges[2 * k + 1] = total; cnt[k] = ranges[2 * k]; }
    if (total <= cap)
        for (int j = 0; j < nv; ++j)
            for (int ty = vis[j].py0 / 16; ty <= vis[j].py1 / 16; ++ty) {
                int a, b;
                if (!or_band_tiles(vis[j].f32, vis[j].px0, vis[j].px1, vis[j].py0, vis[j].py1, bc + 5 * j, ty, &a,
                                   &b))
                    continue;
                for (int tx = a; tx <= b; ++tx) ids[cnt[ty * tw + tx]++] = vis[j].stage;
            }
    free(bc);
    free(cnt);
    free(vis);
    return total;
}

/* ---------------------------------------------------- per-pixel compositing */
typedef struct {
    int32_t px0, px1;
    int32_t txa, txb;      /* tile cover of this row band (-1,-2 if empty) */
    int32_t gid;           /* Gaussian index */
    float u, v, Ap, Bp, Cp, Q2;
    double u64, v64, A, B, C, amp, rgb[3];
} or_cand;

/* e2 = log2(255 * alpha_unclamped) in binary32, pinned chain. */
static inline float or_e2(const or_cand *c, float pxf, float pyf)
{
    const float dx = pxf - c->u;
    const float dy = pyf - c->v;
    const float t1 = c->Bp * dy;
    const float t2 = fmaf(c->Ap, dx, t1);
    const float t3 = c->Cp * dy;
    const float t4 = fmaf(t3, dy, c->Q2);
    return fmaf(dx, t2, t4);
}

#define OR_MAX_LEAVES 4
#define OR_MAX_DEPTH 2
typedef struct {
    double prim_C[3], prim_T;
    int n_alt;
    double alt_C[OR_MAX_LEAVES][3], alt_T[OR_MAX_LEAVES];
    int64_t evaluated, blended;
    int knife;
    double *contrib;       /* per-Gaussian blending weights (nullable, primary path) */
} or_pix;

static void or_leaf(or_pix *P, int primary, const double C[3], double T)
{
    if (primary) { P->prim_C[0] = C[0]; P->prim_C[1] = C[1]; P->prim_C[2] = C[2]; P->prim_T = T; return; }
    if (P->n_alt >= OR_MAX_LEAVES) return;
    for (int c = 0; c < 3; ++c) P->alt_C[P->n_alt][c] = C[c];
    P->alt_T[P->n_alt] = T;
    P->n_alt++;
}

/* Eq. 2 front-to-back over the row candidates (canonical order). */
static void or_composite(const or_cand *cand, int nc, int k0, int i, float pxf, float pyf, double px, double py,
                         double T, const double Cin[3], int depth, int primary, or_pix *P)
{
    double C[3] = {Cin[0], Cin[1], Cin[2]};
    for (int k = k0; k < nc; ++k) {
        const or_cand *c = &cand[k];
        if (i < c->px0 || i > c->px1) continue;
        if (primary && (i >> 4) >= c->txa && (i >> 4) <= c->txb) P->evaluated++;  /* work in covered tiles */
        if (!(or_e2(c, pxf, pyf) >= 0.0f)) continue;
        const double dx = px - c->u64, dy = py - c->v64;
        const double power = 0.5 * (c->A * dx * dx + 2.0 * c->B * dx * dy + c->C * dy * dy);
        double alpha = c->amp * exp(-power);
        if (alpha > OR_ALPHA_MAX) alpha = OR_ALPHA_MAX;
        const double test = T * (1.0 - alpha);
        const int stop = test < OR_T_STOP;
        const int knife = fabs(test / OR_T_STOP - 1.0) < OR_KNIFE;
        if (knife && primary) P->knife++;
        if (knife && depth < OR_MAX_DEPTH) {
            if (stop) {     /* alternative: continue past this Gaussian */
                double C2[3];
                for (int ch = 0; ch < 3; ++ch) C2[ch] = C[ch] + c->rgb[ch] * alpha * T;
                or_composite(cand, nc, k + 1, i, pxf, pyf, px, py, test, C2, depth + 1, 0, P);
            } else {        /* alternative: stop here without blending it */
                or_leaf(P, 0, C, T);
            }
        }
        if (stop) { or_leaf(P, primary, C, T); return; }
        for (int ch = 0; ch < 3; ++ch) C[ch] += c->rgb[ch] * alpha * T;
        if (primary && P->contrib) P->contrib[c->gid] += alpha * T;   /* S^S term of P:251 */
        T = test;
        if (primary) P->blended++;
    }
    or_leaf(P, primary, C, T);
}

/* Exported: per-pixel render of Eq. 2.
 * pix: optional list of n_pix flat pixel indices (y*W+x); NULL = all pixels in
 * row-major order (n_pix ignored).  Outputs per listed pixel:
 *   rgb[3*k..]   primary branch   C + T*bg
 *   T[k]         primary final transmittance
 *   alt_rgb[OR_MAX_LEAVES*3*k..] alternative admissible results, n_alt[k] of them
 * stats[0]=n_act stats[1]=n_vis stats[2]=evaluated pairs (in the pixel AABB and a
 * covered tile, before termination: the Eq. 2 work) stats[3]=blended
 * stats[4]=knife-edge decisions.  Returns 0. */
static int or_render_impl(const or_scene *S, const uint32_t *mask, const or_camera *cam, float t,
                          const int64_t *pix, int64_t n_pix, double *rgb, double *T_out, double *alt_rgb,
                          int32_t *n_alt, int64_t *stats, double *contrib);

int or_render(const or_scene *S, const uint32_t *mask, const or_camera *cam, float t,
              const int64_t *pix, int64_t n_pix,
              double *rgb, double *T_out, double *alt_rgb, int32_t *n_alt, int64_t *stats)
{
    return or_render_impl(S, mask, cam, t, pix, n_pix, rgb, T_out, alt_rgb, n_alt, stats, NULL);
}

/* Exported: per-Gaussian sum over all pixels of the blending weight
 * alpha_i prod_{j<i}(1-alpha_j) of one view at t (the spatial score term of
 * P:249-253), added into contrib[n] (binary64). */
int or_contrib(const or_scene *S, const or_camera *cam, float t, double *contrib)
{
    return or_render_impl(S, NULL, cam, t, NULL, 0, NULL, NULL, NULL, NULL, NULL, contrib);
}

static int or_render_impl(const or_scene *S, const uint32_t *mask, const or_camera *cam, float t,
                          const int64_t *pix, int64_t n_pix, double *rgb, double *T_out, double *alt_rgb,
                          int32_t *n_alt, int64_t *stats, double *contrib)
{
    const int W = cam->width, H = cam->height;
    int nv, na;
    or_gauss *vis = or_visible(S, mask, cam, t, &nv, &na);
    const int64_t npx = pix ? n_pix : (int64_t)W * H;
    /* rows that are requested */
    char *need = (char *)calloc((size_t)H, 1);
    for (int64_t k = 0; k < npx; ++k) need[pix ? (int)(pix[k] / W) : (int)(k / W)] = 1;
    /* row -> list of requested pixel slots */
    int64_t *row_start = (int64_t *)calloc((size_t)H + 1, sizeof(int64_t));
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(npx > 0 ? npx : 1));
    for (int64_t k = 0; k < npx; ++k) row_start[(pix ? pix[k] / W : k / W) + 1]++;
    for (int r = 0; r < H; ++r) row_start[r + 1] += row_start[r];
    {
        int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)H);
        memcpy(fill, row_start, sizeof(int64_t) * (size_t)H);
        for (int64_t k = 0; k < npx; ++k) order[fill[pix ? pix[k] / W : k / W]++] = k;
        free(fill);
    }
    int64_t evaluated = 0, blended = 0, knife = 0;
#pragma omp parallel reduction(+ : evaluated, blended, knife)
    {
        or_cand *cand = (or_cand *)malloc(sizeof(or_cand) * (size_t)(nv > 0 ? nv : 1));
        double *my_contrib = contrib ? (double *)calloc((size_t)(S->n > 0 ? S->n : 1), sizeof(double)) : NULL;
#pragma omp for schedule(dynamic, 1)
        for (int j = 0; j < H; ++j) {
            if (!need[j]) continue;
            int nc = 0;
            for (int q = 0; q < nv; ++q) {      /* candidates covering row j, canonical order */
                const or_gauss *g = &vis[q];
                if (j < g->py0 || j > g->py1) continue;
                or_cand *c = &cand[nc++];
                c->px0 = g->px0; c->px1 = g->px1;
                c->gid = g->stage;
                double bcq[5];
                or_band_consts(g->f32, g->px0, g->px1, g->py0, g->py1, bcq);
                if (!or_band_tiles(g->f32, g->px0, g->px1, g->py0, g->py1, bcq, j >> 4, &c->txa, &c->txb)) {
                    c->txa = -1;
                    c->txb = -2;
                }
                c->u = g->f32[0]; c->v = g->f32[1]; c->Ap = g->f32[2]; c->Bp = g->f32[3]; c->Cp = g->f32[4]; c->Q2 = g->f32[5];
                c->u64 = g->u; c->v64 = g->v; c->A = g->conic[0]; c->B = g->conic[1]; c->C = g->conic[2];
                c->amp = g->amp; c->rgb[0] = g->rgb[0]; c->rgb[1] = g->rgb[1]; c->rgb[2] = g->rgb[2];
            }
            const float pyf = (float)j + 0.5f;
            for (int64_t s = row_start[j]; s < row_start[j + 1]; ++s) {
                const int64_t k = order[s];
                const int64_t flat = pix ? pix[k] : k;
                const int i = (int)(flat % W);
                or_pix P;
                memset(&P, 0, sizeof P);
                P.contrib = my_contrib;
                const double C0[3] = {0.0, 0.0, 0.0};
                or_composite(cand, nc, 0, i, (float)i + 0.5f, pyf, i + 0.5, j + 0.5, 1.0, C0, 0, 1, &P);
                if (rgb)
                    for (int ch = 0; ch < 3; ++ch) rgb[3 * k + ch] = P.prim_C[ch] + P.prim_T * (double)cam->bg[ch];
                if (T_out) T_out[k] = P.prim_T;
                if (n_alt) n_alt[k] = P.n_alt;
                if (alt_rgb)
                    for (int a = 0; a < OR_MAX_LEAVES; ++a)
                        for (int ch = 0; ch < 3; ++ch)
                            alt_rgb[(k * OR_MAX_LEAVES + a) * 3 + ch] =
                                a < P.n_alt ? P.alt_C[a][ch] + P.alt_T[a] * (double)cam->bg[ch] : NAN;
                evaluated += P.evaluated;
                blended += P.blended;
                knife += P.knife;
            }
        }
        free(cand);
        if (my_contrib) {
#pragma omp critical
            for (int q = 0; q < S->n; ++q) contrib[q] += my_contrib[q];
            free(my_contrib);
        }
    }
    if (stats) { stats[0] = na; stats[1] = nv; stats[2] = evaluated; stats[3] = blended; stats[4] = knife; }
    free(order);
    free(row_start);
    free(need);
    free(vis);
    return 0;
}

/* ------------------------------------------------------- Sec. 4.2.2
 * Key-frame mask: bit i = OR over cameras of visible(i, cam, t_key), where
 * visible = temporal & support & near & cover culls of the decision path
 * (reading R3).  Words are LSB-first: bit i of word i/32.        */
void or_keyframe_mask(const or_scene *S, const or_camera *cams, int32_t n_cams, float t_key, uint32_t *out)
{
    const int nw = (S->n + 31) / 32;
#pragma omp parallel for schedule(static)
    for (int w = 0; w < nw; ++w) {
        uint32_t word = 0;
        for (int b = 0; b < 32; ++b) {
            const int i = w * 32 + b;
            if (i >= S->n) break;
            for (int c = 0; c < n_cams; ++c) {
                or_gauss g;
                or_gauss_eval(S, i, &cams[c], t_key, &g);
                if (g.stage == ST_VISIBLE) { word |= 1u << b; break; }
            }
        }
        out[w] = word;
    }
}

/* Sec. 4.2.2 read literally (reading R3b):
 * m_{i,j} = {Gaussians whose blending weights of Eq. 2 in the view-j render at
 * t_key sum to more than `threshold`}, the stored mask the
 * union over the views.  Unmasked renders, primary termination branch. */
void or_keyframe_mask_contrib(const or_scene *S, const or_camera *cams, int32_t n_cams, float t_key,
                              double threshold, uint32_t *out)
{
    const int n = S->n;
    const int nw = (n + 31) / 32;
    for (int w = 0; w < nw; ++w) out[w] = 0;
    double *c = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int j = 0; j < n_cams; ++j) {
        for (int i = 0; i < n; ++i) c[i] = 0.0;
        or_contrib(S, &cams[j], t_key, c);
        for (int i = 0; i < n; ++i)
            if (c[i] > threshold) out[i >> 5] |= 1u << (i & 31);
    }
    free(c);
}

/* Sec. 4.2.1 "Pruning": "All 4D Gaussians are ranked based on their
 * spatial-temporal variation score S_i, and Gaussians with lower scores are
 * pruned."  The kept set is the `keep` highest scores; equal scores are ranked
 * by ascending index (reading R23).  out: bitmask (LSB-first words)
 * of the kept Gaussians. */
static const float *or_prune_scores;
static int or_cmp_rank(const void *a, const void *b)
{
    const int i = *(const int *)a, j = *(const int *)b;
    const float x = or_prune_scores[i], y = or_prune_scores[j];
    if (x != y) return x > y ? -1 : 1;  /* higher score first */
    return (i > j) - (i < j);           /* then lower index   */
}

void or_prune_mask(const float *score, int32_t n, int64_t keep, uint32_t *out)
{
    const int nw = (n + 31) / 32;
    for (int w = 0; w < nw; ++w) out[w] = 0;
    int *idx = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) idx[i] = i;
    or_prune_scores = score;
    qsort(idx, (size_t)n, sizeof(int), or_cmp_rank);
    for (int64_t r = 0; r < keep && r < n; ++r) out[idx[r] >> 5] |= 1u << (idx[r] & 31);
    free(idx);
}

/* Sec. 4.2.2: key-frame schedule and bracketing. */
int or_keyframes(int32_t frames, int32_t interval, int32_t *out)
{
    int k = 0;
    for (int f = 0; f < frames; f += interval) out[k++] = f;
    if (out[k - 1] != frames - 1) out[k++] = frames - 1;
    return k;
}

void or_bracket(const int32_t *kf, int32_t nk, int32_t frame, int32_t *l, int32_t *r)
{
    int li = 0, ri = nk - 1;
    for (int k = 0; k < nk; ++k) if (kf[k] <= frame) li = k;
    for (int k = nk - 1; k >= 0; --k) if (kf[k] >= frame) ri = k;
    if (frame < kf[0]) li = 0;
    if (frame > kf[nk - 1]) ri = nk - 1;
    *l = li;
    *r = ri;
}

void or_mask_or(const uint32_t *a, const uint32_t *b, int32_t n, uint32_t *out)
{
    const int nw = (n + 31) / 32;
    for (int w = 0; w < nw; ++w) out[w] = a[w] | b[w];
}

/* ------------------------------------------------ Sec. 4.2.1
 * Spatial-temporal variation score, time-aligned (reading R20):
 *   S^S_i(t)  = sum over the views and pixels of alpha_i prod_{j<i}(1-alpha_j)
 *               (or_contrib, the renderer's blending weights),
 *   p2_i(t)   = ((t-mu_t)^2/Sigma_t^2 - 1/Sigma_t) p_i(t),
 *   S^TV_i(t) = 1 / (0.5 tanh|p2_i(t)| + 0.5),
 *   gamma_i   = min(V_i / V_p, 1), V_i = s_x s_y s_z s_t (binary32,
 *               left to right), V_p the nearest-rank `percentile` of V
 *               ("normalized following LightGaussian"),
 *   S_i       = sum_t S^TV_i(t) gamma_i S^S_i(t)
 *               (mode 0, time-aligned, reading R20), or
 *   S_i       = gamma_i (sum_t S^TV_i(t)) (sum_t S^S_i(t))           (mode 1: the
 *               literal product of the two sums, S^TV of P:264 already summed
 *               over t and S_i of P:270 summing S^T S^S again).
 * Outputs (nullable except score): score[n], spatial[n_ts][n], tv[n_ts][n],
 * gamma[n]. */
static int or_cmp_float(const void *a, const void *b)
{
    const float x = *(const float *)a, y = *(const float *)b;
    return (x > y) - (x < y);
}

double or_sigma_t(const or_scene *S, int i)
{
    double R4[16];
    or_rotor4(S->rot_l + 4 * (size_t)i, S->rot_r + 4 * (size_t)i, R4);
    double s44 = 0.0;
    for (int j = 0; j < 4; ++j) {
        const double m = R4[12 + j] * (double)S->scale[4 * (size_t)i + j];
        s44 += m * m;
    }
    return s44;
}

double or_tv(double t, double mu_t, double st)
{
    const double dt = t - mu_t;
    const double p = exp(-(dt * dt) / (2.0 * st));
    const double p2 = ((dt * dt) / (st * st) - 1.0 / st) * p;
    return 1.0 / (0.5 * tanh(fabs(p2)) + 0.5);
}

/* Ablation variant (d) of P:653-660: S^TV from the first derivative
 * p1_i(t) = -((t - mu_t) / Sigma_t) p_i(t) instead of p2. */
double or_tv_p1(double t, double mu_t, double st)
{
    const double dt = t - mu_t;
    const double p = exp(-(dt * dt) / (2.0 * st));
    const double p1 = -(dt / st) * p;
    return 1.0 / (0.5 * tanh(fabs(p1)) + 0.5);
}

float or_volume(const or_scene *S, int i)
{
    const float *s = S->scale + 4 * (size_t)i;
    float v = s[0] * s[1];
    v = v * s[2];
    v = v * s[3];
    return v;
}

/* variant (the score ablations of P:636-669, Table ablation_score):
 *   0 full      S_i(t) terms: T = S^TV(p2) gamma,  S = S^S
 *   1 S^S only  T = 1,                            S = S^S
 *   2 S^T only  T = S^TV(p2) gamma,               S = 1
 *   3 w. p1     T = S^TV(p1) gamma,               S = S^S
 *   4 w. Sigma_t T = Sigma_t gamma,               S = S^S
 * mode 0: S_i = sum_t T(t) S(t); mode 1: S_i = (sum_t T(t)) (sum_t S(t)). */
int or_stv_score(const or_scene *S, const or_camera *cams, int32_t n_cams, const float *ts, int32_t n_ts,
                 double percentile, double *score, double *spatial, double *tv, double *gamma, int mode,
                 int variant)
{
    const int n = S->n;
    if (n <= 0) return 0;
    float *vol = (float *)malloc(sizeof(float) * (size_t)n);
    for (int i = 0; i < n; ++i) vol[i] = or_volume(S, i);
    float *sorted = (float *)malloc(sizeof(float) * (size_t)n);
    memcpy(sorted, vol, sizeof(float) * (size_t)n);
    qsort(sorted, (size_t)n, sizeof(float), or_cmp_float);
    int rank = (int)ceil(percentile * (double)n) - 1;
    if (rank < 0) rank = 0;
    if (rank > n - 1) rank = n - 1;
    const double vp = sorted[rank];
    double *sig = (double *)malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) sig[i] = or_sigma_t(S, i);
    double *ss = (double *)malloc(sizeof(double) * (size_t)n);
    double *tv_sum = (double *)calloc((size_t)n, sizeof(double));
    double *ss_sum = (double *)calloc((size_t)n, sizeof(double));
    for (int i = 0; i < n; ++i) score[i] = 0.0;
    for (int k = 0; k < n_ts; ++k) {
        memset(ss, 0, sizeof(double) * (size_t)n);
        for (int c = 0; c < n_cams; ++c) or_contrib(S, &cams[c], ts[k], ss);
        for (int i = 0; i < n; ++i) {
            const double g = fmin((double)vol[i] / vp, 1.0);
            const double mu = (double)S->mean[4 * (size_t)i + 3];
            const double v = or_tv((double)ts[k], mu, sig[i]);
            double Tt = v * g, St = ss[i];
            if (variant == 1) Tt = 1.0;
            if (variant == 2) St = 1.0;
            if (variant == 3) Tt = or_tv_p1((double)ts[k], mu, sig[i]) * g;
            if (variant == 4) Tt = sig[i] * g;
            score[i] += Tt * St;
            tv_sum[i] += Tt;
            ss_sum[i] += St;
            if (spatial) spatial[(size_t)k * n + i] = ss[i];
            if (tv) tv[(size_t)k * n + i] = v;
        }
    }
    if (mode == 1)
        for (int i = 0; i < n; ++i) score[i] = tv_sum[i] * ss_sum[i];
    free(tv_sum);
    free(ss_sum);
    if (gamma)
        for (int i = 0; i < n; ++i) gamma[i] = fmin((double)vol[i] / vp, 1.0);
    free(ss);
    free(sig);
    free(sorted);
    free(vol);
    return 0;
}

void or_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int or_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
