/*
 * oracle/unimgs_oracle.c -- CPU ORACLE for the UniMGS single-pass rasterizer.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2601_19233_b200/csrc) and neither side includes the other.
 *
 * What it computes (PAPER.md = P:<line>):
 *   - Gaussian fragments blended by Eq.1-2, alpha = min(0.99,
 *     o*exp(-q/2)) with the EWA-projected conic ("EWA filter").
 *   - Triangle fragments with M = 4 sub-pixel coverage ("we set M=4"),
 *     depth-adjacent triangles grouped into one entity whose
 *     sub-pixel transmittance follows Eq.7, coverage Eq.8
 *     (P:348-351), colour Eq.9, and background Eq.10-11
 *      under the readings R1-R24 listed in DESIGN.md.
 *   - All primitives are ordered per 16x16 tile by (tile, depth bits, id)
 *     ("incorporate triangle fragments into the depth-sorting process").
 *
 * Precision: everything that decides a key, an order or fragment membership
 * follows DESIGN.md "normative fp32 arithmetic" N0-N7 (IEEE binary32, one
 * rounding per written op, fmaf where written).  Colours, alpha and
 * transmittance are evaluated in double.  Build with
 *   gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -lm
 *
 * parity-unpinned parts (no external pin exists): the absolute appearance of
 * realistic scenes; the sort depth of a triangle (R9); per-tile ordering (R8).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_TILE 16
#define OR_MMAX 16

/* blend modes (the paper's ablation Fig.3 / Fig.4) */
enum { OR_EXACT = 0, OR_NAIVE = 1, OR_MSAA_PIXEL = 2, OR_WHOLE_PIXEL = 3, OR_PAPER_LITERAL = 4 };

typedef struct {
    int32_t width, height;
    float fx, fy, cx, cy;
    float R[9], t[3];
    float near_z, far_z;
} or_camera;

typedef struct {
    float alpha_max, t_eps, dilation;
    float bg[3];
    float bg_alpha;
    int32_t blend_mode; /* OR_EXACT .. OR_PAPER_LITERAL */
    int32_t msaa;       /* M in {1, 2, 4, 8, 16} (P:330 uses 4) */
    int32_t tri_depth;  /* triangle sort depth: 0 = centroid (R9), 1 = plane depth at the tile centre (N8, NEXT 3),
                           2 = N8 keys + a per-pixel resort window over the pixel-centre plane depth (N9) */
    int32_t resort_window; /* tri_depth 2: window size W (<= 0: 4) */
} or_settings;

typedef struct {
    uint32_t id;
    int32_t kind;     /* 0 = Gaussian, 1 = triangle */
    uint32_t mask;    /* triangle coverage bits o^j, j = 0..3 */
    float q;          /* Gaussian: N6 Mahalanobis^2 */
    float depth;      /* sort (key) depth: the order of the pixel's tile list */
    float pdepth;     /* depth at the pixel (tri_depth 2): Gaussian view z; triangle N9 */
    double alpha;
    double rgb[3];
} or_frag;

typedef struct {
    /* scene (borrowed pointers) */
    int64_t N, V, F;
    const float *means, *quats, *scales, *opac, *sh;
    const float *cov3d; /* optional [N][6] xx xy xz yy yz zz: replaces quats/scales (N3) */
    int sh_degree;
    const float *pos, *uvs, *cols, *topac;
    const int32_t *faces;
    const uint8_t *tex;
    int tw, th;
    /* view */
    or_camera cam;
    or_settings set;
    int tiles_x, tiles_y;
    /* Gaussian records */
    float *g_rec;      /* [N][8] u v qmax o ca cb cc depth */
    float *g_cov;      /* [N][3] a b c (dilated cov2d) */
    double *g_rgb;     /* [N][3] */
    int32_t *g_rect;   /* [N][4] x0 y0 x1 y1 (inclusive tiles) */
    uint32_t *g_touched;
    /* triangle records */
    int32_t *t_xy;     /* [F][6] X0 Y0 X1 Y1 X2 Y2 after orientation */
    int32_t *t_vid;    /* [F][3] vertex ids after orientation */
    float *t_z;        /* [F][3] view z after orientation */
    float *t_depth;    /* [F] */
    int32_t *t_rect;   /* [F][4] */
    uint32_t *t_touched;
    /* bins */
    int64_t K;
    uint64_t *keys;
    uint32_t *vals;
    uint32_t *ranges;  /* [tiles][2] */
} or_ctx;

/* ------------------------------------------------------------------------- */

or_ctx *or_create(void) { return (or_ctx *)calloc(1, sizeof(or_ctx)); }

static void or_free_view(or_ctx *c) {
    free(c->g_rec); free(c->g_cov); free(c->g_rgb); free(c->g_rect); free(c->g_touched);
    free(c->t_xy); free(c->t_vid); free(c->t_z); free(c->t_depth); free(c->t_rect); free(c->t_touched);
    free(c->keys); free(c->vals); free(c->ranges);
    c->g_rec = c->g_cov = NULL; c->g_rgb = NULL; c->g_rect = NULL; c->g_touched = NULL;
    c->t_xy = c->t_vid = NULL; c->t_z = c->t_depth = NULL; c->t_rect = NULL; c->t_touched = NULL;
    c->keys = NULL; c->vals = NULL; c->ranges = NULL; c->K = 0;
}

void or_destroy(or_ctx *c) {
    if (!c) return;
    or_free_view(c);
    free(c);
}

void or_set_scene(or_ctx *c, int64_t N, const float *means, const float *quats, const float *scales,
                  const float *opac, const float *sh, int sh_degree,
                  int64_t V, int64_t F, const float *pos, const float *uvs, const float *cols,
                  const int32_t *faces, const float *topac, const uint8_t *tex, int tw, int th) {
    c->N = N; c->means = means; c->quats = quats; c->scales = scales; c->opac = opac; c->sh = sh;
    c->sh_degree = sh_degree;
    c->V = V; c->F = F; c->pos = pos; c->uvs = uvs; c->cols = cols; c->faces = faces; c->topac = topac;
    c->tex = tex; c->tw = tw; c->th = th;
}

void or_set_cov3d(or_ctx *c, const float *cov3d) { c->cov3d = cov3d; }

/* ------------------------------------------------------------------------- */
/* N1 view transform: pv[r] = fma(R[r][0],x, fma(R[r][1],y, fma(R[r][2],z, t[r])))          */
static void view_point(const or_camera *cam, const float *p, float pv[3]) {
    for (int r = 0; r < 3; r++)
        pv[r] = fmaf(cam->R[3 * r + 0], p[0], fmaf(cam->R[3 * r + 1], p[1], fmaf(cam->R[3 * r + 2], p[2], cam->t[r])));
}

static float dot3(const float a[3], const float b[3]) { return fmaf(a[0], b[0], fmaf(a[1], b[1], a[2] * b[2])); }

/* Real SH colour in the 3DGS basis, double precision, +0.5, clamp >= 0. */
static void sh_colour(const float *coef, int deg, const double dir[3], double out[3]) {
    const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
    const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                          -1.0925484305920792, 0.5462742152960396};
    const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                          0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                          -0.5900435899266435};
    double x = dir[0], y = dir[1], z = dir[2];
    double basis[16];
    int k = (deg + 1) * (deg + 1);
    basis[0] = C0;
    if (deg > 0) {
        basis[1] = -C1 * y; basis[2] = C1 * z; basis[3] = -C1 * x;
    }
    if (deg > 1) {
        double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
        basis[4] = C2[0] * xy; basis[5] = C2[1] * yz; basis[6] = C2[2] * (2 * zz - xx - yy);
        basis[7] = C2[3] * xz; basis[8] = C2[4] * (xx - yy);
        if (deg > 2) {
            basis[9] = C3[0] * y * (3 * xx - yy);
            basis[10] = C3[1] * xy * z;
            basis[11] = C3[2] * y * (4 * zz - xx - yy);
            basis[12] = C3[3] * z * (2 * zz - 3 * xx - 3 * yy);
            basis[13] = C3[4] * x * (4 * zz - xx - yy);
            basis[14] = C3[5] * z * (xx - yy);
            basis[15] = C3[6] * x * (xx - 3 * yy);
        }
    }
    for (int ch = 0; ch < 3; ch++) {
        double s = 0.0;
        for (int i = 0; i < k; i++) s += basis[i] * (double)coef[3 * i + ch];
        s += 0.5;
        out[ch] = s > 0.0 ? s : 0.0;
    }
}

void or_sh_basis_colour(const float *coef, int deg, const double *dir, double *out) { sh_colour(coef, deg, dir, out); }

/* Gaussian projection, N1-N5 (EWA; 3DGS conventions S:161-169). */
static void project_gaussian(or_ctx *c, int64_t i) {
    const or_camera *cam = &c->cam;
    float *rec = c->g_rec + 8 * i;
    int32_t *rect = c->g_rect + 4 * i;
    c->g_touched[i] = 0;
    rect[0] = rect[1] = rect[2] = rect[3] = -1;
    memset(rec, 0, 8 * sizeof(float));
    memset(c->g_cov + 3 * i, 0, 3 * sizeof(float));
    memset(c->g_rgb + 3 * i, 0, 3 * sizeof(double));

    float pv[3];
    view_point(cam, c->means + 3 * i, pv);
    if (!(pv[2] > cam->near_z) || pv[2] > cam->far_z) return;                 /* N1 */
    float xz = pv[0] / pv[2], yz = pv[1] / pv[2];                               /* N2 */
    float u = fmaf(cam->fx, xz, cam->cx), v = fmaf(cam->fy, yz, cam->cy);

    float Sig[3][3];
    if (c->cov3d) { /* given covariance (e.g. deformed by Eq.13) */
        const float *cv = c->cov3d + 6 * i;
        Sig[0][0] = cv[0]; Sig[0][1] = Sig[1][0] = cv[1]; Sig[0][2] = Sig[2][0] = cv[2];
        Sig[1][1] = cv[3]; Sig[1][2] = Sig[2][1] = cv[4]; Sig[2][2] = cv[5];
    } else {
    /* N3: quaternion (w,x,y,z) -> R, Sigma = R S^2 R^T */
    const float *q = c->quats + 4 * i;
    const float *s = c->scales + 3 * i;
    float w = q[0], x = q[1], y = q[2], z = q[3];
    float n2 = fmaf(w, w, fmaf(x, x, fmaf(y, y, z * z)));
    float k = 1.0f / sqrtf(n2);
    w *= k; x *= k; y *= k; z *= k;
    float qxx = x * x, qyy = y * y, qzz = z * z, qxy = x * y, qxz = x * z, qyz = y * z;
    float qwx = w * x, qwy = w * y, qwz = w * z;
    float r[3][3];
    r[0][0] = 1.0f - 2.0f * (qyy + qzz); r[0][1] = 2.0f * (qxy - qwz); r[0][2] = 2.0f * (qxz + qwy);
    r[1][0] = 2.0f * (qxy + qwz); r[1][1] = 1.0f - 2.0f * (qxx + qzz); r[1][2] = 2.0f * (qyz - qwx);
    r[2][0] = 2.0f * (qxz - qwy); r[2][1] = 2.0f * (qyz + qwx); r[2][2] = 1.0f - 2.0f * (qxx + qyy);
    float m[3][3];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) m[a][b] = r[a][b] * s[b];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) Sig[a][b] = dot3(m[a], m[b]);
    }
    /* A = W Sigma, Sigma_v = A W^T, W = R_w2c */
    float W[3][3], A[3][3], Sv[3][3];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) W[a][b] = cam->R[3 * a + b];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            float col[3] = {Sig[0][b], Sig[1][b], Sig[2][b]};
            A[a][b] = dot3(W[a], col);
        }
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) Sv[a][b] = dot3(A[a], W[b]);

    /* N4: Jacobian at the mean with the 1.3x FoV clamp, cov2d = J Sv J^T + dilation I */
    float lx = 1.3f * (0.5f * (float)cam->width / cam->fx);
    float ly = 1.3f * (0.5f * (float)cam->height / cam->fy);
    float tx = fminf(fmaxf(xz, -lx), lx) * pv[2];
    float ty = fminf(fmaxf(yz, -ly), ly) * pv[2];
    float zz2 = pv[2] * pv[2];
    float J[2][3];
    J[0][0] = cam->fx / pv[2]; J[0][1] = 0.0f; J[0][2] = -(cam->fx * tx) / zz2;
    J[1][0] = 0.0f; J[1][1] = cam->fy / pv[2]; J[1][2] = -(cam->fy * ty) / zz2;
    float B[2][3];
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 3; b++) {
            float col[3] = {Sv[0][b], Sv[1][b], Sv[2][b]};
            B[a][b] = dot3(J[a], col);
        }
    float cov00 = dot3(B[0], J[0]), cov01 = dot3(B[0], J[1]), cov11 = dot3(B[1], J[1]);
    float ca_ = cov00 + c->set.dilation, cb_ = cov01, cc_ = cov11 + c->set.dilation;
    float det = fmaf(ca_, cc_, -(cb_ * cb_));
    if (!(det > 0.0f)) return;
    float inv = 1.0f / det;
    float ka = cc_ * inv, kb = -cb_ * inv, kc = ca_ * inv;
    if (!(ka > 0.0f && fmaf(ka, kc, -(kb * kb)) > 0.0f)) return;

    /* N5: support {alpha >= 1/255} as q <= q_max, padded ellipse bbox, tile rect */
    float o = c->opac[i];
    if (!(255.0 * (double)o >= 1.0)) return;
    float qmax = (float)(2.0 * log(255.0 * (double)o));
    float ex = fmaf(sqrtf(qmax * ca_), 1.0009765625f, 0.00390625f);
    float ey = fmaf(sqrtf(qmax * cc_), 1.0009765625f, 0.00390625f);
    float flx = floorf((u - ex) * 0.0625f), fhx = floorf((u + ex) * 0.0625f);
    float fly = floorf((v - ey) * 0.0625f), fhy = floorf((v + ey) * 0.0625f);
    if (!(fhx >= 0.0f && flx <= (float)(c->tiles_x - 1) && fhy >= 0.0f && fly <= (float)(c->tiles_y - 1)))
        return;
    int x0 = (int)fmaxf(flx, 0.0f), x1 = (int)fminf(fhx, (float)(c->tiles_x - 1));
    int y0 = (int)fmaxf(fly, 0.0f), y1 = (int)fminf(fhy, (float)(c->tiles_y - 1));

    rec[0] = u; rec[1] = v; rec[2] = qmax; rec[3] = o;
    rec[4] = ka; rec[5] = kb; rec[6] = kc; rec[7] = pv[2];
    c->g_cov[3 * i + 0] = ca_; c->g_cov[3 * i + 1] = cb_; c->g_cov[3 * i + 2] = cc_;
    rect[0] = x0; rect[1] = y0; rect[2] = x1; rect[3] = y1;
    c->g_touched[i] = (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));

    /* colour: SH at dir = normalize(mu - campos), campos = -R^T t (double) */
    double cp[3], d[3], nrm = 0.0;
    for (int a = 0; a < 3; a++)
        cp[a] = -((double)cam->R[a] * cam->t[0] + (double)cam->R[3 + a] * cam->t[1] + (double)cam->R[6 + a] * cam->t[2]);
    for (int a = 0; a < 3; a++) { d[a] = (double)c->means[3 * i + a] - cp[a]; nrm += d[a] * d[a]; }
    nrm = sqrt(nrm);
    for (int a = 0; a < 3; a++) d[a] /= nrm;
    int kcoef = (c->sh_degree + 1) * (c->sh_degree + 1);
    sh_colour(c->sh + (int64_t)i * kcoef * 3, c->sh_degree, d, c->g_rgb + 3 * i);
}

static int64_t floor_div(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
    return q;
}

/* Triangle setup, N7. */
static void setup_triangle(or_ctx *c, int64_t f) {
    const or_camera *cam = &c->cam;
    int32_t *xy = c->t_xy + 6 * f, *vid = c->t_vid + 3 * f, *rect = c->t_rect + 4 * f;
    float *tz = c->t_z + 3 * f;
    c->t_touched[f] = 0;
    rect[0] = rect[1] = rect[2] = rect[3] = -1;
    memset(xy, 0, 6 * sizeof(int32_t));
    c->t_depth[f] = 0.0f;
    int32_t X[3], Y[3], id[3];
    float z[3];
    for (int k = 0; k < 3; k++) {
        id[k] = c->faces[3 * f + k];
        if (id[k] < 0 || id[k] >= c->V) return;
        float pv[3];
        view_point(cam, c->pos + 3 * (int64_t)id[k], pv);
        if (!(pv[2] > cam->near_z) || pv[2] > cam->far_z) return;
        float u = fmaf(cam->fx, pv[0] / pv[2], cam->cx), v = fmaf(cam->fy, pv[1] / pv[2], cam->cy);
        if (!(fabsf(u) < 32768.0f && fabsf(v) < 32768.0f)) return;
        X[k] = (int32_t)rintf(u * 256.0f);
        Y[k] = (int32_t)rintf(v * 256.0f);
        z[k] = pv[2];
    }
    float depth = ((z[0] + z[1]) + z[2]) / 3.0f;  /* original face order, before the swap */
    int64_t A2 = (int64_t)(X[1] - X[0]) * (Y[2] - Y[0]) - (int64_t)(X[2] - X[0]) * (Y[1] - Y[0]);
    if (A2 == 0) return;
    if (A2 < 0) {  /* two-sided (R14): swap vertices 1 and 2 with their attributes */
        int32_t t;
        float tf;
        t = X[1]; X[1] = X[2]; X[2] = t;
        t = Y[1]; Y[1] = Y[2]; Y[2] = t;
        t = id[1]; id[1] = id[2]; id[2] = t;
        tf = z[1]; z[1] = z[2]; z[2] = tf;
    }
    int32_t mnx = X[0], mxx = X[0], mny = Y[0], mxy = Y[0];
    for (int k = 1; k < 3; k++) {
        if (X[k] < mnx) mnx = X[k];
        if (X[k] > mxx) mxx = X[k];
        if (Y[k] < mny) mny = Y[k];
        if (Y[k] > mxy) mxy = Y[k];
    }
    int64_t x0 = floor_div(mnx, 4096), x1 = floor_div(mxx, 4096);
    int64_t y0 = floor_div(mny, 4096), y1 = floor_div(mxy, 4096);
    if (x1 < 0 || x0 > c->tiles_x - 1 || y1 < 0 || y0 > c->tiles_y - 1) return;
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (x1 > c->tiles_x - 1) x1 = c->tiles_x - 1;
    if (y1 > c->tiles_y - 1) y1 = c->tiles_y - 1;
    for (int k = 0; k < 3; k++) {
        xy[2 * k] = X[k]; xy[2 * k + 1] = Y[k]; vid[k] = id[k]; tz[k] = z[k];
    }
    c->t_depth[f] = depth;
    rect[0] = (int32_t)x0; rect[1] = (int32_t)y0; rect[2] = (int32_t)x1; rect[3] = (int32_t)y1;
    c->t_touched[f] = (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));
}

int or_project(or_ctx *c, const or_camera *cam, const or_settings *set, int nthreads) {
    or_free_view(c);
    c->cam = *cam;
    c->set = *set;
    c->tiles_x = (cam->width + OR_TILE - 1) / OR_TILE;
    c->tiles_y = (cam->height + OR_TILE - 1) / OR_TILE;
    int64_t N = c->N, F = c->F;
    c->g_rec = (float *)malloc(sizeof(float) * 8 * (N + 1));
    c->g_cov = (float *)malloc(sizeof(float) * 3 * (N + 1));
    c->g_rgb = (double *)malloc(sizeof(double) * 3 * (N + 1));
    c->g_rect = (int32_t *)malloc(sizeof(int32_t) * 4 * (N + 1));
    c->g_touched = (uint32_t *)malloc(sizeof(uint32_t) * (N + 1));
    c->t_xy = (int32_t *)malloc(sizeof(int32_t) * 6 * (F + 1));
    c->t_vid = (int32_t *)malloc(sizeof(int32_t) * 3 * (F + 1));
    c->t_z = (float *)malloc(sizeof(float) * 3 * (F + 1));
    c->t_depth = (float *)malloc(sizeof(float) * (F + 1));
    c->t_rect = (int32_t *)malloc(sizeof(int32_t) * 4 * (F + 1));
    c->t_touched = (uint32_t *)malloc(sizeof(uint32_t) * (F + 1));
    if (!c->g_rec || !c->g_cov || !c->g_rgb || !c->g_rect || !c->g_touched || !c->t_xy || !c->t_vid ||
        !c->t_z || !c->t_depth || !c->t_rect || !c->t_touched)
        return 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) project_gaussian(c, i);
#pragma omp parallel for schedule(static)
    for (int64_t f = 0; f < F; f++) setup_triangle(c, f);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Binning: one key per (tile, primitive) = tile<<32 | bits(depth); sort (key, id). */

/* N8 ("incorporate triangle fragments into the
 * depth-sorting process"): the per-tile sort depth of triangle f in tile (tx, ty) is
 * the view z of its plane at the tile centre, clamped to the triangle's z range.
 * 1/z is affine in screen space, so with the exact integer edge functions E_k of
 * N7 at the tile centre P and A2 = 2 x area:  1/z(P) = sum_k (E_k(P) / A2) / z_k.
 * Evaluated in double, in this order:  w_k = E_k / z_k;  s = (w_0 + w_1) + w_2;
 * z = (float)(A2 / s), clamped to [min z_k, max z_k];  s <= 0 (the plane's
 * horizon lies between P and the triangle) gives max z_k.                     */
float or_tri_tile_depth(const or_ctx *c, int64_t f, int tx, int ty) {
    const int32_t *xy = c->t_xy + 6 * f;
    const float *z = c->t_z + 3 * f;
    const int64_t PX = 4096 * (int64_t)tx + 2048, PY = 4096 * (int64_t)ty + 2048;
    int64_t E[3];
    for (int k = 0; k < 3; k++) {
        const int a = (k + 1) % 3, b = (k + 2) % 3;
        const int64_t Xa = xy[2 * a], Ya = xy[2 * a + 1], Xb = xy[2 * b], Yb = xy[2 * b + 1];
        E[k] = (Xb - Xa) * (PY - Ya) - (Yb - Ya) * (PX - Xa);
    }
    const int64_t A2 = (int64_t)(xy[2] - xy[0]) * (xy[5] - xy[1]) - (int64_t)(xy[4] - xy[0]) * (xy[3] - xy[1]);
    const double s = ((double)E[0] / (double)z[0] + (double)E[1] / (double)z[1]) + (double)E[2] / (double)z[2];
    const float zmin = fminf(fminf(z[0], z[1]), z[2]), zmax = fmaxf(fmaxf(z[0], z[1]), z[2]);
    if (!(s > 0.0)) return zmax;
    return fminf(fmaxf((float)((double)A2 / s), zmin), zmax);
}

/* sort depth of triangle f for the tile holding (tx, ty) (R9 or N8) */
static float tri_key_depth(const or_ctx *c, int64_t f, int tx, int ty) {
    return c->set.tri_depth >= 1 ? or_tri_tile_depth(c, f, tx, ty) : c->t_depth[f];
}

/* N9 (tri_depth 2; "plane-interpolated depth at the pixel centre"):
 * N8's formula at the pixel centre P = (256 x + 128, 256 y + 128) instead of the tile
 * centre -- w_k = E_k(P) / z_k, s = (w_0 + w_1) + w_2 in double, z = (float)(A2 / s)
 * clamped to [min z_k, max z_k], s <= 0 gives max z_k.                              */
float or_tri_point_depth(const or_ctx *c, int64_t f, int64_t PX, int64_t PY) {
    const int32_t *xy = c->t_xy + 6 * f;
    const float *z = c->t_z + 3 * f;
    int64_t E[3];
    for (int k = 0; k < 3; k++) {
        const int a = (k + 1) % 3, b = (k + 2) % 3;
        const int64_t Xa = xy[2 * a], Ya = xy[2 * a + 1], Xb = xy[2 * b], Yb = xy[2 * b + 1];
        E[k] = (Xb - Xa) * (PY - Ya) - (Yb - Ya) * (PX - Xa);
    }
    const int64_t A2 = (int64_t)(xy[2] - xy[0]) * (xy[5] - xy[1]) - (int64_t)(xy[4] - xy[0]) * (xy[3] - xy[1]);
    const double s = ((double)E[0] / (double)z[0] + (double)E[1] / (double)z[1]) + (double)E[2] / (double)z[2];
    const float zmin = fminf(fminf(z[0], z[1]), z[2]), zmax = fmaxf(fmaxf(z[0], z[1]), z[2]);
    if (!(s > 0.0)) return zmax;
    return fminf(fmaxf((float)((double)A2 / s), zmin), zmax);
}

float or_tri_pixel_depth(const or_ctx *c, int64_t f, int x, int y) {
    return or_tri_point_depth(c, f, 256 * (int64_t)x + 128, 256 * (int64_t)y + 128);
}

static float prim_depth(const or_ctx *c, uint32_t id) {
    return (int64_t)id < c->F ? c->t_depth[id] : c->g_rec[8 * ((int64_t)id - c->F) + 7];
}

static uint32_t f32_bits(float f) {
    uint32_t b;
    memcpy(&b, &f, 4);
    return b;
}

typedef struct { uint64_t key; uint32_t val; } or_pair;

static int pair_cmp(const void *a, const void *b) {
    const or_pair *x = (const or_pair *)a, *y = (const or_pair *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    if (x->val != y->val) return x->val < y->val ? -1 : 1;
    return 0;
}

int64_t or_bin(or_ctx *c) {
    int64_t F = c->F, P = c->F + c->N;
    int64_t K = 0;
    for (int64_t p = 0; p < P; p++) K += p < F ? c->t_touched[p] : c->g_touched[p - F];
    or_pair *pairs = (or_pair *)malloc(sizeof(or_pair) * (K + 1));
    if (!pairs) return -1;
    int64_t n = 0;
    for (int64_t p = 0; p < P; p++) {
        const int32_t *rect = p < F ? c->t_rect + 4 * p : c->g_rect + 4 * (p - F);
        uint32_t touched = p < F ? c->t_touched[p] : c->g_touched[p - F];
        if (!touched) continue;
        const uint32_t db = f32_bits(prim_depth(c, (uint32_t)p));
        for (int ty = rect[1]; ty <= rect[3]; ty++)
            for (int tx = rect[0]; tx <= rect[2]; tx++) {
                uint64_t tile = (uint64_t)ty * (uint64_t)c->tiles_x + (uint64_t)tx;
                const uint32_t d = p < F ? f32_bits(tri_key_depth(c, p, tx, ty)) : db;
                pairs[n].key = (tile << 32) | d;
                pairs[n].val = (uint32_t)p;
                n++;
            }
    }
    qsort(pairs, (size_t)n, sizeof(or_pair), pair_cmp);
    int64_t T = (int64_t)c->tiles_x * c->tiles_y;
    free(c->keys); free(c->vals); free(c->ranges);
    c->keys = (uint64_t *)malloc(sizeof(uint64_t) * (n + 1));
    c->vals = (uint32_t *)malloc(sizeof(uint32_t) * (n + 1));
    c->ranges = (uint32_t *)calloc((size_t)(2 * T), sizeof(uint32_t));
    for (int64_t i = 0; i < n; i++) { c->keys[i] = pairs[i].key; c->vals[i] = pairs[i].val; }
    free(pairs);
    for (int64_t i = 0; i < n; i++) {
        uint64_t tile = c->keys[i] >> 32;
        if (i == 0 || (c->keys[i - 1] >> 32) != tile) c->ranges[2 * tile] = (uint32_t)i;
        if (i == n - 1 || (c->keys[i + 1] >> 32) != tile) c->ranges[2 * tile + 1] = (uint32_t)(i + 1);
    }
    c->K = n;
    return n;
}

/* ------------------------------------------------------------------------- */
/* Fragment evaluation at pixel (x, y).                                         */

/* Direct3D standard multisample patterns in 1/16 px from the pixel centre (R10);
 * M = 4 is the paper's setting. */
static const int OR_PAT1[1][2] = {{0, 0}};
static const int OR_PAT2[2][2] = {{4, 4}, {-4, -4}};
static const int OR_PAT4[4][2] = {{-2, -6}, {6, -2}, {-6, 2}, {2, 6}};
static const int OR_PAT8[8][2] = {{1, -3}, {-1, 3}, {5, 1}, {-3, -5}, {-5, 5}, {-7, -1}, {3, 7}, {7, -7}};
static const int OR_PAT16[16][2] = {{1, 1}, {-1, -3}, {-3, 2}, {4, -1}, {-5, -2}, {2, 5}, {5, 3}, {3, -5},
                                    {-2, 6}, {0, -7}, {-4, -6}, {-6, 4}, {-8, 0}, {7, -4}, {6, 7}, {-7, -8}};

static const int (*or_pattern(int M))[2] {
    switch (M) {
        case 1: return OR_PAT1;
        case 2: return OR_PAT2;
        case 8: return OR_PAT8;
        case 16: return OR_PAT16;
        default: return OR_PAT4;
    }
}

static int or_msaa(const or_settings *s) { return (s->msaa == 1 || s->msaa == 2 || s->msaa == 8 || s->msaa == 16) ? s->msaa : 4; }

/* N6: q at the pixel centre; fragment iff q <= q_max (equivalent to alpha >= 1/255) */
static int gaussian_fragment(const or_ctx *c, int64_t g, int x, int y, or_frag *fr) {
    const float *rec = c->g_rec + 8 * g;
    float dx = ((float)x + 0.5f) - rec[0];
    float dy = ((float)y + 0.5f) - rec[1];
    float q = fmaf(rec[4], dx * dx, fmaf(rec[6], dy * dy, (rec[5] + rec[5]) * (dx * dy)));
    if (!(q <= rec[2])) return 0;
    double a = (double)rec[3] * exp(-0.5 * (double)q);
    if (a > (double)c->set.alpha_max) a = (double)c->set.alpha_max;
    fr->id = (uint32_t)(g + c->F);
    fr->kind = 0;
    fr->mask = 0;
    fr->q = q;
    fr->depth = rec[7];
    fr->pdepth = rec[7];
    fr->alpha = a;
    for (int k = 0; k < 3; k++) fr->rgb[k] = c->g_rgb[3 * g + k];
    return 1;
}

static int64_t edge_fn(const int32_t *xy, int k, int64_t PX, int64_t PY) {
    int a = (k + 1) % 3, b = (k + 2) % 3;
    int64_t Xa = xy[2 * a], Ya = xy[2 * a + 1], Xb = xy[2 * b], Yb = xy[2 * b + 1];
    return (Xb - Xa) * (PY - Ya) - (Yb - Ya) * (PX - Xa);
}

static int edge_inclusive(const int32_t *xy, int k) {
    int a = (k + 1) % 3, b = (k + 2) % 3;
    int64_t dx = (int64_t)xy[2 * b] - xy[2 * a], dy = (int64_t)xy[2 * b + 1] - xy[2 * a + 1];
    return dy > 0 || (dy == 0 && dx < 0);
}

/* point (PX, PY) in 1/256 px inside the oriented triangle, top-left-style rule (N7, R11) */
static int or_inside(const int32_t *xy, int64_t PX, int64_t PY) {
    for (int k = 0; k < 3; k++) {
        int64_t e = edge_fn(xy, k, PX, PY);
        if (e < (edge_inclusive(xy, k) ? 0 : 1)) return 0;
    }
    return 1;
}

uint32_t or_coverage_mask_m(const int32_t *xy, int x, int y, int M) {
    const int (*pat)[2] = or_pattern(M);
    uint32_t m = 0;
    for (int j = 0; j < M; j++)
        if (or_inside(xy, 256 * (int64_t)x + 128 + 16 * pat[j][0], 256 * (int64_t)y + 128 + 16 * pat[j][1])) m |= 1u << j;
    return m;
}

uint32_t or_coverage_mask(const int32_t *xy, int x, int y) {
    uint32_t m = 0;
    for (int j = 0; j < 4; j++) {
        int64_t PX = 256 * (int64_t)x + 128 + 16 * OR_PAT4[j][0];
        int64_t PY = 256 * (int64_t)y + 128 + 16 * OR_PAT4[j][1];
        int in = 1;
        for (int k = 0; k < 3; k++) {
            int64_t e = edge_fn(xy, k, PX, PY);
            if (e < (edge_inclusive(xy, k) ? 0 : 1)) { in = 0; break; }
        }
        if (in) m |= 1u << j;
    }
    return m;
}

static double texel(const or_ctx *c, int64_t i, int64_t j, int ch) {
    if (i < 0) i = 0;
    if (i > c->tw - 1) i = c->tw - 1;
    if (j < 0) j = 0;
    if (j > c->th - 1) j = c->th - 1;
    return (double)c->tex[(j * c->tw + i) * 4 + ch] / 255.0;
}

/* Triangle colour at (PX, PY) in 1/256 px: perspective-correct, unclamped barycentrics (R12). */
static void triangle_colour_at(const or_ctx *c, int64_t f, int64_t PX, int64_t PY, double rgb[3]) {
    const int32_t *xy = c->t_xy + 6 * f;
    const int32_t *vid = c->t_vid + 3 * f;
    const float *tz = c->t_z + 3 * f;
    int64_t A2 = (int64_t)(xy[2] - xy[0]) * (xy[5] - xy[1]) - (int64_t)(xy[4] - xy[0]) * (xy[3] - xy[1]);
    double b[3], w[3], sw = 0.0, lam[3];
    for (int k = 0; k < 3; k++) {
        b[k] = (double)edge_fn(xy, k, PX, PY) / (double)A2;
        w[k] = b[k] / (double)tz[k];
        sw += w[k];
    }
    if (sw != 0.0 && isfinite(sw)) {
        for (int k = 0; k < 3; k++) lam[k] = w[k] / sw;
    } else {
        for (int k = 0; k < 3; k++) lam[k] = b[k];
    }
    if (c->tex && c->uvs) {
        double uu = 0.0, vv = 0.0;
        for (int k = 0; k < 3; k++) {
            uu += lam[k] * (double)c->uvs[2 * (int64_t)vid[k]];
            vv += lam[k] * (double)c->uvs[2 * (int64_t)vid[k] + 1];
        }
        /* bilinear, texel centres at (i+0.5)/W, clamp-to-edge, row 0 at v = 0 */
        double tx = uu * c->tw - 0.5, ty = vv * c->th - 0.5;
        double fi = floor(tx), fj = floor(ty);
        double ax = tx - fi, ay = ty - fj;
        int64_t i0 = (int64_t)fi, j0 = (int64_t)fj;
        for (int ch = 0; ch < 3; ch++) {
            double t00 = texel(c, i0, j0, ch), t10 = texel(c, i0 + 1, j0, ch);
            double t01 = texel(c, i0, j0 + 1, ch), t11 = texel(c, i0 + 1, j0 + 1, ch);
            rgb[ch] = (1 - ay) * ((1 - ax) * t00 + ax * t10) + ay * ((1 - ax) * t01 + ax * t11);
        }
    } else if (c->cols) {
        for (int ch = 0; ch < 3; ch++) {
            double s = 0.0;
            for (int k = 0; k < 3; k++) s += lam[k] * (double)c->cols[3 * (int64_t)vid[k] + ch];
            rgb[ch] = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
        }
    } else {
        rgb[0] = rgb[1] = rgb[2] = 1.0;
    }
}

/* at the pixel centre (R12) */
static void triangle_colour(const or_ctx *c, int64_t f, int x, int y, double rgb[3]) {
    triangle_colour_at(c, f, 256 * (int64_t)x + 128, 256 * (int64_t)y + 128, rgb);
}

static int triangle_fragment(const or_ctx *c, int64_t f, int x, int y, or_frag *fr) {
    if (!c->t_touched[f]) return 0;
    uint32_t m = or_coverage_mask_m(c->t_xy + 6 * f, x, y, or_msaa(&c->set));
    if (!m) return 0;
    fr->id = (uint32_t)f;
    fr->kind = 1;
    fr->mask = m;
    fr->q = 0.0f;
    fr->depth = tri_key_depth(c, f, x / OR_TILE, y / OR_TILE);
    fr->pdepth = c->set.tri_depth == 2 ? or_tri_pixel_depth(c, f, x, y) : fr->depth;
    fr->alpha = (double)c->topac[f];
    triangle_colour(c, f, x, y, fr->rgb);
    return 1;
}

/* ------------------------------------------------------------------------- */
/* The unified blend (state machine of DESIGN.md "oracle definition"):
 *   Gaussian: Eq.1-2 (closing an open entity first);
 *   triangle: Eq.7 sub-pixel t^j, Eq.8 O_i, Eq.9 colour with T_in = T at entry;
 *   exit T = T_e * mean_j t^j (R3); out = C + T * bg_alpha * C_bg (R5);
 *   blend-then-test termination T_eff < t_eps (R16).                          */
typedef struct {
    double C[3], T, Te, t[OR_MMAX], Teff;
    double G;   /* OR_WHOLE_PIXEL: Gaussian attenuation since the entity opened */
    double Tl;  /* OR_PAPER_LITERAL: pixel T updated per triangle by Eq.6 (geometric O) */
    int open, done, M, mode;
} or_pix;

static void pix_init(or_pix *s, const or_settings *set) {
    memset(s, 0, sizeof(*s));
    s->T = 1.0;
    s->Teff = 1.0;
    s->M = or_msaa(set);
    s->mode = set->blend_mode;
}

static double mean_t(const or_pix *s) {
    double a = 0.0;
    for (int j = 0; j < s->M; j++) a += s->t[j];
    return a / s->M;
}

static double popc_frac(const or_pix *s, uint32_t m) {
    int n = 0;
    for (int j = 0; j < s->M; j++) n += (m >> j) & 1u;
    return (double)n / s->M;
}

/* The entity's exit transmittance under the active mode. */
static double exit_T(const or_pix *s) {
    if (s->mode == OR_PAPER_LITERAL) return s->Tl;
    if (s->mode == OR_WHOLE_PIXEL) return s->Te * mean_t(s) * s->G;
    return s->Te * mean_t(s); /* R3 */
}

static void pix_apply(or_pix *s, const or_frag *fr, const or_settings *set) {
    const int mode = s->mode;
    if (fr->kind == 0) {
        if (mode == OR_WHOLE_PIXEL && s->open) {
            /* Fig.3b/c: one entity spans the whole list; the Gaussian blends with the current
             * transmittance but does not attenuate the entity's sub-pixel state */
            double Tn = s->Te * mean_t(s) * s->G;
            for (int k = 0; k < 3; k++) s->C[k] += Tn * fr->alpha * fr->rgb[k];
            s->G *= (1.0 - fr->alpha);
            s->Teff = s->Te * mean_t(s) * s->G;
        } else {
            if (s->open) { s->T = exit_T(s); s->open = 0; } /* depth-adjacency broken */
            for (int k = 0; k < 3; k++) s->C[k] += s->T * fr->alpha * fr->rgb[k];
            s->T = s->T * (1.0 - fr->alpha);
            s->Teff = s->T;
        }
    } else if (mode == OR_NAIVE) {
        /* Fig.3a / 4a: a triangle fragment blends like a Gaussian at full coverage */
        for (int k = 0; k < 3; k++) s->C[k] += s->T * fr->alpha * fr->rgb[k];
        s->T = s->T * (1.0 - fr->alpha);
        s->Teff = s->T;
    } else if (mode == OR_MSAA_PIXEL) {
        /* Eq.5-6: geometric coverage, pixel-level transmittance */
        double O = popc_frac(s, fr->mask);
        for (int k = 0; k < 3; k++) s->C[k] += s->T * O * fr->alpha * fr->rgb[k];
        s->T = s->T * (1.0 - O * fr->alpha);
        s->Teff = s->T;
    } else {
        if (!s->open) {
            s->open = 1;
            s->Te = s->T;
            s->G = 1.0;
            s->Tl = s->T;
            for (int j = 0; j < s->M; j++) s->t[j] = 1.0;
        }
        double O = 0.0;
        for (int j = 0; j < s->M; j++)
            if (fr->mask >> j & 1u) O += s->t[j];
        O /= s->M;
        for (int k = 0; k < 3; k++) s->C[k] += s->Te * O * fr->alpha * fr->rgb[k];
        for (int j = 0; j < s->M; j++)
            if (fr->mask >> j & 1u) s->t[j] *= (1.0 - fr->alpha);
        s->Tl *= (1.0 - popc_frac(s, fr->mask) * fr->alpha);
        s->Teff = exit_T(s);
    }
    if (s->Teff < (double)set->t_eps) s->done = 1;
}

static void pix_finish(or_pix *s, const or_settings *set, double out[4]) {
    if (s->open) { s->T = exit_T(s); s->open = 0; }
    for (int k = 0; k < 3; k++) out[k] = s->C[k] + s->T * (double)set->bg_alpha * (double)set->bg[k];
    out[3] = s->T;
}

/* Blend an explicit fragment list (worked examples, pins). trace[i] = T_eff after fragment i. */
int or_blend_fragments(const or_frag *fr, int n, const or_settings *set, double out[4], double *trace) {
    or_pix s;
    pix_init(&s, set);
    int used = 0;
    for (int i = 0; i < n && !s.done; i++) {
        pix_apply(&s, fr + i, set);
        if (trace) trace[i] = s.Teff;
        used++;
    }
    pix_finish(&s, set, out);
    return used;
}

/* tri_depth 2: the per-pixel resort window.  The pixel's fragments arrive in tile-list
 * order (keys of N8); each is pushed into a window of W entries; when the window is
 * full the entry with the smallest (bits(pdepth), id) -- incoming one included -- is
 * blended; at the end of the list the rest are blended in that order.  A bounded
 * priority queue: it sorts the fragments by their depth at the pixel exactly whenever
 * none is displaced by W or more positions from its place (always, if W >= the number
 * of the pixel's fragments).  Blending stops at termination (R16) as usual.          */
#define OR_WMAX 64
typedef struct {
    or_frag w[OR_WMAX];
    int n, cap;
} or_window;

static int frag_pless(const or_frag *a, const or_frag *b) {
    const uint32_t da = f32_bits(a->pdepth), db = f32_bits(b->pdepth);
    return da != db ? da < db : a->id < b->id;
}

static int win_cap(const or_settings *set) {
    const int w = set->resort_window > 0 ? set->resort_window : 4;
    return w > OR_WMAX ? OR_WMAX : w;
}

/* push fr; if the window overflows, write the fragment to blend into *out and return 1 */
static int win_push(or_window *win, const or_frag *fr, or_frag *out) {
    if (win->n < win->cap) {
        win->w[win->n++] = *fr;
        return 0;
    }
    int m = -1;
    for (int i = 0; i < win->n; i++)
        if (m < 0 || frag_pless(&win->w[i], &win->w[m])) m = i;
    if (frag_pless(fr, &win->w[m])) {
        *out = *fr;
    } else {
        *out = win->w[m];
        win->w[m] = *fr;
    }
    return 1;
}

/* pop the smallest remaining entry; 0 when empty */
static int win_pop(or_window *win, or_frag *out) {
    if (!win->n) return 0;
    int m = 0;
    for (int i = 1; i < win->n; i++)
        if (frag_pless(&win->w[i], &win->w[m])) m = i;
    *out = win->w[m];
    win->w[m] = win->w[--win->n];
    return 1;
}

/* Blend one fragment of the pixel's list order, through the window for tri_depth 2. */
static void pix_feed(or_pix *s, or_window *win, const or_frag *fr, const or_settings *set, uint32_t *cnt) {
    or_frag e;
    const or_frag *apply = fr;
    if (set->tri_depth == 2) {
        if (!win_push(win, fr, &e)) return;
        apply = &e;
    }
    pix_apply(s, apply, set);
    if (cnt) {
        cnt[apply->kind == 0 ? 0 : 1]++;
        cnt[2] = apply->id;
    }
}

static void pix_drain(or_pix *s, or_window *win, const or_settings *set, uint32_t *cnt) {
    or_frag e;
    while (set->tri_depth == 2 && !s->done && win_pop(win, &e)) {
        pix_apply(s, &e, set);
        if (cnt) {
            cnt[e.kind == 0 ? 0 : 1]++;
            cnt[2] = e.id;
        }
    }
}

/* Tiled render: per pixel, walk its tile's sorted list (keys, ranges from or_bin). */
static void render_pixel_tiled(const or_ctx *c, int x, int y, double out[4]) {
    int tile = (y / OR_TILE) * c->tiles_x + (x / OR_TILE);
    uint32_t b = c->ranges[2 * tile], e = c->ranges[2 * tile + 1];
    or_pix s;
    pix_init(&s, &c->set);
    or_window win;
    win.n = 0;
    win.cap = win_cap(&c->set);
    or_frag fr;
    for (uint32_t i = b; i < e && !s.done; i++) {
        uint32_t p = c->vals[i];
        int hit = (int64_t)p < c->F ? triangle_fragment(c, p, x, y, &fr)
                                    : gaussian_fragment(c, (int64_t)p - c->F, x, y, &fr);
        if (hit) pix_feed(&s, &win, &fr, &c->set, NULL);
    }
    pix_drain(&s, &win, &c->set, NULL);
    pix_finish(&s, &c->set, out);
}

/* Fragment bookkeeping of the tiled render (C.1 membership, R16 termination):
 * per pixel {Gaussian fragments blended, triangle fragments blended, unified id of
 * the last fragment blended (0xFFFFFFFF: none), 0}, over the listed tiles (all if
 * tiles == NULL) into out[H][W][4].  With t_eps = 0 these are all fragments of
 * the pixel (nothing terminates).                                              */
static void count_pixel_tiled(const or_ctx *c, int x, int y, uint32_t out[4]) {
    int tile = (y / OR_TILE) * c->tiles_x + (x / OR_TILE);
    uint32_t b = c->ranges[2 * tile], e = c->ranges[2 * tile + 1];
    or_pix s;
    pix_init(&s, &c->set);
    or_window win;
    win.n = 0;
    win.cap = win_cap(&c->set);
    or_frag fr;
    out[0] = out[1] = out[3] = 0;
    out[2] = 0xFFFFFFFFu;
    for (uint32_t i = b; i < e && !s.done; i++) {
        uint32_t p = c->vals[i];
        int hit = (int64_t)p < c->F ? triangle_fragment(c, p, x, y, &fr)
                                    : gaussian_fragment(c, (int64_t)p - c->F, x, y, &fr);
        if (hit) pix_feed(&s, &win, &fr, &c->set, out);
    }
    pix_drain(&s, &win, &c->set, out);
}

int or_render_counts(const or_ctx *c, uint32_t *out, const int32_t *tiles, int64_t n_tiles, int nthreads) {
    if (!c->ranges) return 1;
    int64_t T = (int64_t)c->tiles_x * c->tiles_y;
    if (!tiles) n_tiles = T;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t ti = 0; ti < n_tiles; ti++) {
        int64_t tile = tiles ? tiles[ti] : ti;
        if (tile < 0 || tile >= T) continue;
        int tx = (int)(tile % c->tiles_x), ty = (int)(tile / c->tiles_x);
        for (int y = ty * OR_TILE; y < (ty + 1) * OR_TILE && y < c->cam.height; y++)
            for (int x = tx * OR_TILE; x < (tx + 1) * OR_TILE && x < c->cam.width; x++)
                count_pixel_tiled(c, x, y, out + 4 * ((int64_t)y * c->cam.width + x));
    }
    return 0;
}

/* Render the listed tiles (all tiles if tiles == NULL) into out[H][W][4]. */
int or_render(or_ctx *c, double *out, const int32_t *tiles, int64_t n_tiles, int nthreads) {
    if (!c->ranges) return 1;
    int64_t T = (int64_t)c->tiles_x * c->tiles_y;
    if (!tiles) n_tiles = T;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t ti = 0; ti < n_tiles; ti++) {
        int64_t tile = tiles ? tiles[ti] : ti;
        if (tile < 0 || tile >= T) continue;
        int tx = (int)(tile % c->tiles_x), ty = (int)(tile / c->tiles_x);
        for (int y = ty * OR_TILE; y < (ty + 1) * OR_TILE && y < c->cam.height; y++)
            for (int x = tx * OR_TILE; x < (tx + 1) * OR_TILE && x < c->cam.width; x++)
                render_pixel_tiled(c, x, y, out + 4 * ((int64_t)y * c->cam.width + x));
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Brute force: per pixel test every primitive (membership of DESIGN.md C.1),
 * then order by (depth bits, id).  No keys, no ranges.                         */

static int frag_cmp(const void *a, const void *b) {
    const or_frag *x = (const or_frag *)a, *y = (const or_frag *)b;
    uint32_t dx = f32_bits(x->depth), dy = f32_bits(y->depth);
    if (dx != dy) return dx < dy ? -1 : 1;
    if (x->id != y->id) return x->id < y->id ? -1 : 1;
    return 0;
}

/* All fragments of pixel (x, y) in blend order; returns the count (<= cap written). */
int64_t or_pixel_fragments(const or_ctx *c, int x, int y, or_frag *outf, int64_t cap) {
    int tx = x / OR_TILE, ty = y / OR_TILE;
    int64_t n = 0;
    or_frag fr;
    for (int64_t f = 0; f < c->F; f++)
        if (triangle_fragment(c, f, x, y, &fr)) {
            if (n < cap) outf[n] = fr;
            n++;
        }
    for (int64_t g = 0; g < c->N; g++) {
        if (!c->g_touched[g]) continue;
        const int32_t *r = c->g_rect + 4 * g;
        if (tx < r[0] || tx > r[2] || ty < r[1] || ty > r[3]) continue;
        if (gaussian_fragment(c, g, x, y, &fr)) {
            if (n < cap) outf[n] = fr;
            n++;
        }
    }
    if (n <= cap) qsort(outf, (size_t)n, sizeof(or_frag), frag_cmp);
    return n;
}

/* Pairs (pixel, Gaussian) with q <= q_max whose tile is outside the Gaussian's rect. */
int64_t or_support_truncation(const or_ctx *c) {
    int64_t cnt = 0;
    for (int64_t g = 0; g < c->N; g++) {
        if (!c->g_touched[g]) continue;
        const int32_t *r = c->g_rect + 4 * g;
        for (int y = 0; y < c->cam.height; y++)
            for (int x = 0; x < c->cam.width; x++) {
                int tx = x / OR_TILE, ty = y / OR_TILE;
                if (tx >= r[0] && tx <= r[2] && ty >= r[1] && ty <= r[3]) continue;
                or_frag fr;
                if (gaussian_fragment(c, g, x, y, &fr)) cnt++;
            }
    }
    return cnt;
}

int or_render_bruteforce(or_ctx *c, double *out, int nthreads) {
    if (!c->g_rec) return 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int64_t cap = c->N + c->F + 1;
    int H = c->cam.height, W = c->cam.width;
#pragma omp parallel
    {
        or_frag *buf = (or_frag *)malloc(sizeof(or_frag) * cap);
#pragma omp for schedule(dynamic, 4)
        for (int y = 0; y < H; y++)
            for (int x = 0; x < W; x++) {
                int64_t n = or_pixel_fragments(c, x, y, buf, cap);
                double *o = out + 4 * ((int64_t)y * W + x);
                or_pix s;
                pix_init(&s, &c->set);
                or_window win;
                win.n = 0;
                win.cap = win_cap(&c->set);
                for (int64_t i = 0; i < n && !s.done; i++) pix_feed(&s, &win, buf + i, &c->set, NULL);
                pix_drain(&s, &win, &c->set, NULL);
                pix_finish(&s, &c->set, o);
            }
        free(buf);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Supersampled ground truth (used for the Fig.4 overflow / AA
 * checks, not for parity): each pixel = mean over S x S sub-samples of exact
 * ordered alpha blending at the sub-sample -- Gaussian alpha evaluated there,
 * triangle coverage point-wise (same integer edge test) and colour shaded
 * there; every fragment is a full-coverage alpha blend (Eq.1-2).  Brute force
 * over all projected primitives, order (depth bits, id).                       */
int or_render_supersampled(or_ctx *c, double *out, int S, int nthreads) {
    if (!c->g_rec || S < 1 || 256 % S) return 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    const int64_t P = c->F + c->N;
    const int H = c->cam.height, W = c->cam.width;
#pragma omp parallel
    {
        or_frag *buf = (or_frag *)malloc(sizeof(or_frag) * (P + 1));
#pragma omp for schedule(dynamic, 1)
        for (int y = 0; y < H; y++)
            for (int x = 0; x < W; x++) {
                double acc[4] = {0, 0, 0, 0};
                for (int sj = 0; sj < S; sj++)
                    for (int si = 0; si < S; si++) {
                        const int64_t PX = 256 * (int64_t)x + (2 * si + 1) * (128 / S);
                        const int64_t PY = 256 * (int64_t)y + (2 * sj + 1) * (128 / S);
                        const double px = PX / 256.0, py = PY / 256.0;
                        int64_t n = 0;
                        for (int64_t f = 0; f < c->F; f++) {
                            if (!c->t_touched[f] || !or_inside(c->t_xy + 6 * f, PX, PY)) continue;
                            buf[n].id = (uint32_t)f; buf[n].kind = 1; buf[n].mask = 1;
                            /* tri_depth 2: the truth orders by the plane depth at the sub-sample */
                            buf[n].depth = c->set.tri_depth == 2 ? or_tri_point_depth(c, f, PX, PY)
                                                                 : tri_key_depth(c, f, x / OR_TILE, y / OR_TILE);
                            buf[n].alpha = (double)c->topac[f];
                            triangle_colour_at(c, f, PX, PY, buf[n].rgb);
                            n++;
                        }
                        for (int64_t g = 0; g < c->N; g++) {
                            if (!c->g_touched[g]) continue;
                            const float *rec = c->g_rec + 8 * g;
                            const double dx = px - rec[0], dy = py - rec[1];
                            const double q = rec[4] * dx * dx + 2.0 * rec[5] * dx * dy + rec[6] * dy * dy;
                            if (!(q <= rec[2])) continue;
                            double a = (double)rec[3] * exp(-0.5 * q);
                            if (a > (double)c->set.alpha_max) a = (double)c->set.alpha_max;
                            buf[n].id = (uint32_t)(g + c->F); buf[n].kind = 0; buf[n].mask = 0; buf[n].depth = rec[7];
                            buf[n].alpha = a;
                            for (int k = 0; k < 3; k++) buf[n].rgb[k] = c->g_rgb[3 * g + k];
                            n++;
                        }
                        qsort(buf, (size_t)n, sizeof(or_frag), frag_cmp);
                        double T = 1.0, C[3] = {0, 0, 0};
                        for (int64_t i = 0; i < n; i++) {
                            for (int k = 0; k < 3; k++) C[k] += T * buf[i].alpha * buf[i].rgb[k];
                            T *= 1.0 - buf[i].alpha;
                        }
                        for (int k = 0; k < 3; k++) acc[k] += C[k] + T * (double)c->set.bg_alpha * (double)c->set.bg[k];
                        acc[3] += T;
                    }
                double *o = out + 4 * ((int64_t)y * W + x);
                for (int k = 0; k < 4; k++) o[k] = acc[k] / ((double)S * S);
            }
        free(buf);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Deformation transfer, Eq.12-13, double precision.
 * Per Gaussian and bound anchor i (K = 1 centre ray or 8 BBX corners)
 * on face (v1, v2, v3) with barycentrics (u, v, w):
 *   Delta_i = u Delta^1 + v Delta^2 + w Delta^3,  R_i = u log R^1 + v log R^2 + w log R^3,
 *   S_i = u S^1 + v S^2 + w S^3                                            (Eq.12)
 *   R' = exp(mean_i R_i), S' = mean_i S_i, Sigma' = R'S' Sigma (R'S')^T,
 *   mu' = mu + mean_i Delta_i                                             (Eq.13)
 * log R is an axis-angle vector (so(3)); exp by Rodrigues' formula.  Anchors with
 * face < 0 are unbound and skipped (the means are over the bound anchors; a
 * Gaussian with none keeps mu and Sigma).  Sigma comes from quats/scales
 * (Sigma = R S^2 R^T) or from cov3d when the scene has one.                 */
static void or_rodrigues(const double w[3], double R[3][3]) {
    const double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    double K[3][3] = {{0, -w[2], w[1]}, {w[2], 0, -w[0]}, {-w[1], w[0], 0}};
    double a, b; /* R = I + a K + b K^2 with a = sin th / th, b = (1 - cos th) / th^2 */
    if (th < 1e-6) { a = 1.0 - th * th / 6.0; b = 0.5 - th * th / 24.0; }
    else { a = sin(th) / th; b = (1.0 - cos(th)) / (th * th); }
    for (int r = 0; r < 3; r++)
        for (int c2 = 0; c2 < 3; c2++) {
            double k2 = 0.0;
            for (int m = 0; m < 3; m++) k2 += K[r][m] * K[m][c2];
            R[r][c2] = (r == c2 ? 1.0 : 0.0) + a * K[r][c2] + b * k2;
        }
}

void or_rodrigues_public(const double *w, double *R) { or_rodrigues(w, (double(*)[3])R); }

int or_deform(const or_ctx *c, int K, const int32_t *face, const float *bary, const int32_t *faces, int64_t F,
              int64_t V, const float *delta, const float *log_rot, const float *shear, double *mu_out,
              double *cov_out) {
    if (K < 1 || K > 8) return 1;
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < c->N; g++) {
        double Sig[3][3];
        if (c->cov3d) {
            const float *cv = c->cov3d + 6 * g;
            Sig[0][0] = cv[0]; Sig[0][1] = Sig[1][0] = cv[1]; Sig[0][2] = Sig[2][0] = cv[2];
            Sig[1][1] = cv[3]; Sig[1][2] = Sig[2][1] = cv[4]; Sig[2][2] = cv[5];
        } else {
            const float *q = c->quats + 4 * g, *sc = c->scales + 3 * g;
            double w = q[0], x = q[1], y = q[2], z = q[3];
            const double n = sqrt(w * w + x * x + y * y + z * z);
            w /= n; x /= n; y /= n; z /= n;
            const double Rg[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                                     {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                                     {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
            for (int a = 0; a < 3; a++)
                for (int b = 0; b < 3; b++) {
                    double acc = 0.0;
                    for (int m = 0; m < 3; m++) acc += Rg[a][m] * (double)sc[m] * (double)sc[m] * Rg[b][m];
                    Sig[a][b] = acc;
                }
        }
        double sd[3] = {0, 0, 0}, sl[3] = {0, 0, 0}, ss[6] = {0, 0, 0, 0, 0, 0};
        int n = 0;
        for (int i = 0; i < K; i++) {
            const int32_t f = face[g * K + i];
            if (f < 0 || f >= F) continue;
            /* a face with a vertex id outside [0, V) is invalid input, culled as a value like an
             * unbound anchor (SPEC S:165 error-as-value; include/unimgs.h unimgs_deform) */
            if (faces[3 * (int64_t)f] < 0 || faces[3 * (int64_t)f] >= V || faces[3 * (int64_t)f + 1] < 0 ||
                faces[3 * (int64_t)f + 1] >= V || faces[3 * (int64_t)f + 2] < 0 || faces[3 * (int64_t)f + 2] >= V)
                continue;
            const float *bw = bary + 3 * (g * K + i);
            for (int j = 0; j < 3; j++) {
                const int64_t v = faces[3 * (int64_t)f + j];
                const double wj = bw[j];
                for (int a = 0; a < 3; a++) {
                    sd[a] += wj * delta[3 * v + a];
                    sl[a] += wj * log_rot[3 * v + a];
                }
                for (int a = 0; a < 6; a++) ss[a] += wj * shear[6 * v + a];
            }
            n++;
        }
        double *mo = mu_out + 3 * g, *co = cov_out + 6 * g;
        if (n == 0) {
            for (int a = 0; a < 3; a++) mo[a] = c->means[3 * g + a];
            co[0] = Sig[0][0]; co[1] = Sig[0][1]; co[2] = Sig[0][2]; co[3] = Sig[1][1]; co[4] = Sig[1][2]; co[5] = Sig[2][2];
            continue;
        }
        double Rm[3][3], L[3] = {sl[0] / n, sl[1] / n, sl[2] / n};
        or_rodrigues(L, Rm);
        const double S[3][3] = {{ss[0] / n, ss[1] / n, ss[2] / n}, {ss[1] / n, ss[3] / n, ss[4] / n},
                                {ss[2] / n, ss[4] / n, ss[5] / n}};
        double A[3][3], AS[3][3], Sp[3][3];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) {
                double acc = 0.0;
                for (int m = 0; m < 3; m++) acc += Rm[a][m] * S[m][b];
                A[a][b] = acc;
            }
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) {
                double acc = 0.0;
                for (int m = 0; m < 3; m++) acc += A[a][m] * Sig[m][b];
                AS[a][b] = acc;
            }
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) {
                double acc = 0.0;
                for (int m = 0; m < 3; m++) acc += AS[a][m] * A[b][m];
                Sp[a][b] = acc;
            }
        for (int a = 0; a < 3; a++) mo[a] = (double)c->means[3 * g + a] + sd[a] / n;
        co[0] = Sp[0][0]; co[1] = Sp[0][1]; co[2] = Sp[0][2]; co[3] = Sp[1][1]; co[4] = Sp[1][2]; co[5] = Sp[2][2];
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* accessors                                                                    */
int64_t or_num_pairs(const or_ctx *c) { return c->K; }
int or_tiles_x(const or_ctx *c) { return c->tiles_x; }
int or_tiles_y(const or_ctx *c) { return c->tiles_y; }

void or_get_gaussian_records(const or_ctx *c, float *rec8, float *cov3, double *rgb, int32_t *rect, uint32_t *touched) {
    if (rec8) memcpy(rec8, c->g_rec, sizeof(float) * 8 * c->N);
    if (cov3) memcpy(cov3, c->g_cov, sizeof(float) * 3 * c->N);
    if (rgb) memcpy(rgb, c->g_rgb, sizeof(double) * 3 * c->N);
    if (rect) memcpy(rect, c->g_rect, sizeof(int32_t) * 4 * c->N);
    if (touched) memcpy(touched, c->g_touched, sizeof(uint32_t) * c->N);
}

void or_get_triangle_records(const or_ctx *c, int32_t *xy6, int32_t *vid3, float *z3, float *depth, int32_t *rect,
                             uint32_t *touched) {
    if (xy6) memcpy(xy6, c->t_xy, sizeof(int32_t) * 6 * c->F);
    if (vid3) memcpy(vid3, c->t_vid, sizeof(int32_t) * 3 * c->F);
    if (z3) memcpy(z3, c->t_z, sizeof(float) * 3 * c->F);
    if (depth) memcpy(depth, c->t_depth, sizeof(float) * c->F);
    if (rect) memcpy(rect, c->t_rect, sizeof(int32_t) * 4 * c->F);
    if (touched) memcpy(touched, c->t_touched, sizeof(uint32_t) * c->F);
}

void or_get_bins(const or_ctx *c, uint64_t *keys, uint32_t *vals, uint32_t *ranges) {
    if (keys) memcpy(keys, c->keys, sizeof(uint64_t) * c->K);
    if (vals) memcpy(vals, c->vals, sizeof(uint32_t) * c->K);
    if (ranges) memcpy(ranges, c->ranges, sizeof(uint32_t) * 2 * (int64_t)c->tiles_x * c->tiles_y);
}
