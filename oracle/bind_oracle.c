/*
 * oracle/bind_oracle.c -- CPU ORACLE of the Gaussian-centric ray-cast binding
 * (§3.3.1).  TEST INFRASTRUCTURE ONLY:
 * only tests/ may load it; it shares no code with the CUDA path.
 *
 * What it computes, by exhaustive search (every ray against every triangle,
 * no acceleration structure -- SPEC's exhaustive_bind):
 *   "we cast rays from these cameras toward the center of a Gaussian.  If a ray
 *   hits a face, we record the face index, the barycentric coordinate of the
 *   intersection point, and the distance from the intersection point to the
 *   Gaussian center.  The Gaussian is then bound to the nearest candidate face"
 *   (P:390-392); bbx8: "each camera casts 8 rays toward the corners of a
 *   Gaussian's BBX.  For each ray, we retain the face closest to the Gaussian"
 *   (P:394-396).
 *
 * Readings (B1-B6):
 *   B1 targets: the centre mu (mode 0) or the 8 corners of the oriented box
 *      mu + R (sx k s0, sy k s1, sz k s2), corner i: s* = +1 iff bit (0,1,2) of i.
 *   B2 rays: from the camera centre c = -R^T t through the target, direction
 *      normalised; cameras with the target at view z <= 0 are skipped.
 *   B3 hit: Moller-Trumbore, |det| < 1e-9 = miss, t > 1e-6, u, v >= 0, u+v <= 1;
 *      the nearest hit along a ray (ties: lower face id).
 *   B4 selection over cameras: minimum squared distance from the hit point to
 *      mu (ties: lower face id, then the earlier camera).
 *   B5 output: face (-1 = no hit from any camera) and barycentrics
 *      (1 - u - v, u, v) of the face's vertices (face[0], face[1], face[2]).
 *   B6 arithmetic: IEEE double, one rounding per written op, in the order
 *      written, no contraction (gcc -ffp-contract=off).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static double b_dot(const double a[3], const double b[3]) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

static void b_cross(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

/* B3: Moller-Trumbore.  Returns 1 on a hit with t, u, v. */
int or_ray_triangle(const double o[3], const double d[3], const double v0[3], const double v1[3], const double v2[3],
                    double *t, double *u, double *v) {
    double e1[3], e2[3], p[3], s[3], q[3];
    for (int a = 0; a < 3; a++) {
        e1[a] = v1[a] - v0[a];
        e2[a] = v2[a] - v0[a];
    }
    b_cross(d, e2, p);
    const double det = b_dot(e1, p);
    if (fabs(det) < 1e-9) return 0;
    const double inv = 1.0 / det;
    for (int a = 0; a < 3; a++) s[a] = o[a] - v0[a];
    const double uu = b_dot(s, p) * inv;
    if (uu < 0.0 || uu > 1.0) return 0;
    b_cross(s, e1, q);
    const double vv = b_dot(d, q) * inv;
    if (vv < 0.0 || uu + vv > 1.0) return 0;
    const double tt = b_dot(e2, q) * inv;
    if (!(tt > 1e-6)) return 0;
    *t = tt;
    *u = uu;
    *v = vv;
    return 1;
}

static void vert(const float *pos, int32_t i, double o[3]) {
    for (int a = 0; a < 3; a++) o[a] = (double)pos[3 * (int64_t)i + a];
}

/* nearest hit of one ray over all faces (B3); returns the face or -1 */
int64_t or_ray_cast(const double o[3], const double d[3], int64_t V, const float *pos, int64_t F,
                    const int32_t *faces, double *t_out, double *u_out, double *v_out) {
    int64_t best = -1;
    double bt = 0.0, bu = 0.0, bv = 0.0;
    for (int64_t f = 0; f < F; f++) {
        const int32_t *fc = faces + 3 * f;
        if (fc[0] < 0 || fc[1] < 0 || fc[2] < 0 || fc[0] >= V || fc[1] >= V || fc[2] >= V) continue;
        double v0[3], v1[3], v2[3], t, u, v;
        vert(pos, fc[0], v0);
        vert(pos, fc[1], v1);
        vert(pos, fc[2], v2);
        if (!or_ray_triangle(o, d, v0, v1, v2, &t, &u, &v)) continue;
        if (best < 0 || t < bt) {  /* faces ascend: an equal t keeps the lower id */
            best = f;
            bt = t; bu = u; bv = v;
        }
    }
    *t_out = bt;
    *u_out = bu;
    *v_out = bv;
    return best;
}

/* B1: target points of Gaussian i (1 or 8), in double */
void or_bind_targets(const float *mean, const float *quat, const float *scale, int mode, float k_sigma,
                     double *out /* [8][3] */) {
    const double mu[3] = {mean[0], mean[1], mean[2]};
    if (mode == 0) {
        for (int a = 0; a < 3; a++) out[a] = mu[a];
        return;
    }
    double w = quat[0], x = quat[1], y = quat[2], z = quat[3];
    const double n = sqrt(((w * w + x * x) + y * y) + z * z);
    w = w / n; x = x / n; y = y / n; z = z / n;
    const double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                         2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                         2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
    const double k = (double)k_sigma;
    for (int i = 0; i < 8; i++) {
        const double l[3] = {((i & 1) ? k : -k) * (double)scale[0], ((i & 2) ? k : -k) * (double)scale[1],
                             ((i & 4) ? k : -k) * (double)scale[2]};
        for (int a = 0; a < 3; a++) out[3 * i + a] = mu[a] + ((R[3 * a] * l[0] + R[3 * a + 1] * l[1]) + R[3 * a + 2] * l[2]);
    }
}

/* The binding table (B1-B5).  cams: [C][12] = R (row-major world->camera) then t. */
int or_bind(int64_t N, const float *means, const float *quats, const float *scales, int64_t V, const float *pos,
            int64_t F, const int32_t *faces, int ncams, const float *cams, int mode, float k_sigma,
            int32_t *face_out, double *bary_out, double *dist2_out, int nthreads) {
    if (ncams < 1 || (mode != 0 && mode != 1)) return 1;
    const int K = mode == 0 ? 1 : 8;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < N; i++) {
        double tg[24];
        or_bind_targets(means + 3 * i, quats + 4 * i, scales + 3 * i, mode, k_sigma, tg);
        const double mu[3] = {means[3 * i], means[3 * i + 1], means[3 * i + 2]};
        for (int k = 0; k < K; k++) {
            const double *P = tg + 3 * k;
            int64_t bf = -1;
            double bd = 0.0, bu = 0.0, bv = 0.0;
            for (int cidx = 0; cidx < ncams; cidx++) {
                const float *Rf = cams + 12 * cidx, *tf = Rf + 9;
                double c[3], vz;
                for (int a = 0; a < 3; a++)
                    c[a] = -(((double)Rf[a] * tf[0] + (double)Rf[3 + a] * tf[1]) + (double)Rf[6 + a] * tf[2]);
                vz = (((double)Rf[6] * P[0] + (double)Rf[7] * P[1]) + (double)Rf[8] * P[2]) + (double)tf[2];
                if (!(vz > 0.0)) continue;  /* B2: target behind this camera */
                double d[3] = {P[0] - c[0], P[1] - c[1], P[2] - c[2]};
                const double len = sqrt(b_dot(d, d));
                if (!(len > 0.0)) continue;
                for (int a = 0; a < 3; a++) d[a] = d[a] / len;
                double t, u, v;
                const int64_t f = or_ray_cast(c, d, V, pos, F, faces, &t, &u, &v);
                if (f < 0) continue;
                double h[3], e[3];
                for (int a = 0; a < 3; a++) {
                    h[a] = c[a] + t * d[a];
                    e[a] = h[a] - mu[a];
                }
                const double d2 = b_dot(e, e);
                if (bf < 0 || d2 < bd || (d2 == bd && f < bf)) {
                    bf = f;
                    bd = d2; bu = u; bv = v;
                }
            }
            face_out[i * K + k] = (int32_t)bf;
            double *b = bary_out + 3 * (i * K + k);
            if (bf >= 0) {
                b[0] = (1.0 - bu) - bv;
                b[1] = bu;
                b[2] = bv;
            } else {
                b[0] = b[1] = b[2] = 0.0;
            }
            if (dist2_out) dist2_out[i * K + k] = bf >= 0 ? bd : -1.0;
        }
    }
    return 0;
}
