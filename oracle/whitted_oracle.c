/*
 * whitted_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU reference for the stereo Whitted ray
 * tracer that arXiv 1702.01530 runs on the GPU.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 * The product path (paper_1702_01530_b200/) never links, imports or calls it,
 * and it shares no code, header, table or constant generator with the CUDA path.
 *
 * Arithmetic: IEEE double, no BVH (every ray tests every primitive, in global-ID
 * order), recursion exactly as the definition reads.  Compile with
 *     gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp
 * OpenMP parallelises over independent pixels only.
 *
 * Citations: P:NN = /root/reference/PAPER.md line NN, S:NN = SPEC.md line NN,
 * R#n = DESIGN.md "Readings" item n (the readings of SURVEY.md §8(c)).
 *
 * Pinned by tests/test_oracle_*.py against closed forms, SPEC worked examples
 * (tests/golden/spec_examples.json), invariants and brute force; see DESIGN.md §3.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_VERSION 1

/* S:156 (tracer-core/TraceSettings defaults): t_min = 1e-4, shadow_bias = 1e-4; R#8 */
static const double T_MIN = 1e-4;
static const double BIAS = 1e-4;

/* ------------------------------------------------------------------ vectors */
typedef struct { double x, y, z; } v3;
static v3 mk(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 ld3(const double* p) { return mk(p[0], p[1], p[2]); }
static v3 add(v3 a, v3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 sub(v3 a, v3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 scl(v3 a, double s) { return mk(a.x * s, a.y * s, a.z * s); }
static v3 mul(v3 a, v3 b) { return mk(a.x * b.x, a.y * b.y, a.z * b.z); }
static double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 cross(v3 a, v3 b) { return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x); }
static double len(v3 a) { return sqrt(dot(a, a)); }
static v3 nrm(v3 a) { return scl(a, 1.0 / len(a)); }

/* ------------------------------------------------------------------ scene */
/* Global primitive ID (R#9): spheres [0,S), planes [S,S+P), triangles [S+P,S+P+T). */
typedef struct {
    int32_t n_spheres;  const double* spheres;  const int32_t* sphere_mat;  /* (cx,cy,cz,r)       */
    int32_t n_planes;   const double* planes;   const int32_t* plane_mat;   /* (nx,ny,nz,k): n.x=k */
    int32_t n_vertices; const double* vertices;                             /* (x,y,z)            */
    int32_t n_tris;     const int32_t* tris;    const int32_t* tri_mat;     /* CCW = outward      */
    int32_t n_mats;     const double* mats;     /* kd[3] ks[3] shininess kr kt ior             */
    int32_t n_lights;   const double* lights;   /* pos[3] intensity[3]                          */
    double ambient[3];
    double background[3];
} oracle_scene;

/* Stereo rig after derivation (S:422-430 derive_eyes). */
typedef struct {
    double eye[2][3];   /* 0 = left, 1 = right */
    double f[3], r[3], u[3];
    double th, aspect;
    double sigma[2];
    int32_t width, height;
} oracle_cam;

/* Fragility thresholds (north star exclusion set; R#22). */
typedef struct {
    double eps_t;      /* relative t band for competing hits, grazing, gates   (1e-4) */
    double eps_sphere; /* angular band around sphere silhouettes               (1e-4) */
    double eps_edge;   /* angular band around triangle edges                   (1e-6) */
    double eps_abs;    /* absolute band (x (1+|o|)) around t_min               (1e-5) */
    double perturb;    /* F7: primary-ray perturbation angle (rad), 0 = off    (1e-6; also /10, /33) */
    double perturb_tol;/* F7: radiance change that marks the pixel unstable    (1e-3) */
} oracle_eps;

enum {
    FRAG_COMPETE = 1,    /* F1: another primitive hit within eps_t*t of the nearest hit      */
    FRAG_BOUNDARY = 2,   /* F2/F3: a primitive boundary passes within band of the ray       */
    FRAG_GRAZE = 4,      /* F4: |n.d| <= eps_t at the hit                                   */
    FRAG_RANGE = 8,      /* F5: a candidate t near t_min or near the shadow segment end     */
    FRAG_SHADE = 16,     /* F6: n.l gate or TIR decision within eps_t                        */
    FRAG_SHADOW = 32,    /* a shadow ray whose visibility is not robustly decided           */
    FRAG_UNSTABLE = 64   /* F7: radiance moves > perturb_tol when the primary ray turns by   */
                         /*     perturb rad (error amplified along the ray tree)            */
};

typedef struct {
    long long primary, reflection, refraction, shadow;
} ray_counts;

/* --------------------------------------------------------- camera */
int oracle_setup_rig(const double eye[3], const double look_at[3], const double up[3],
                     double vfov_deg, double interocular, double convergence,
                     int32_t width, int32_t height, oracle_cam* out)
{
    v3 e = ld3(eye), la = ld3(look_at), up3 = ld3(up);
    if (width <= 0 || height <= 0) return 1;
    if (!(vfov_deg > 0.0 && vfov_deg < 180.0)) return 1;
    v3 fl = sub(la, e);
    if (len(fl) == 0.0) return 1;                           /* S:62 position != look_at */
    /* right_axis = normalize(forward x up); u = r x f */
    v3 f = nrm(fl);
    v3 rr = cross(f, up3);
    if (len(rr) == 0.0) return 1;                           /* S:62 up not parallel */
    v3 r = nrm(rr);
    v3 u = cross(r, f);
    double s = interocular;
    /* left = base - (sep/2) r, right = base + (sep/2) r */
    v3 eL = sub(e, scl(r, 0.5 * s)), eR = add(e, scl(r, 0.5 * s));
    out->eye[0][0] = eL.x; out->eye[0][1] = eL.y; out->eye[0][2] = eL.z;
    out->eye[1][0] = eR.x; out->eye[1][1] = eR.y; out->eye[1][2] = eR.z;
    out->f[0] = f.x; out->f[1] = f.y; out->f[2] = f.z;
    out->r[0] = r.x; out->r[1] = r.y; out->r[2] = r.z;
    out->u[0] = u.x; out->u[1] = u.y; out->u[2] = u.z;
    out->th = tan(0.5 * vfov_deg * M_PI / 180.0);           /* vertical fov */
    out->aspect = (double)width / (double)height;
    /* R#13: off-axis window shift, zero parallax at distance C; C<=0 or inf -> parallel rig */
    if (convergence > 0.0 && isfinite(convergence)) {
        out->sigma[0] = +s / (2.0 * convergence);
        out->sigma[1] = -s / (2.0 * convergence);
    } else {
        out->sigma[0] = out->sigma[1] = 0.0;
    }
    out->width = width; out->height = height;
    return 0;
}

/* ray through the centre (px+0.5, py+0.5) of pixel (px,py), (0,0) top-left,
 * image plane at unit distance, direction normalised. */
void oracle_primary_ray(const oracle_cam* c, int32_t eye, int32_t px, int32_t py,
                        double o[3], double d[3])
{
    double sx = (2.0 * (px + 0.5) / c->width - 1.0) * c->th * c->aspect;
    double sy = (1.0 - 2.0 * (py + 0.5) / c->height) * c->th;
    v3 f = ld3(c->f), r = ld3(c->r), u = ld3(c->u);
    v3 dir = nrm(add(add(f, scl(r, sx + c->sigma[eye])), scl(u, sy)));
    o[0] = c->eye[eye][0]; o[1] = c->eye[eye][1]; o[2] = c->eye[eye][2];
    d[0] = dir.x; d[1] = dir.y; d[2] = dir.z;
}

/* ------------------------------------------------ primitive intersection */
/* Sphere: |o + t d - c|^2 = r^2 with |d| = 1; textbook roots (R#21), ascending. */
static int sphere_roots(v3 o, v3 d, const double* s, double* t0, double* t1)
{
    v3 oc = sub(o, ld3(s));
    double b = dot(oc, d);
    double c0 = dot(oc, oc) - s[3] * s[3];
    double disc = b * b - c0;
    if (disc < 0.0) return 0;
    double q = sqrt(disc);
    *t0 = -b - q;
    *t1 = -b + q;
    return 1;
}

/* Plane n.x = k: t = (k - n.o)/(n.d); n.d == 0 -> no intersection. */
static int plane_t(v3 o, v3 d, const double* p, double* t)
{
    v3 n = ld3(p);
    double den = dot(n, d);
    if (den == 0.0) return 0;
    *t = (p[3] - dot(n, o)) / den;
    return 1;
}

/* Triangle: Moller-Trumbore barycentric solve; det == 0 -> no solution. */
static int tri_solve(v3 o, v3 d, v3 v0, v3 v1, v3 v2, double* t, double* bu, double* bv)
{
    v3 e1 = sub(v1, v0), e2 = sub(v2, v0);
    v3 p = cross(d, e2);
    double det = dot(e1, p);
    if (det == 0.0) return 0;
    double inv = 1.0 / det;
    v3 s = sub(o, v0);
    *bu = dot(s, p) * inv;
    v3 q = cross(s, e1);
    *bv = dot(d, q) * inv;
    *t = dot(e2, q) * inv;
    return 1;
}

static void tri_verts(const oracle_scene* sc, int i, v3* v0, v3* v1, v3* v2)
{
    const int32_t* t = sc->tris + 3 * i;
    *v0 = ld3(sc->vertices + 3 * t[0]);
    *v1 = ld3(sc->vertices + 3 * t[1]);
    *v2 = ld3(sc->vertices + 3 * t[2]);
}

static int n_prims(const oracle_scene* sc) { return sc->n_spheres + sc->n_planes + sc->n_tris; }

/* Smallest t > tmin at which primitive `id` meets the ray, or 0 if none.
 * Triangles: inclusive edges u>=0, v>=0, u+v<=1. */
static int prim_hit(const oracle_scene* sc, int id, v3 o, v3 d, double tmin, double* t_out)
{
    if (id < sc->n_spheres) {
        double t0, t1;
        if (!sphere_roots(o, d, sc->spheres + 4 * id, &t0, &t1)) return 0;
        if (t0 > tmin) { *t_out = t0; return 1; }
        if (t1 > tmin) { *t_out = t1; return 1; }
        return 0;
    }
    id -= sc->n_spheres;
    if (id < sc->n_planes) {
        double t;
        if (!plane_t(o, d, sc->planes + 4 * id, &t)) return 0;
        if (t > tmin) { *t_out = t; return 1; }
        return 0;
    }
    id -= sc->n_planes;
    {
        v3 v0, v1, v2;
        double t, bu, bv;
        tri_verts(sc, id, &v0, &v1, &v2);
        if (!tri_solve(o, d, v0, v1, v2, &t, &bu, &bv)) return 0;
        if (bu < 0.0 || bv < 0.0 || bu + bv > 1.0) return 0;
        if (t > tmin) { *t_out = t; return 1; }
        return 0;
    }
}

/* S:180-188 intersect_scene: nearest t > t_min over every primitive; ties go to the
 * smallest global ID (loop runs in ID order and only a strictly smaller t replaces). */
int oracle_nearest(const oracle_scene* sc, const double o3[3], const double d3[3],
                   double* t_out, int32_t* id_out)
{
    v3 o = ld3(o3), d = ld3(d3);
    double best = INFINITY;
    int best_id = -1;
    int n = n_prims(sc);
    for (int i = 0; i < n; ++i) {
        double t;
        if (prim_hit(sc, i, o, d, T_MIN, &t) && t < best) { best = t; best_id = i; }
    }
    *t_out = best;
    *id_out = best_id;
    return best_id >= 0;
}

/* R#4: binary visibility -- occluded iff any primitive has t_min < t < dist. */
static int occluded(const oracle_scene* sc, v3 o, v3 d, double dist)
{
    int n = n_prims(sc);
    for (int i = 0; i < n; ++i) {
        double t;
        if (prim_hit(sc, i, o, d, T_MIN, &t) && t < dist) return 1;
    }
    return 0;
}

/* Geometric unit normal at p of primitive id (sphere outward, plane as given,
 * triangle normalize(e1 x e2) -- CCW outward). */
static v3 geo_normal(const oracle_scene* sc, int id, v3 p)
{
    if (id < sc->n_spheres) {
        const double* s = sc->spheres + 4 * id;
        return scl(sub(p, ld3(s)), 1.0 / s[3]);
    }
    id -= sc->n_spheres;
    if (id < sc->n_planes) return nrm(ld3(sc->planes + 4 * id));
    id -= sc->n_planes;
    v3 v0, v1, v2;
    tri_verts(sc, id, &v0, &v1, &v2);
    return nrm(cross(sub(v1, v0), sub(v2, v0)));
}

static int prim_material(const oracle_scene* sc, int id)
{
    if (id < sc->n_spheres) return sc->sphere_mat[id];
    id -= sc->n_spheres;
    if (id < sc->n_planes) return sc->plane_mat[id];
    return sc->tri_mat[id - sc->n_planes];
}

/* ------------------------------------------------------------ fragility */
/* Distance from point q to segment [a,b]. */
static double seg_dist(v3 q, v3 a, v3 b)
{
    v3 ab = sub(b, a);
    double l2 = dot(ab, ab);
    double s = l2 > 0.0 ? dot(sub(q, a), ab) / l2 : 0.0;
    if (s < 0.0) s = 0.0;
    if (s > 1.0) s = 1.0;
    return len(sub(q, add(a, scl(ab, s))));
}

/* Does primitive id's boundary pass within band*t of the ray at a parameter
 * t in (lo, hi]?  Triangle: the ray/plane point's distance to the nearest edge
 * segment; sphere: |D - r| at the closest-approach parameter (R#22). */
static int boundary_near(const oracle_scene* sc, int id, v3 o, v3 d, double lo, double hi,
                         const oracle_eps* eps, double* margin)
{
    if (id < sc->n_spheres) {
        const double* s = sc->spheres + 4 * id;
        v3 oc = sub(o, ld3(s));
        if (dot(oc, oc) <= s[3] * s[3]) return 0;           /* origin inside: no silhouette */
        double tc = -dot(oc, d);
        if (!(tc > lo && tc <= hi)) return 0;
        double D = len(add(oc, scl(d, tc)));
        double rel = fabs(D - s[3]) / tc;
        if (margin && rel < *margin) *margin = rel;
        return rel <= eps->eps_sphere;
    }
    id -= sc->n_spheres;
    if (id < sc->n_planes) return 0;                         /* infinite: no boundary */
    id -= sc->n_planes;
    v3 v0, v1, v2;
    tri_verts(sc, id, &v0, &v1, &v2);
    v3 n = cross(sub(v1, v0), sub(v2, v0));
    double den = dot(n, d);
    if (den == 0.0) return 0;
    double tp = dot(n, sub(v0, o)) / den;
    if (!(tp > lo && tp <= hi)) return 0;
    v3 q = add(o, scl(d, tp));
    double bd = seg_dist(q, v0, v1);
    double b2 = seg_dist(q, v1, v2), b3 = seg_dist(q, v2, v0);
    if (b2 < bd) bd = b2;
    if (b3 < bd) bd = b3;
    double rel = bd / tp;
    if (margin && rel < *margin) *margin = rel;
    return rel <= eps->eps_edge;
}

/* Any raw candidate parameter of primitive id (inside its extent, ignoring t_min)
 * within `band` of the value `at`? */
static int candidate_near(const oracle_scene* sc, int id, v3 o, v3 d, double at, double band)
{
    if (id < sc->n_spheres) {
        double t0, t1;
        if (!sphere_roots(o, d, sc->spheres + 4 * id, &t0, &t1)) return 0;
        return fabs(t0 - at) <= band || fabs(t1 - at) <= band;
    }
    id -= sc->n_spheres;
    if (id < sc->n_planes) {
        double t;
        if (!plane_t(o, d, sc->planes + 4 * id, &t)) return 0;
        return fabs(t - at) <= band;
    }
    id -= sc->n_planes;
    v3 v0, v1, v2;
    double t, bu, bv;
    tri_verts(sc, id, &v0, &v1, &v2);
    if (!tri_solve(o, d, v0, v1, v2, &t, &bu, &bv)) return 0;
    double tol = 1e-6;
    if (bu < -tol || bv < -tol || bu + bv > 1.0 + tol) return 0;
    return fabs(t - at) <= band;
}

static double abs_band(v3 o, const oracle_eps* eps)
{
    double m = fabs(o.x);
    if (fabs(o.y) > m) m = fabs(o.y);
    if (fabs(o.z) > m) m = fabs(o.z);
    return eps->eps_abs * (1.0 + m);
}

/* Fragility of a nearest-hit query (F1-F5) whose answer is (tstar, hit). */
static unsigned nearest_fragility(const oracle_scene* sc, v3 o, v3 d, double tstar, int hit,
                                  const oracle_eps* eps, double* margin)
{
    unsigned fl = 0;
    int n = n_prims(sc);
    double lim = isinf(tstar) ? INFINITY : tstar * (1.0 + eps->eps_t);
    double ab = abs_band(o, eps);
    for (int i = 0; i < n; ++i) {
        double t;
        if (i != hit && !isinf(tstar) && prim_hit(sc, i, o, d, T_MIN, &t) &&
            fabs(t - tstar) <= eps->eps_t * tstar)
            fl |= FRAG_COMPETE;
        if (boundary_near(sc, i, o, d, 0.5 * T_MIN, lim, eps, margin)) fl |= FRAG_BOUNDARY;
        if (candidate_near(sc, i, o, d, T_MIN, ab)) fl |= FRAG_RANGE;
    }
    if (hit >= 0) {
        v3 p = add(o, scl(d, tstar));
        v3 ng = geo_normal(sc, hit, p);
        if (fabs(dot(ng, d)) <= eps->eps_t) fl |= FRAG_GRAZE;
    }
    return fl;
}

/* Fragility of a shadow query over (t_min, dist): only matters when no primitive
 * robustly occludes the segment. */
static unsigned shadow_fragility(const oracle_scene* sc, v3 o, v3 d, double dist, const oracle_eps* eps)
{
    int n = n_prims(sc);
    double ab = abs_band(o, eps);
    unsigned fl = 0;
    for (int i = 0; i < n; ++i) {
        double t;
        if (prim_hit(sc, i, o, d, T_MIN + ab, &t) && t < dist * (1.0 - eps->eps_t) &&
            !boundary_near(sc, i, o, d, 0.5 * T_MIN, dist, eps, NULL))
            return 0;                                          /* robust occluder */
    }
    for (int i = 0; i < n; ++i) {
        if (boundary_near(sc, i, o, d, 0.5 * T_MIN, dist * (1.0 + eps->eps_t), eps, NULL)) fl |= FRAG_SHADOW;
        if (candidate_near(sc, i, o, d, T_MIN, ab)) fl |= FRAG_SHADOW;
        if (candidate_near(sc, i, o, d, dist, eps->eps_t * dist)) fl |= FRAG_SHADOW;
    }
    return fl;
}

/* ---------------------------------------------------------- near-tie candidates
 * R#22: the IDs a nearest query may legitimately return when its ray is turned by up
 * to the exclusion band, instead of excluding an ID-fragile pixel from the ID check altogether.
 * A primitive is a candidate if the band-widened ray meets it no farther than the nearest
 * primitive the band-widened ray meets robustly (whole band inside it), +eps_t relative:
 *   sphere   : closest-approach distance D <= r + eps_sphere*tc (robust: D <= r - eps_sphere*tc,
 *              or the origin inside the sphere); its t is the entry root (or tc when D > r);
 *   plane    : hit (robust unless grazing, |n.d| <= eps_t);
 *   triangle : the ray/plane point within b = eps_edge*t/max(|n.d|, eps_t) of the triangle (an
 *              angular turn a moves the point by a*t/|n.d| in the plane; robust: inside and more
 *              than b from every edge).
 * A robust hit at t_r bounds the candidates at t_r (1 + eps_t + eps_edge tan(theta_r)): the turn
 * moves the robust surface's own t by up to eps_edge tan(theta_r) relative (theta_r = its angle
 * of incidence), and eps_t is the competing-hit band of F1.
 * Candidates must lie beyond t_min - band_abs; one within band_abs of t_min is never robust (F5).
 * -1 (miss) is a candidate when nothing is hit robustly.  Returns the candidate count; the IDs
 * (ascending, -1 last) go to cand[0..min(count, kmax)). */
static int ray_candidates(const oracle_scene* sc, v3 o, v3 d, const oracle_eps* eps, int32_t* cand, int kmax)
{
    int n = n_prims(sc), nc = 0;
    double ab = abs_band(o, eps);
    double tlim = INFINITY;
    int robust_any = 0;
    /* pass 1: the nearest robust hit bounds the candidates */
    for (int pass = 0; pass < 2; ++pass) {
        for (int i = 0; i < n; ++i) {
            double t = 0.0, tan_th = 0.0;
            int hit = 0, robust = 0;
            if (i < sc->n_spheres) {
                const double* sp = sc->spheres + 4 * i;
                v3 oc = sub(o, ld3(sp));
                double r = sp[3];
                if (dot(oc, oc) <= r * r) {                       /* origin inside: exit root */
                    double t0, t1;
                    if (sphere_roots(o, d, sp, &t0, &t1)) { t = t1; hit = 1; robust = 1; }
                } else {
                    double tc = -dot(oc, d);
                    if (tc > 0.0) {
                        double D = len(add(oc, scl(d, tc)));
                        if (D <= r + eps->eps_sphere * tc) {
                            hit = 1;
                            robust = D <= r - eps->eps_sphere * tc;
                            t = tc;
                            double t0, t1;
                            if (D <= r && sphere_roots(o, d, sp, &t0, &t1)) t = t0;
                        }
                    }
                }
            } else if (i < sc->n_spheres + sc->n_planes) {
                const double* pl = sc->planes + 4 * (i - sc->n_spheres);
                if (plane_t(o, d, pl, &t)) {
                    double cosn = fabs(dot(nrm(ld3(pl)), d));
                    hit = 1;
                    robust = cosn > eps->eps_t;
                    tan_th = robust ? sqrt(1.0 - cosn * cosn) / cosn : 0.0;
                }
            } else {
                v3 v0, v1, v2;
                tri_verts(sc, i - sc->n_spheres - sc->n_planes, &v0, &v1, &v2);
                v3 nn = cross(sub(v1, v0), sub(v2, v0));
                double den = dot(nn, d);
                if (den != 0.0) {
                    t = dot(nn, sub(v0, o)) / den;
                    double cosn = fabs(den) / len(nn);
                    double b = eps->eps_edge * fabs(t) / (cosn > eps->eps_t ? cosn : eps->eps_t);
                    v3 q = add(o, scl(d, t));
                    double e = seg_dist(q, v0, v1), e2 = seg_dist(q, v1, v2), e3 = seg_dist(q, v2, v0);
                    if (e2 < e) e = e2;
                    if (e3 < e) e = e3;
                    /* inside test of q in the triangle's plane (same-side of every edge) */
                    double s0 = dot(cross(sub(v1, v0), sub(q, v0)), nn);
                    double s1 = dot(cross(sub(v2, v1), sub(q, v1)), nn);
                    double s2 = dot(cross(sub(v0, v2), sub(q, v2)), nn);
                    int inside = s0 >= 0.0 && s1 >= 0.0 && s2 >= 0.0;
                    hit = inside || e <= b;
                    robust = inside && e > b && cosn > eps->eps_t;
                    tan_th = robust ? sqrt(1.0 - cosn * cosn) / cosn : 0.0;
                }
            }
            if (!hit || t <= T_MIN - ab) continue;
            if (fabs(t - T_MIN) <= ab) robust = 0;                 /* F5: the t_min decision */
            if (pass == 0) {
                if (robust) {
                    double lim = t * (1.0 + eps->eps_t + eps->eps_edge * tan_th);
                    robust_any = 1;
                    if (lim < tlim) tlim = lim;
                }
            } else if (t <= tlim) {
                if (nc < kmax) cand[nc] = i;
                ++nc;
            }
        }
    }
    if (!robust_any) {
        if (nc < kmax) cand[nc] = -1;
        ++nc;
    }
    return nc;
}

/* ------------------------------------------------------------------ trace */
typedef struct {
    const oracle_scene* sc;
    const oracle_eps* eps;   /* NULL: no fragility analysis */
    unsigned flags;          /* union over every ray of the tree */
    ray_counts cnt;
} trace_ctx;

/* S:200-208 trace + S:190-198 shade, extended per SURVEY §8(c) step 4:
 * ambient*kd + sum_lights visible*(kd*I*ndl + ks*I*max(0, r.v)^n)   (R#1-3)
 * + kt*trace(refracted) (R#5-6) + kr_eff*trace(reflected)
 * max_depth = bounces still allowed (R#7). */
static v3 trace(trace_ctx* cx, v3 o, v3 d, int depth, int is_primary, int32_t* id_out,
                unsigned* primary_flags, double* margin)
{
    const oracle_scene* sc = cx->sc;
    double tstar;
    int32_t hit;
    double o3[3] = {o.x, o.y, o.z}, d3[3] = {d.x, d.y, d.z};
    oracle_nearest(sc, o3, d3, &tstar, &hit);
    if (cx->eps) {
        unsigned f = nearest_fragility(sc, o, d, tstar, hit, cx->eps, is_primary ? margin : NULL);
        cx->flags |= f;
        if (is_primary && primary_flags) *primary_flags = f;
    }
    if (is_primary && id_out) *id_out = hit;
    if (hit < 0) return ld3(sc->background);                    /* S:203 miss -> background */

    v3 p = add(o, scl(d, tstar));
    v3 ng = geo_normal(sc, hit, p);
    int front = dot(d, ng) < 0.0;
    v3 nf = front ? ng : scl(ng, -1.0);                          /* S:150 faces the ray */
    const double* m = sc->mats + 10 * prim_material(sc, hit);
    v3 kd = ld3(m), ks = ld3(m + 3);
    double shin = m[6], kr = m[7], kt = m[8], ior = m[9];

    v3 c = mul(ld3(sc->ambient), kd);                            /* S:193 ambient*diffuse */
    for (int j = 0; j < sc->n_lights; ++j) {
        const double* L = sc->lights + 6 * j;
        v3 Lv = sub(ld3(L), p);
        v3 l = nrm(Lv);
        double ndl = dot(nf, l);
        if (cx->eps && fabs(ndl) <= cx->eps->eps_t) cx->flags |= FRAG_SHADE;
        if (ndl <= 0.0) continue;                                /* R#2 gate */
        v3 os = add(p, scl(nf, BIAS));                           /* S:193 p + bias*n */
        v3 sv = sub(ld3(L), os);
        double dist = len(sv);
        v3 sd = scl(sv, 1.0 / dist);
        cx->cnt.shadow++;
        if (cx->eps) cx->flags |= shadow_fragility(sc, os, sd, dist, cx->eps);
        if (occluded(sc, os, sd, dist)) continue;
        v3 I = ld3(L + 3);
        v3 rv = sub(scl(nf, 2.0 * ndl), l);                      /* r = 2(n.l)n - l */
        double rdv = -dot(rv, d);
        double spec = rdv > 0.0 ? pow(rdv, shin) : 0.0;
        c = add(c, scl(mul(kd, I), ndl));                        /* no falloff, R#3 */
        c = add(c, scl(mul(ks, I), spec));
    }
    if (depth > 0) {
        double kr_eff = kr;
        if (kt > 0.0) {
            double eta = front ? 1.0 / ior : ior;                /* R#6 outside ior = 1 */
            double cosi = -dot(d, nf);
            double k = 1.0 - eta * eta * (1.0 - cosi * cosi);
            if (cx->eps && fabs(k) <= cx->eps->eps_t) cx->flags |= FRAG_SHADE;
            if (k < 0.0) {
                kr_eff += kt;                                    /* R#5 TIR */
            } else {
                v3 td = nrm(add(scl(d, eta), scl(nf, eta * cosi - sqrt(k))));
                cx->cnt.refraction++;
                v3 ct = trace(cx, sub(p, scl(nf, BIAS)), td, depth - 1, 0, NULL, NULL, NULL);
                c = add(c, scl(ct, kt));
            }
        }
        if (kr_eff > 0.0) {
            v3 rd = nrm(sub(d, scl(nf, 2.0 * dot(d, nf))));      /* S:211 d - 2(d.n)n */
            cx->cnt.reflection++;
            v3 cr = trace(cx, add(p, scl(nf, BIAS)), rd, depth - 1, 0, NULL, NULL, NULL);
            c = add(c, scl(cr, kr_eff));
        }
    }
    return c;
}

/* Trace one arbitrary ray (tests).  rgb = unclamped radiance. */
void oracle_trace_ray(const oracle_scene* sc, const double o[3], const double d[3], int32_t depth,
                      double rgb[3], long long counts[4])
{
    trace_ctx cx;
    memset(&cx, 0, sizeof cx);
    cx.sc = sc;
    v3 c = trace(&cx, ld3(o), nrm(ld3(d)), depth, 0, NULL, NULL, NULL);
    rgb[0] = c.x; rgb[1] = c.y; rgb[2] = c.z;
    if (counts) {
        counts[0] = cx.cnt.primary; counts[1] = cx.cnt.reflection;
        counts[2] = cx.cnt.refraction; counts[3] = cx.cnt.shadow;
    }
}

/* Trace one ray with the fragility analysis on (pins of F1-F6 and the shadow flags): rgb =
 * unclamped radiance, *flags = union of the flags of every ray of the tree (R#22). */
void oracle_trace_ray_ex(const oracle_scene* sc, const double o[3], const double d[3], int32_t depth,
                         const oracle_eps* eps, double rgb[3], long long counts[4], uint32_t* flags)
{
    trace_ctx cx;
    memset(&cx, 0, sizeof cx);
    cx.sc = sc;
    cx.eps = eps;
    v3 c = trace(&cx, ld3(o), nrm(ld3(d)), depth, 0, NULL, NULL, NULL);
    rgb[0] = c.x; rgb[1] = c.y; rgb[2] = c.z;
    if (counts) {
        counts[0] = cx.cnt.primary; counts[1] = cx.cnt.reflection;
        counts[2] = cx.cnt.refraction; counts[3] = cx.cnt.shadow;
    }
    if (flags) *flags = cx.flags;
}

/* Fragility of ONE query (pins of the classifier):
 *   kind 0: nearest-hit query along (o, d) -> F1-F5 flags of its answer (+ min boundary margin)
 *   kind 1: shadow (any-hit) query over (t_min, dist) -> FRAG_SHADOW or 0 */
uint32_t oracle_ray_flags(const oracle_scene* sc, const double o3[3], const double d3[3], int32_t kind,
                          double dist, const oracle_eps* eps, double* margin)
{
    v3 o = ld3(o3), d = nrm(ld3(d3));
    if (kind == 1) return shadow_fragility(sc, o, d, dist, eps);
    double dn[3] = {d.x, d.y, d.z}, t;
    int32_t id;
    oracle_nearest(sc, o3, dn, &t, &id);
    double mg = INFINITY;
    uint32_t f = nearest_fragility(sc, o, d, t, id, eps, &mg);
    if (margin) *margin = mg;
    return f;
}

/* Near-tie candidate IDs of the nearest query along (o, d) (see ray_candidates). */
int32_t oracle_ray_candidates(const oracle_scene* sc, const double o3[3], const double d3[3],
                              const oracle_eps* eps, int32_t* cand, int32_t kmax)
{
    return ray_candidates(sc, ld3(o3), nrm(ld3(d3)), eps, cand, kmax);
}

/* byte = clamp(round(c*255)), round half away from zero (= floor(x+0.5), x>=0). */
static uint8_t q8(double c)
{
    if (!(c > 0.0)) c = 0.0;
    if (c > 1.0) c = 1.0;
    return (uint8_t)floor(255.0 * c + 0.5);
}

/* IEEE binary16 bits of c (c in [0,1] after clamp), round-to-nearest-even (R#16). */
uint16_t oracle_half_bits(double c)
{
    if (!(c > 0.0)) return 0;
    if (c >= 1.0) return 0x3C00;
    int e;
    double m = frexp(c, &e);          /* c = m * 2^e, m in [0.5,1) */
    int E = e - 1;                    /* c = (2m) * 2^E, 2m in [1,2) */
    if (E < -14) {                    /* subnormal: units of 2^-24 */
        double q = nearbyint(ldexp(c, 24));
        return (uint16_t)q;           /* q <= 1024 -> 0x0400 is the smallest normal, still correct */
    }
    double frac = nearbyint((2.0 * m - 1.0) * 1024.0);   /* 10-bit mantissa, RNE */
    int ex = E + 15;
    if (frac >= 1024.0) { frac = 0.0; ex += 1; }
    return (uint16_t)((ex << 10) | (int)frac);
}

/*
 * Render a list of pixels (or every pixel of both eyes when pix == NULL; order
 * eye-major, then row-major, top row first -- S:499).
 *   pix       : n_pix (eye, px, py) int32 triples, or NULL
 *   radiance  : n*3 doubles, UNclamped linear radiance                (may be NULL)
 *   rgba8     : n*4 bytes, S:494 quantisation, A = 255                (may be NULL)
 *   rgba16    : n*4 uint16 binary16 of the clamped radiance, A = 1.0  (may be NULL)
 *   prim_id   : n int32 primary nearest-hit global ID, -1 = miss (R#20) (may be NULL)
 *   pflags    : n primary-ray fragility masks (F1-F5)                 (may be NULL)
 *   tflags    : n fragility masks over every ray of the pixel's tree   (may be NULL)
 *   margin    : n min relative boundary distance seen by the primary ray (may be NULL)
 *   counts    : 4 totals (primary, reflection, refraction, shadow)     (may be NULL)
 *   eps       : fragility thresholds, NULL -> no fragility analysis
 *   cand      : n*cand_k near-tie candidate IDs of the primary ray, only for pixels with an
 *               ID-fragile primary (F1-F5); padding -2                 (may be NULL; needs eps)
 *   ncand     : n candidate counts (0 for ID-robust pixels)            (may be NULL)
 */
int oracle_render(const oracle_scene* sc, const oracle_cam* cam, int32_t max_depth,
                  int64_t n_pix, const int32_t* pix,
                  double* radiance, uint8_t* rgba8, uint16_t* rgba16, int32_t* prim_id,
                  uint32_t* pflags, uint32_t* tflags, double* margin,
                  long long* counts, const oracle_eps* eps, int32_t n_threads,
                  int32_t* cand, int32_t cand_k, int32_t* ncand)
{
    int64_t n = pix ? n_pix : 2LL * cam->width * cam->height;
    long long c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    if (max_depth < 0) return 1;
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
    #pragma omp parallel for schedule(dynamic, 16) reduction(+:c0,c1,c2,c3)
    for (int64_t k = 0; k < n; ++k) {
        int32_t eye, px, py;
        if (pix) { eye = pix[3 * k]; px = pix[3 * k + 1]; py = pix[3 * k + 2]; }
        else {
            int64_t wh = (int64_t)cam->width * cam->height;
            eye = (int32_t)(k / wh);
            px = (int32_t)((k % wh) % cam->width);
            py = (int32_t)((k % wh) / cam->width);
        }
        double o[3], d[3];
        oracle_primary_ray(cam, eye, px, py, o, d);
        trace_ctx cx;
        memset(&cx, 0, sizeof cx);
        cx.sc = sc;
        cx.eps = eps;
        cx.cnt.primary = 1;
        int32_t id = -1;
        unsigned pf = 0;
        double mg = INFINITY;
        v3 c = trace(&cx, ld3(o), ld3(d), max_depth, 1, &id, &pf, &mg);
        if (eps && eps->perturb > 0.0) {
            /* F7 (reading 22): curved mirrors and glass amplify angular error at every
             * bounce (~2D/r), so a deep ray can cross a silhouette that the unperturbed tree misses
             * by more than the band.  Re-trace with the primary ray turned in four directions by
             * `perturb`, perturb / 10 and perturb / 33 rad (1e-6, 1e-7, 3e-8: from ~10x down to the
             * FP32 rounding of a unit direction; the response is not monotonic in the turn -- a deep
             * ray can graze a boundary at one scale and not at the others, as the full-frame C3
             * report found); a clamped radiance change above perturb_tol marks the pixel unstable. */
            v3 dv = ld3(d);
            v3 a = fabs(dv.y) < 0.9 ? mk(0, 1, 0) : mk(1, 0, 0);
            v3 u = nrm(cross(dv, a)), w = cross(dv, u);
            v3 dirs[4] = {u, scl(u, -1.0), w, scl(w, -1.0)};
            const double scale[3] = {1.0, 0.1, 1.0 / 33.0};
            for (int q = 0; q < 12 && !(cx.flags & FRAG_UNSTABLE); ++q) {
                trace_ctx cq;
                memset(&cq, 0, sizeof cq);
                cq.sc = sc;
                v3 dq = nrm(add(dv, scl(dirs[q & 3], eps->perturb * scale[q >> 2])));
                v3 cc = trace(&cq, ld3(o), dq, max_depth, 0, NULL, NULL, NULL);
                double dc[3] = {cc.x, cc.y, cc.z}, c0[3] = {c.x, c.y, c.z};
                for (int k = 0; k < 3; ++k) {
                    double x0 = c0[k] < 0 ? 0 : (c0[k] > 1 ? 1 : c0[k]);
                    double x1 = dc[k] < 0 ? 0 : (dc[k] > 1 ? 1 : dc[k]);
                    if (fabs(x1 - x0) > eps->perturb_tol) cx.flags |= FRAG_UNSTABLE;
                }
            }
        }
        if (radiance) { radiance[3 * k] = c.x; radiance[3 * k + 1] = c.y; radiance[3 * k + 2] = c.z; }
        if (rgba8) {
            rgba8[4 * k] = q8(c.x); rgba8[4 * k + 1] = q8(c.y); rgba8[4 * k + 2] = q8(c.z);
            rgba8[4 * k + 3] = 255;
        }
        if (rgba16) {
            rgba16[4 * k] = oracle_half_bits(c.x); rgba16[4 * k + 1] = oracle_half_bits(c.y);
            rgba16[4 * k + 2] = oracle_half_bits(c.z); rgba16[4 * k + 3] = 0x3C00;
        }
        if (cand && cand_k > 0) {
            for (int q = 0; q < cand_k; ++q) cand[k * cand_k + q] = -2;
            int32_t nc = 0;
            if (eps && (pf & (FRAG_COMPETE | FRAG_BOUNDARY | FRAG_GRAZE | FRAG_RANGE)))
                nc = ray_candidates(sc, ld3(o), ld3(d), eps, cand + k * cand_k, cand_k);
            if (ncand) ncand[k] = nc;
        }
        if (prim_id) prim_id[k] = id;
        if (pflags) pflags[k] = pf;
        if (tflags) tflags[k] = cx.flags;
        if (margin) margin[k] = mg;
        c0 += cx.cnt.primary; c1 += cx.cnt.reflection; c2 += cx.cnt.refraction; c3 += cx.cnt.shadow;
    }
    if (counts) { counts[0] = c0; counts[1] = c1; counts[2] = c2; counts[3] = c3; }
    return 0;
}

/* PAPER.md:56 post-processing "anaglyph/Anamorphic transformation"; SPEC.md:445 compose_anaglyph:
 * out(r,g,b) = (left.r, right.g, right.b), alpha 255.  RGBA8, W x H, row-major. */
void oracle_compose_anaglyph(const uint8_t* L, const uint8_t* R, int32_t W, int32_t H, uint8_t* out)
{
    for (int64_t i = 0; i < (int64_t)W * H; ++i) {
        out[4 * i + 0] = L[4 * i + 0];
        out[4 * i + 1] = R[4 * i + 1];
        out[4 * i + 2] = R[4 * i + 2];
        out[4 * i + 3] = 255;
    }
}

/* SPEC.md:455 compose_sbs: each channel squeezed to floor(W/2) columns by column-pair
 * averaging (per-channel integer mean, round half up), left | right; out is 2*floor(W/2) x H. */
void oracle_compose_sbs(const uint8_t* L, const uint8_t* R, int32_t W, int32_t H, uint8_t* out)
{
    int32_t half = W / 2, ow = 2 * half;
    for (int32_t y = 0; y < H; ++y) {
        for (int32_t x = 0; x < ow; ++x) {
            const uint8_t* img = x < half ? L : R;
            int32_t j = x < half ? x : x - half;
            const uint8_t* a = img + 4 * ((int64_t)y * W + 2 * j);
            const uint8_t* b = a + 4;
            uint8_t* o = out + 4 * ((int64_t)y * ow + x);
            for (int k = 0; k < 3; ++k) {
                int sum = a[k] + b[k];
                o[k] = (uint8_t)(sum / 2 + sum % 2);   /* mean rounded half up */
            }
            o[3] = 255;
        }
    }
}

int oracle_version(void) { return ORACLE_VERSION; }
