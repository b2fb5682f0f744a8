/*
 * sg_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the contiguous
 * sparse-grid hot path of Gu & Hu, "Contiguous Storage of Grid Data for
 * Heterogeneous Computing" (arXiv 2512.11473; /root/reference/PAPER.md, cited
 * below as P:<line>).  Everything is fp64 on a DENSE fine grid of M = 4N points
 * per axis; the sparse package structure is produced only as the tables the
 * paper defines (background table, meta, 27-neighbour table), so that the CUDA
 * path's tables can be checked for identity and its fields scattered/gathered
 * against dense arrays.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code, header,
 * helper or constant generator with the CUDA path (paper_2512_11473_b200/)
 * and neither side includes or imports the other.
 *
 * Where PAPER.md is silent the reading taken is the one listed in DESIGN.md
 * "Readings" (R-1 .. R-20, same numbering as SURVEY.md 8(c.3)).
 *
 * Build: gcc -O3 -march=native -fopenmp -ffp-contract=off -fPIC -shared (no
 * -ffast-math; one library per host CPU): every double operation is a
 * separately rounded IEEE operation in the order written, which is what makes
 * the tagging decision |f| < l_c reproducible.
 *
 * Box windows (or_grid.win_lo / win_n): O6-O10 may be evaluated on a box of
 * the dense grid only (the definition restricted to the box; values outside
 * it are the initial phi) -- how C3 / C5 are checked and timed, where the
 * whole dense grid does not fit in memory (69 GB / 550 GB per field).
 *
 * Parity status per function:
 *   or_sdf            pinned: closed forms + brute-force surface sampling
 *   or_tag/or_compact pinned: brute-force definition on tiny grids, invariants,
 *                     independent counts
 *   or_neighbours     pinned: definition by brute force, invariants
 *   or_phi_dense      pinned: closed-form SDF values
 *   or_reinit_dense   pinned: planar closed form, 2*SDF convergence, no sign
 *                     flip, one-step Godunov closed forms at ridges/valleys
 *                     of both signs along each axis (upwind selection), phi=0
 *                     stationary; multi-step drift near kinks/medial axes of
 *                     real geometries: the composition of the pinned step
 *   or_gradient_dense pinned: affine exactness, sphere radial, and bit for bit
 *                     numpy.gradient's central difference on the far-filled
 *                     dense field at every interior active point, band edge
 *                     included
 *   or_kernel_dense   pinned: S closed forms, S/2 at planar interface, sum gw=0,
 *                     first moment sum gw_x o_x dx -> int W = 1 (G scale),
 *                     scaling identity r W' = -h dW/dh - 3W from the weights,
 *                     Heaviside C^1 conditions H'(0)=1/eps, H'(+-eps)=0
 *   or_probe          pinned: affine reproduction, data-point identity, far/OOB
 *   or_relax          pinned: lone particle at rest, pair symmetry, pair-force
 *                     magnitude through the normalisation int 4 pi r^2 W = 1,
 *                     bounding onto phi = -off on a plane
 *   or_table1_dense   pinned: Laplacian of x^2+y^2+z^2 = 6, of affine = 0
 *   or_sdf leak post-op / or_sign_correct
 *                     pinned: on leaky spheres / tori the corrected signs equal
 *                     the closed-form containment sign at every data point and
 *                     cell, magnitudes are unchanged, a watertight input is a
 *                     fixed point, flood sweep counts = scipy taxicab distance
 *   or_mesh_sdf       pinned: a 12-triangle box mesh reproduces the box SDF
 *                     closed form; icosphere distances within the sagitta of
 *                     the sphere's, signs = containment; invariance under
 *                     triangle re-ordering
 *   or_clean          pinned: planar slab (K = S/2 at the surface) is a fixed
 *                     point, a fin thinner than h is removed while a thick fin
 *                     and the slab keep their signs, a second call raises
 *                     nothing (idempotence)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Primitive kinds: the numeric values are part of the C-ABI contract
 * (include/sg.h documents the same numbers); they are restated here, not
 * shared. */
enum {
    OR_SPHERE = 0,     /* p = cx cy cz r                         */
    OR_SHELL = 1,      /* p = cx cy cz r_in r_out                */
    OR_BOX = 2,        /* p = cx cy cz bx by bz (half extents)   */
    OR_TORUS_X = 3,    /* p = cx cy cz R r, symmetry axis x      */
    OR_TORUS_Y = 4,    /* p = cx cy cz R r, symmetry axis y      */
    OR_TORUS_Z = 5,    /* p = cx cy cz R r, symmetry axis z      */
    OR_TRIPRISM_Z = 6, /* p = ax ay bx by cx cy z0 z1 (ccw in xy) */
    OR_LEAK = 7        /* p = cx cy cz r margin: sign-error ball   */
};

typedef struct {
    int32_t kind;
    int32_t pad;
    double p[12];
} or_prim;

typedef struct {
    double lower[3];
    double cell;      /* l_c, Fig. 2 caption P:189-191 */
    int32_t n[3];     /* background cells per axis                */
    int32_t pad;
    double far;       /* far-field magnitude, reading R-4          */
    double init_scale;
    /* Box window (0 = the whole domain): the dense arrays of O6-O10 cover
     * only the fine points [win_lo, win_lo + win_n) per axis (global fine
     * indices).  A dense value read outside the box but inside the domain is
     * the initial phi O6 of that point (the window-edge condition): after k
     * reinit sweeps its error has travelled k points into the box (the
     * 7-point dependence cone), so the box interior at depth > k plus the
     * stencil radius of later steps is the whole-domain definition exactly.
     * This is the definition restricted to a box, for configurations whose
     * dense grid does not fit in memory (C3, C5).  O7 sign
     * correction, cleaning and relaxation are whole-domain only. */
    int32_t win_lo[3];
    int32_t win_n[3];
} or_grid;

static inline int full_domain(const or_grid* g) {
    return g->win_n[0] <= 0 || g->win_n[1] <= 0 || g->win_n[2] <= 0;
}

#define PKG 4 /* subdivision size, "default by 4"; fixed (R-9) */

/* ------------------------------------------------------------------ O1 -- */
/* Signed distance of the analytic primitives; negative inside.  The paper
 * evaluates the level set from a signed-distance function; analytic
 * SDFs stand in for the triangle-mesh SDF (out of scope). */

static double sdf_prim(const or_prim* q, const double x[3]) {
    const double* p = q->p;
    switch (q->kind) {
    case OR_SPHERE: {
        double ex = x[0] - p[0], ey = x[1] - p[1], ez = x[2] - p[2];
        return sqrt((ex * ex + ey * ey) + ez * ez) - p[3];
    }
    case OR_SHELL: {
        double ex = x[0] - p[0], ey = x[1] - p[1], ez = x[2] - p[2];
        double rm = 0.5 * (p[3] + p[4]);
        double hw = 0.5 * (p[4] - p[3]);
        return fabs(sqrt((ex * ex + ey * ey) + ez * ez) - rm) - hw;
    }
    case OR_BOX: {
        double qx = fabs(x[0] - p[0]) - p[3];
        double qy = fabs(x[1] - p[1]) - p[4];
        double qz = fabs(x[2] - p[2]) - p[5];
        double mx = fmax(qx, 0.0), my = fmax(qy, 0.0), mz = fmax(qz, 0.0);
        return sqrt((mx * mx + my * my) + mz * mz) + fmin(fmax(qx, fmax(qy, qz)), 0.0);
    }
    case OR_TORUS_X: {
        double ex = x[0] - p[0], ey = x[1] - p[1], ez = x[2] - p[2];
        double t = sqrt(ey * ey + ez * ez) - p[3];
        return sqrt(t * t + ex * ex) - p[4];
    }
    case OR_TORUS_Y: {
        double ex = x[0] - p[0], ey = x[1] - p[1], ez = x[2] - p[2];
        double t = sqrt(ex * ex + ez * ez) - p[3];
        return sqrt(t * t + ey * ey) - p[4];
    }
    case OR_TORUS_Z: {
        double ex = x[0] - p[0], ey = x[1] - p[1], ez = x[2] - p[2];
        double t = sqrt(ex * ex + ey * ey) - p[3];
        return sqrt(t * t + ez * ez) - p[4];
    }
    case OR_TRIPRISM_Z: {
        /* exact 2-D triangle SDF: clamped point-segment distance to each
         * edge, negative iff strictly left of all three (ccw) edges */
        double dmin = 0.0;
        int inside = 1;
        for (int e = 0; e < 3; ++e) {
            double ax = p[2 * e], ay = p[2 * e + 1];
            double bx = p[2 * ((e + 1) % 3)], by = p[2 * ((e + 1) % 3) + 1];
            double ux = bx - ax, uy = by - ay;
            double wx = x[0] - ax, wy = x[1] - ay;
            double t = (wx * ux + wy * uy) / (ux * ux + uy * uy);
            t = fmin(fmax(t, 0.0), 1.0);
            double dx = wx - ux * t, dy = wy - uy * t;
            double d2 = dx * dx + dy * dy;
            dmin = (e == 0) ? d2 : fmin(dmin, d2);
            double cr = ux * wy - uy * wx;
            if (!(cr > 0.0)) inside = 0;
        }
        double d2s = inside ? -sqrt(dmin) : sqrt(dmin);
        double zc = 0.5 * (p[6] + p[7]);
        double hl = 0.5 * (p[7] - p[6]);
        double qz = fabs(x[2] - zc) - hl;
        double mxy = fmax(d2s, 0.0), mz = fmax(qz, 0.0);
        return fmin(fmax(d2s, qz), 0.0) + sqrt(mxy * mxy + mz * mz);
    }
    default:
        return NAN;
    }
}

/* ------------------------------------------------------------ NEXT-4 -- */
/* Signed distance to a closed triangle mesh ("using the
 * sign-distance function from triangle mesh", ref. baerentzen2005robust;
 * reading R-24): nearest triangle by squared distance (ties: lowest index),
 * closest point on a triangle by its Voronoi regions (Ericson, RTCD 5.1.5),
 * sign of (x - q) . N with N the angle-weighted pseudonormal of the closest
 * feature.  Brute force over every triangle.  One registered mesh at a time
 * (test infrastructure); a geometry with no primitives means "the mesh". */
static struct {
    int32_t nv, nt;
    double *V, *fn, *en, *vn;
    int32_t* T;
} g_mesh;

static double dot3(const double* a, const double* b) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

void or_mesh_set(const double* V, const int32_t* T, int32_t nv, int32_t nt) {
    free(g_mesh.V);
    free(g_mesh.T);
    free(g_mesh.fn);
    free(g_mesh.en);
    free(g_mesh.vn);
    memset(&g_mesh, 0, sizeof(g_mesh));
    if (nt <= 0) return;
    g_mesh.nv = nv;
    g_mesh.nt = nt;
    g_mesh.V = (double*)malloc(sizeof(double) * 3 * nv);
    g_mesh.T = (int32_t*)malloc(sizeof(int32_t) * 3 * nt);
    memcpy(g_mesh.V, V, sizeof(double) * 3 * nv);
    memcpy(g_mesh.T, T, sizeof(int32_t) * 3 * nt);
    g_mesh.fn = (double*)calloc((size_t)3 * nt, sizeof(double));
    g_mesh.en = (double*)calloc((size_t)9 * nt, sizeof(double));
    g_mesh.vn = (double*)calloc((size_t)3 * nv, sizeof(double));
    /* unit face normals (b - a) x (c - a) / |.| */
    for (int t = 0; t < nt; ++t) {
        const double *a = V + 3 * T[3 * t], *b = V + 3 * T[3 * t + 1], *c = V + 3 * T[3 * t + 2];
        double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        double w[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
        double n[3] = {u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2],
                       u[0] * w[1] - u[1] * w[0]};
        double l = sqrt(dot3(n, n));
        for (int k = 0; k < 3; ++k) g_mesh.fn[3 * t + k] = l > 0.0 ? n[k] / l : 0.0;
    }
    /* vertex pseudonormal: sum over corners (triangle order) of angle * n */
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) {
            int i = T[3 * t + k], j = T[3 * t + (k + 1) % 3], m = T[3 * t + (k + 2) % 3];
            const double* p = V + 3 * i;
            double u[3] = {V[3 * j] - p[0], V[3 * j + 1] - p[1], V[3 * j + 2] - p[2]};
            double w[3] = {V[3 * m] - p[0], V[3 * m + 1] - p[1], V[3 * m + 2] - p[2]};
            double lu = sqrt(dot3(u, u)), lw = sqrt(dot3(w, w));
            double cs = (lu > 0.0 && lw > 0.0) ? dot3(u, w) / (lu * lw) : 1.0;
            if (cs > 1.0) cs = 1.0;
            if (cs < -1.0) cs = -1.0;
            double ang = acos(cs);
            for (int q = 0; q < 3; ++q) g_mesh.vn[3 * i + q] += ang * g_mesh.fn[3 * t + q];
        }
    /* edge pseudonormal: n_t + n_t' of the two faces of an edge (brute-force
     * search for the triangle holding the reversed edge) */
    for (int t = 0; t < nt; ++t)
        for (int e = 0; e < 3; ++e) {
            int i = T[3 * t + e], j = T[3 * t + (e + 1) % 3], other = -1;
            for (int u = 0; u < nt && other < 0; ++u)
                for (int f = 0; f < 3; ++f)
                    if (T[3 * u + f] == j && T[3 * u + (f + 1) % 3] == i) {
                        other = u;
                        break;
                    }
            for (int q = 0; q < 3; ++q)
                g_mesh.en[9 * t + 3 * e + q] =
                    other < 0 ? g_mesh.fn[3 * t + q] : g_mesh.fn[3 * t + q] + g_mesh.fn[3 * other + q];
        }
}

/* closest point q of p on triangle (a, b, c); region 0 face, 1..3 vertex
 * a/b/c, 4..6 edge ab/bc/ca (Ericson, RTCD 5.1.5) */
static int tri_closest(const double* a, const double* b, const double* c, const double* p,
                       double* q) {
    double ab[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    double ac[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
    double ap[3] = {p[0] - a[0], p[1] - a[1], p[2] - a[2]};
    double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0) {
        memcpy(q, a, 3 * sizeof(double));
        return 1;
    }
    double bp[3] = {p[0] - b[0], p[1] - b[1], p[2] - b[2]};
    double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
    if (d3 >= 0.0 && d4 <= d3) {
        memcpy(q, b, 3 * sizeof(double));
        return 2;
    }
    double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        double v = d1 / (d1 - d3);
        for (int k = 0; k < 3; ++k) q[k] = a[k] + v * ab[k];
        return 4;
    }
    double cp[3] = {p[0] - c[0], p[1] - c[1], p[2] - c[2]};
    double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
    if (d6 >= 0.0 && d5 <= d6) {
        memcpy(q, c, 3 * sizeof(double));
        return 3;
    }
    double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        double w = d2 / (d2 - d6);
        for (int k = 0; k < 3; ++k) q[k] = a[k] + w * ac[k];
        return 6;
    }
    double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        for (int k = 0; k < 3; ++k) q[k] = b[k] + w * (c[k] - b[k]);
        return 5;
    }
    double den = 1.0 / ((va + vb) + vc);
    double v = vb * den, w = vc * den;
    for (int k = 0; k < 3; ++k) q[k] = (a[k] + ab[k] * v) + ac[k] * w;
    return 0;
}

double or_mesh_sdf(const double x[3]) {
    double best = 0.0, bq[3] = {0.0, 0.0, 0.0};
    int bt = -1, breg = 0;
    for (int t = 0; t < g_mesh.nt; ++t) {
        const int32_t* tv = g_mesh.T + 3 * t;
        double q[3];
        int reg = tri_closest(g_mesh.V + 3 * tv[0], g_mesh.V + 3 * tv[1], g_mesh.V + 3 * tv[2], x, q);
        double e0 = x[0] - q[0], e1 = x[1] - q[1], e2 = x[2] - q[2];
        double d2 = (e0 * e0 + e1 * e1) + e2 * e2;
        if (bt < 0 || d2 < best) {
            best = d2;
            bt = t;
            breg = reg;
            memcpy(bq, q, sizeof(bq));
        }
    }
    if (bt < 0) return INFINITY;
    double d = sqrt(best);
    const double* N;
    if (breg == 0) N = g_mesh.fn + 3 * bt;
    else if (breg <= 3) N = g_mesh.vn + 3 * g_mesh.T[3 * bt + breg - 1];
    else N = g_mesh.en + 9 * bt + 3 * (breg - 4);
    double s = ((x[0] - bq[0]) * N[0] + (x[1] - bq[1]) * N[1]) + (x[2] - bq[2]) * N[2];
    return s < 0.0 ? -d : d;
}

static int mesh_mode(int32_t n_prims) { return n_prims == 0 && g_mesh.nt > 0; }

/* union = min over the primitives, in order; then the leak post-operation
 * (include/sg.h SG_LEAK; models the wrong signs of a triangle-mesh SDF on
 * leaky input): f -> -f strictly inside any leak ball where
 * |f| >= margin. */
double or_sdf(const or_prim* prims, int32_t n_prims, const double x[3]) {
    if (mesh_mode(n_prims)) return or_mesh_sdf(x);
    double f = INFINITY;
    int first = 1;
    for (int i = 0; i < n_prims; ++i) {
        if (prims[i].kind == OR_LEAK) continue;
        double g = sdf_prim(&prims[i], x);
        f = first ? g : fmin(f, g);
        first = 0;
    }
    int flip = 0;
    for (int i = 0; i < n_prims; ++i) {
        if (prims[i].kind != OR_LEAK) continue;
        const double* l = prims[i].p;
        double ex = x[0] - l[0], ey = x[1] - l[1], ez = x[2] - l[2];
        if ((ex * ex + ey * ey) + ez * ez < l[3] * l[3] && fabs(f) >= l[4]) flip = 1;
    }
    return flip ? -f : f;
}

void or_sdf_batch(const or_prim* prims, int32_t n_prims, int64_t n, const double* x,
                  double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = or_sdf(prims, n_prims, x + 3 * i);
}

/* ------------------------------------------------------------- helpers -- */

static inline int64_t lin_cell(const or_grid* g, int64_t cx, int64_t cy, int64_t cz) {
    /* R-1: x fastest, z slowest */
    return cx + (int64_t)g->n[0] * (cy + (int64_t)g->n[1] * cz);
}

/* O2: centre of background cell c; multiply and add rounded separately */
static inline void cell_centre(const or_grid* g, int64_t cx, int64_t cy, int64_t cz,
                               double x[3]) {
    x[0] = g->lower[0] + ((double)cx + 0.5) * g->cell;
    x[1] = g->lower[1] + ((double)cy + 0.5) * g->cell;
    x[2] = g->lower[2] + ((double)cz + 0.5) * g->cell;
}

static inline double data_spacing(const or_grid* g) { return g->cell / (double)PKG; }

/* R-11: data point I sits at lower + (I + 0.5) dx */
static inline void point_pos(const or_grid* g, int64_t ix, int64_t iy, int64_t iz,
                             double x[3]) {
    double dx = data_spacing(g);
    x[0] = g->lower[0] + ((double)ix + 0.5) * dx;
    x[1] = g->lower[1] + ((double)iy + 0.5) * dx;
    x[2] = g->lower[2] + ((double)iz + 0.5) * dx;
}

double or_far(const or_grid* g) {
    /* R-4: far = 4 l_c max(1, init_scale) unless given */
    if (g->far > 0.0) return g->far;
    double s = g->init_scale > 0.0 ? g->init_scale : 1.0;
    return 4.0 * g->cell * (s > 1.0 ? s : 1.0);
}

static inline double init_scale(const or_grid* g) {
    return g->init_scale > 0.0 ? g->init_scale : 1.0;
}

/* ------------------------------------------------------------ O3 / O4 -- */
/* Category per background cell:
 *   0 inactive, far-field negative (inside)     P:189-191, R-5
 *   1 inactive, far-field positive (outside)
 *   2 inner   (not core, some 26-neighbour core) P:507, R-3
 *   3 core    (|f(centre)| < l_c)                P:499-502, R-2
 * near_tie (optional) counts cells with ||f| - l_c| < 1e-12 l_c. */
void or_tag(const or_grid* g, const or_prim* prims, int32_t n_prims, uint8_t* cat,
            int64_t* near_tie) {
    const int64_t nx = g->n[0], ny = g->n[1], nz = g->n[2];
    const int64_t ncell = nx * ny * nz;
    uint8_t* core = (uint8_t*)malloc((size_t)ncell);
    uint8_t* neg = (uint8_t*)malloc((size_t)ncell);
    int64_t ties = 0;
#pragma omp parallel for collapse(2) schedule(static) reduction(+ : ties)
    for (int64_t cz = 0; cz < nz; ++cz)
        for (int64_t cy = 0; cy < ny; ++cy)
            for (int64_t cx = 0; cx < nx; ++cx) {
                double x[3];
                cell_centre(g, cx, cy, cz, x);
                double f = or_sdf(prims, n_prims, x);
                int64_t L = lin_cell(g, cx, cy, cz);
                core[L] = fabs(f) < g->cell;
                neg[L] = f < 0.0;
                if (fabs(fabs(f) - g->cell) < 1e-12 * g->cell) ties++;
            }
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t cz = 0; cz < nz; ++cz)
        for (int64_t cy = 0; cy < ny; ++cy)
            for (int64_t cx = 0; cx < nx; ++cx) {
                int64_t L = lin_cell(g, cx, cy, cz);
                if (core[L]) {
                    cat[L] = 3;
                    continue;
                }
                int inner = 0;
                for (int64_t oz = -1; oz <= 1 && !inner; ++oz)
                    for (int64_t oy = -1; oy <= 1 && !inner; ++oy)
                        for (int64_t ox = -1; ox <= 1 && !inner; ++ox) {
                            int64_t qx = cx + ox, qy = cy + oy, qz = cz + oz;
                            if (qx < 0 || qy < 0 || qz < 0 || qx >= nx || qy >= ny || qz >= nz)
                                continue; /* R-3: clipped to the domain */
                            if (core[lin_cell(g, qx, qy, qz)]) inner = 1;
                        }
                cat[L] = inner ? 2 : (neg[L] ? 0 : 1);
            }
    free(core);
    free(neg);
    if (near_tie) *near_tie = ties;
}

/* O4: ids 2.. in ascending linear cell order (R-1).
 * bg[L] = id (active) or 0/1 (inactive, by sign).  meta_cell / meta_cat have
 * room for ncell + 2 entries (caller sizes them); returns n_pkg incl. 0 and 1.
 * plane_count[cz] (optional) = number of packages in background plane cz. */
int64_t or_compact(const or_grid* g, const uint8_t* cat, uint32_t* bg, uint32_t* meta_cell,
                   uint8_t* meta_cat, int64_t* plane_count) {
    const int64_t nx = g->n[0], ny = g->n[1], nz = g->n[2];
    const int64_t ncell = nx * ny * nz;
    int64_t id = 2;
    meta_cell[0] = 0xFFFFFFFFu;
    meta_cat[0] = 0;
    meta_cell[1] = 0xFFFFFFFFu;
    meta_cat[1] = 1;
    for (int64_t L = 0; L < ncell; ++L) {
        uint8_t c = cat[L];
        if (c >= 2) {
            bg[L] = (uint32_t)id;
            meta_cell[id] = (uint32_t)L;
            meta_cat[id] = c;
            if (plane_count) plane_count[L / (nx * ny)]++;
            id++;
        } else {
            bg[L] = c; /* 0 negative far field, 1 positive far field */
        }
    }
    return id;
}

/* Sign-based far package of a (possibly out-of-domain) background cell
 * (R-6): 0 if f(centre) < 0 else 1.  In-domain cells read bg. */
static inline uint32_t far_pkg_virtual(const or_grid* g, const or_prim* prims, int32_t n_prims,
                                       int64_t cx, int64_t cy, int64_t cz) {
    double x[3];
    if (mesh_mode(n_prims)) { /* R-24: sign of the nearest in-domain cell */
        cx = cx < 0 ? 0 : (cx >= g->n[0] ? g->n[0] - 1 : cx);
        cy = cy < 0 ? 0 : (cy >= g->n[1] ? g->n[1] - 1 : cy);
        cz = cz < 0 ? 0 : (cz >= g->n[2] ? g->n[2] - 1 : cz);
    }
    cell_centre(g, cx, cy, cz, x);
    return or_sdf(prims, n_prims, x) < 0.0 ? 0u : 1u;
}

static inline int in_domain(const or_grid* g, int64_t cx, int64_t cy, int64_t cz) {
    return cx >= 0 && cy >= 0 && cz >= 0 && cx < g->n[0] && cy < g->n[1] && cz < g->n[2];
}

/* O5: nb[id][ox + 3 oy + 9 oz] = package of cell c + o - 1 (P:303-313,
 * R-8); singular rows point to themselves. */
void or_neighbours(const or_grid* g, const or_prim* prims, int32_t n_prims, const uint32_t* bg,
                   const uint32_t* meta_cell, int64_t n_pkg, uint32_t* nb) {
    const int64_t nx = g->n[0], ny = g->n[1];
    for (int s = 0; s < 27; ++s) {
        nb[s] = 0;
        nb[27 + s] = 1;
    }
#pragma omp parallel for schedule(static)
    for (int64_t id = 2; id < n_pkg; ++id) {
        int64_t L = meta_cell[id];
        int64_t cx = L % nx, cy = (L / nx) % ny, cz = L / (nx * ny);
        for (int oz = 0; oz < 3; ++oz)
            for (int oy = 0; oy < 3; ++oy)
                for (int ox = 0; ox < 3; ++ox) {
                    int64_t qx = cx + ox - 1, qy = cy + oy - 1, qz = cz + oz - 1;
                    uint32_t v = in_domain(g, qx, qy, qz)
                                     ? bg[lin_cell(g, qx, qy, qz)]
                                     : far_pkg_virtual(g, prims, n_prims, qx, qy, qz);
                    nb[id * 27 + ox + 3 * oy + 9 * oz] = v;
                }
    }
}

/* -------------------------------------------------------- dense access -- */
/* Dense fine grid: I = ix + M0 (iy + M1 iz), M = 4 N.  A dense value of a
 * point in an inactive cell is the far constant of its sign (the singular
 * package value); a point outside the domain takes the sign of f
 * at its virtual cell centre (R-6). */

typedef struct {
    const or_grid* g;
    const or_prim* prims;
    int32_t n_prims;
    const uint32_t* bg;
    int64_t m[3];  /* fine points of the domain per axis            */
    int64_t o[3];  /* box origin (fine index); 0 for the whole domain */
    int64_t w[3];  /* box extent; m for the whole domain              */
    double far;
} dense_ctx;

static void dense_init(dense_ctx* d, const or_grid* g, const or_prim* prims, int32_t n_prims,
                       const uint32_t* bg) {
    d->g = g;
    d->prims = prims;
    d->n_prims = n_prims;
    d->bg = bg;
    for (int k = 0; k < 3; ++k) {
        d->m[k] = (int64_t)PKG * g->n[k];
        d->o[k] = full_domain(g) ? 0 : g->win_lo[k];
        d->w[k] = full_domain(g) ? d->m[k] : g->win_n[k];
    }
    d->far = or_far(g);
}

/* array index of global fine point I inside the box; in_box tests it */
static inline int in_box(const dense_ctx* d, int64_t ix, int64_t iy, int64_t iz) {
    return ix >= d->o[0] && iy >= d->o[1] && iz >= d->o[2] && ix < d->o[0] + d->w[0] &&
           iy < d->o[1] + d->w[1] && iz < d->o[2] + d->w[2];
}
static inline int64_t box_index(const dense_ctx* d, int64_t ix, int64_t iy, int64_t iz) {
    return (ix - d->o[0]) + d->w[0] * ((iy - d->o[1]) + d->w[1] * (iz - d->o[2]));
}
static inline int64_t box_volume(const dense_ctx* d) { return d->w[0] * d->w[1] * d->w[2]; }

static inline int64_t fdiv4(int64_t i) { return i >= 0 ? i / 4 : -((-i + 3) / 4); }

/* value of a scalar dense field at fine index (ix,iy,iz), possibly outside */
double or_phi_point(const or_grid* g, const or_prim* prims, int32_t n_prims, const uint32_t* bg,
                    int64_t ix, int64_t iy, int64_t iz);

static inline double dense_get(const dense_ctx* d, const double* a, int64_t ix, int64_t iy,
                               int64_t iz) {
    if (in_box(d, ix, iy, iz)) return a[box_index(d, ix, iy, iz)];
    if (ix >= 0 && iy >= 0 && iz >= 0 && ix < d->m[0] && iy < d->m[1] && iz < d->m[2])
        /* window edge (box mode only): the initial phi of the point */
        return or_phi_point(d->g, d->prims, d->n_prims, d->bg, ix, iy, iz);
    uint32_t s = far_pkg_virtual(d->g, d->prims, d->n_prims, fdiv4(ix), fdiv4(iy), fdiv4(iz));
    return s == 0 ? -d->far : d->far;
}

/* is the cell owning fine index I active?  (in-domain only) */
static inline int point_active(const dense_ctx* d, int64_t ix, int64_t iy, int64_t iz) {
    return d->bg[lin_cell(d->g, ix / 4, iy / 4, iz / 4)] >= 2;
}

/* ----------------------------------------------------------------- O6 -- */
/* Initial level set at every data point of every package:
 * phi = init_scale * f(point) for points of active cells, far constant by
 * sign elsewhere (Fig. 2 caption). */
void or_phi_dense(const or_grid* g, const or_prim* prims, int32_t n_prims, const uint32_t* bg,
                  double* phi) {
    dense_ctx d;
    dense_init(&d, g, prims, n_prims, bg);
    const double s = init_scale(g);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t iz = d.o[2]; iz < d.o[2] + d.w[2]; ++iz)
        for (int64_t iy = d.o[1]; iy < d.o[1] + d.w[1]; ++iy)
            for (int64_t ix = d.o[0]; ix < d.o[0] + d.w[0]; ++ix) {
                uint32_t b = bg[lin_cell(g, ix / 4, iy / 4, iz / 4)];
                double v;
                if (b >= 2) {
                    double x[3];
                    point_pos(g, ix, iy, iz, x);
                    v = s * or_sdf(prims, n_prims, x);
                } else {
                    v = b == 0 ? -d.far : d.far;
                }
                phi[box_index(&d, ix, iy, iz)] = v;
            }
}

/* one point of O6 (for sampled checks at sizes where dense is too big) */
double or_phi_point(const or_grid* g, const or_prim* prims, int32_t n_prims, const uint32_t* bg,
                    int64_t ix, int64_t iy, int64_t iz) {
    dense_ctx d;
    dense_init(&d, g, prims, n_prims, bg);
    if (!(ix >= 0 && iy >= 0 && iz >= 0 && ix < d.m[0] && iy < d.m[1] && iz < d.m[2])) {
        uint32_t sgn = far_pkg_virtual(g, prims, n_prims, fdiv4(ix), fdiv4(iy), fdiv4(iz));
        return sgn == 0 ? -d.far : d.far;
    }
    uint32_t b = bg[lin_cell(g, ix / 4, iy / 4, iz / 4)];
    if (b < 2) return b == 0 ? -d.far : d.far;
    double x[3];
    point_pos(g, ix, iy, iz, x);
    return init_scale(g) * or_sdf(prims, n_prims, x);
}

/* ----------------------------------------------------------------- O7 -- */
/* One Jacobi step of upwind Godunov reinitialisation (reading R-12: named by
 * BASELINE.json north_star; the paper implies it):
 *   s   = phi / sqrt(phi^2 + dx^2)
 *   a_k = (phi_I - phi_{I-e_k}) / dx,  b_k = (phi_{I+e_k} - phi_I) / dx
 *   phi > 0: g_k^2 = max(max(a,0)^2, min(b,0)^2)
 *   phi < 0: g_k^2 = max(min(a,0)^2, max(b,0)^2)
 *   phi' = phi - cfl dx s (sqrt(sum g_k^2) - 1);  phi == 0 stays 0.
 * Active points only; inactive points are copied. */
static inline double reinit_point(double c, const double nbm[3], const double nbp[3], double dx,
                                  double cfl) {
    if (c == 0.0) return c;
    double s = c / sqrt(c * c + dx * dx);
    double g2 = 0.0;
    for (int k = 0; k < 3; ++k) {
        double a = (c - nbm[k]) / dx;
        double b = (nbp[k] - c) / dx;
        double u, v;
        if (c > 0.0) {
            u = fmax(a, 0.0);
            v = fmin(b, 0.0);
        } else {
            u = fmin(a, 0.0);
            v = fmax(b, 0.0);
        }
        g2 += fmax(u * u, v * v);
    }
    return c - cfl * dx * s * (sqrt(g2) - 1.0);
}

void or_reinit_dense(const or_grid* g, const or_prim* prims, int32_t n_prims, const uint32_t* bg,
                     const double* phi, double* out, double cfl) {
    dense_ctx d;
    dense_init(&d, g, prims, n_prims, bg);
    const double dx = data_spacing(g);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t iz = d.o[2]; iz < d.o[2] + d.w[2]; ++iz)
        for (int64_t iy = d.o[1]; iy < d.o[1] + d.w[1]; ++iy)
            for (int64_t ix = d.o[0]; ix < d.o[0] + d.w[0]; ++ix) {
                int64_t I = box_index(&d, ix, iy, iz);
                if (!point_active(&d, ix, iy, iz)) {
                    out[I] = phi[I];
                    continue;
                }
                double nbm[3] = {dense_get(&d, phi, ix - 1, iy, iz), dense_get(&d, phi, ix, iy - 1, iz),
                                 dense_get(&d, phi, ix, iy, iz - 1)};
                double nbp[3] = {dense_get(&d, phi, ix + 1, iy, iz), dense_get(&d, phi, ix, iy + 1, iz),
                                 dense_get(&d, phi, ix, iy, iz + 1)};
                out[I] = reinit_point(phi[I], nbm, nbp, dx, cfl);
            }
}

/* first reinit step at one point, inputs from O6 (sampled checks) */
double or_reinit_point_from_init(const or_grid* g, const or_prim* prims, int32_t n_prims,
                                 const uint32_t* bg, int64_t ix, int64_t iy, int64_t iz,
                                 double cfl) {
    double c = or_phi_point(g, prims, n_prims, bg, ix, iy, iz);
    if (bg[lin_cell(g, ix / 4, iy / 4, iz / 4)] < 2) return c;
    double nbm[3] = {or_phi_point(g, prims, n_prims, bg, ix - 1, iy, iz),
                     or_phi_point(g, prims, n_prims, bg, ix, iy - 1, iz),
                     or_phi_point(g, prims, n_prims, bg, ix, iy, iz - 1)};
    double nbp[3] = {or_phi_point(g, prims, n_prims, bg, ix + 1, iy, iz),
                     or_phi_point(g, prims, n_prims, bg, ix, iy + 1, iz),
                     or_phi_point(g, prims, n_prims, bg, ix, iy, iz + 1)};
    return reinit_point(c, nbm, nbp, data_spacing(g), cfl);
}

/* ----------------------------------------------------------------- O8 -- */
/* Gradient by Lst. 5 with regularize(d+, d-) = (d+ + d-)/2 and
 * division by dx (R-13):  grad_k = (phi_{I+e_k} - phi_{I-e_k}) / (2 dx);
 * normal = grad/|grad| (0 if |grad| == 0).  Inactive points: 0 (R-16).
 * grad, normal: three dense planes each (component-major), may be NULL. */
void or_gradient_dense(const or_grid* g, const or_prim* prims, int32_t n_prims,
                       const uint32_t* bg, const double* phi, double* grad, double* normal) {
    dense_ctx d;
    dense_init(&d, g, prims, n_prims, bg);
    const double dx = data_spacing(g);
    const int64_t plane = box_volume(&d);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t iz = d.o[2]; iz < d.o[2] + d.w[2]; ++iz)
        for (int64_t iy = d.o[1]; iy < d.o[1] + d.w[1]; ++iy)
            for (int64_t ix = d.o[0]; ix < d.o[0] + d.w[0]; ++ix) {
                int64_t I = box_index(&d, ix, iy, iz);
                double gv[3] = {0.0, 0.0, 0.0};
                if (point_active(&d, ix, iy, iz)) {
                    gv[0] = (dense_get(&d, phi, ix + 1, iy, iz) - dense_get(&d, phi, ix - 1, iy, iz)) / (2.0 * dx);
                    gv[1] = (dense_get(&d, phi, ix, iy + 1, iz) - dense_get(&d, phi, ix, iy - 1, iz)) / (2.0 * dx);
                    gv[2] = (dense_get(&d, phi, ix, iy, iz + 1) - dense_get(&d, phi, ix, iy, iz - 1)) / (2.0 * dx);
                }
                double mag = sqrt((gv[0] * gv[0] + gv[1] * gv[1]) + gv[2] * gv[2]);
                for (int k = 0; k < 3; ++k) {
                    if (grad) grad[k * plane + I] = gv[k];
                    if (normal) normal[k * plane + I] = mag > 0.0 ? gv[k] / mag : 0.0;
                }
            }
}

/* ----------------------------------------------------------------- O9 -- */
/* Kernel integrals with an SPH smoothing kernel on the sparse grid
 * (kernel and Heaviside are reading R-14):
 *   Wendland C2 (3-D), h = h_ratio dx, support 2h,
 *   w[o]  = W(|o| dx) dx^3,  gw[o] = W'(|o| dx) (-o/|o|) dx^3,
 *   H(u)  = smoothed Heaviside, eps = dx,
 *   K_I = sum_o w[o] H(-phi_{I+o}),  G_I = sum_o gw[o] H(-phi_{I+o}).
 * Inactive points: K = S (negative far field) or 0, G = 0 (R-16). */

#define OR_MAX_TAPS 512

typedef struct {
    int n;
    int o[OR_MAX_TAPS][3];
    double w[OR_MAX_TAPS];
    double gw[OR_MAX_TAPS][3];
} taps_t;

static void make_taps(double h_ratio, double dx, taps_t* t) {
    const double PI = 3.14159265358979323846;
    const double h = h_ratio * dx;
    const double sigma = 21.0 / (16.0 * PI * h * h * h);
    const int R = (int)ceil(2.0 * h_ratio);
    t->n = 0;
    for (int oz = -R; oz <= R; ++oz)
        for (int oy = -R; oy <= R; ++oy)
            for (int ox = -R; ox <= R; ++ox) {
                double len = sqrt((double)(ox * ox + oy * oy + oz * oz));
                double r = len * dx;
                if (!(r < 2.0 * h)) continue;
                double q = r / h;
                double omq = 1.0 - 0.5 * q;
                double W = sigma * omq * omq * omq * omq * (2.0 * q + 1.0);
                double dW = -5.0 * sigma * q * omq * omq * omq / h;
                int k = t->n++;
                t->o[k][0] = ox;
                t->o[k][1] = oy;
                t->o[k][2] = oz;
                t->w[k] = W * dx * dx * dx;
                double o3[3] = {(double)ox, (double)oy, (double)oz};
                for (int a = 0; a < 3; ++a)
                    t->gw[k][a] = len > 0.0 ? dW * (-o3[a] / len) * dx * dx * dx : 0.0;
            }
}

/* tap table export: returns count; o (n x 3 int), w (n), gw (n x 3) */
int32_t or_kernel_taps(double h_ratio, double dx, int32_t* o, double* w, double* gw) {
    taps_t t;
    make_taps(h_ratio, dx, &t);
    for (int k = 0; k < t.n; ++k) {
        for (int a = 0; a < 3; ++a) {
            if (o) o[3 * k + a] = t.o[k][a];
            if (gw) gw[3 * k + a] = t.gw[k][a];
        }
        if (w) w[k] = t.w[k];
    }
    return t.n;
}

double or_heaviside(double u, double eps) {
    const double PI = 3.14159265358979323846;
    if (u < -eps) return 0.0;
    if (u > eps) return 1.0;
    return 0.5 * (1.0 + u / eps + sin(PI * u / eps) / PI);
}

void or_kernel_dense(const or_grid* g, const or_prim* prims, int32_t n_prims, const uint32_t* bg,
                     const double* phi, double h_ratio, double* K, double* G) {
    dense_ctx d;
    dense_init(&d, g, prims, n_prims, bg);
    const double dx = data_spacing(g);
    const int64_t plane = box_volume(&d);
    taps_t* t = (taps_t*)malloc(sizeof(taps_t));
    make_taps(h_ratio, dx, t);
    double S = 0.0;
    for (int k = 0; k < t->n; ++k) S += t->w[k];
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
    for (int64_t iz = d.o[2]; iz < d.o[2] + d.w[2]; ++iz)
        for (int64_t iy = d.o[1]; iy < d.o[1] + d.w[1]; ++iy)
            for (int64_t ix = d.o[0]; ix < d.o[0] + d.w[0]; ++ix) {
                int64_t I = box_index(&d, ix, iy, iz);
                double k_acc = 0.0, gacc[3] = {0.0, 0.0, 0.0};
                uint32_t b = bg[lin_cell(g, ix / 4, iy / 4, iz / 4)];
                if (b >= 2) {
                    for (int k = 0; k < t->n; ++k) {
                        double v = dense_get(&d, phi, ix + t->o[k][0], iy + t->o[k][1], iz + t->o[k][2]);
                        double H = or_heaviside(-v, dx);
                        k_acc += t->w[k] * H;
                        for (int a = 0; a < 3; ++a) gacc[a] += t->gw[k][a] * H;
                    }
                } else if (b == 0) {
                    k_acc = S;
                }
                if (K) K[I] = k_acc;
                if (G)
                    for (int a = 0; a < 3; ++a) G[a * plane + I] = gacc[a];
            }
    free(t);
}

/* ---------------------------------------------------------- Table 1 --- */
/* The paper's access-pattern benchmark (Table 1):
 *   "sequential": a minor change to every active value -- phi + value;
 *   "stencil": the seven-point Laplacian at every active data point,
 *              (sum of the 6 axis neighbours - 6 phi) / dx^2.
 * Inactive points: the input value (sequential) / 0 (stencil). */
void or_table1_dense(const or_grid* g, const or_prim* prims, int32_t n_prims, const uint32_t* bg,
                     const double* phi, int32_t op, double value, double* out) {
    dense_ctx d;
    dense_init(&d, g, prims, n_prims, bg);
    const double dx = data_spacing(g);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t iz = d.o[2]; iz < d.o[2] + d.w[2]; ++iz)
        for (int64_t iy = d.o[1]; iy < d.o[1] + d.w[1]; ++iy)
            for (int64_t ix = d.o[0]; ix < d.o[0] + d.w[0]; ++ix) {
                int64_t I = box_index(&d, ix, iy, iz);
                int act = point_active(&d, ix, iy, iz);
                if (op == 0) {
                    out[I] = act ? phi[I] + value : phi[I];
                } else if (!act) {
                    out[I] = 0.0;
                } else {
                    double s6 = ((dense_get(&d, phi, ix - 1, iy, iz) + dense_get(&d, phi, ix + 1, iy, iz)) +
                                 (dense_get(&d, phi, ix, iy - 1, iz) + dense_get(&d, phi, ix, iy + 1, iz))) +
                                (dense_get(&d, phi, ix, iy, iz - 1) + dense_get(&d, phi, ix, iy, iz + 1));
                    out[I] = (s6 - 6.0 * phi[I]) / (dx * dx);
                }
            }
}

/* ---------------------------------------------------------------- O10 -- */
/* Grid-particle coupling: containing-cell lookup through the
 * background table, far constant for inactive cells, otherwise trilinear
 * interpolation over the 8 data points around the position (R-15).  Index
 * arithmetic in double: division and floor only.  Out-of-domain or NaN
 * positions return (+far, 0) and are counted.
 *   pos: n x 3 doubles; grad3: dense 3-plane gradient or NULL;
 *   out_phi: n; out_grad: n x 3 or NULL.  Returns the OOB count. */
int64_t or_probe(const or_grid* g, const or_prim* prims, int32_t n_prims, const uint32_t* bg,
                 const double* phi, const double* grad3, int64_t n, const double* pos,
                 double* out_phi, double* out_grad) {
    dense_ctx d;
    dense_init(&d, g, prims, n_prims, bg);
    const double dx = data_spacing(g);
    const int64_t plane = box_volume(&d);
    int64_t oob = 0;
#pragma omp parallel for schedule(static) reduction(+ : oob)
    for (int64_t p = 0; p < n; ++p) {
        const double* x = pos + 3 * p;
        double rphi = d.far, rg[3] = {0.0, 0.0, 0.0};
        int ok = 1;
        int64_t c[3];
        for (int k = 0; k < 3; ++k) {
            double upper = g->lower[k] + (double)g->n[k] * g->cell;
            if (!(x[k] >= g->lower[k] && x[k] < upper)) {
                ok = 0;
                break;
            }
            c[k] = (int64_t)floor((x[k] - g->lower[k]) / g->cell);
            if (c[k] > g->n[k] - 1) c[k] = g->n[k] - 1;
        }
        if (!ok) {
            oob++;
        } else {
            uint32_t b = bg[lin_cell(g, c[0], c[1], c[2])];
            if (b < 2) {
                rphi = b == 0 ? -d.far : d.far;
            } else {
                int64_t a[3];
                double t[3];
                for (int k = 0; k < 3; ++k) {
                    double u = (x[k] - g->lower[k]) / dx - 0.5;
                    double fl = floor(u);
                    a[k] = (int64_t)fl;
                    t[k] = u - fl;
                }
                rphi = 0.0;
                for (int bidx = 0; bidx < 8; ++bidx) {
                    int b0 = bidx & 1, b1 = (bidx >> 1) & 1, b2 = (bidx >> 2) & 1;
                    double w = ((b0 ? t[0] : 1.0 - t[0]) * (b1 ? t[1] : 1.0 - t[1])) *
                               (b2 ? t[2] : 1.0 - t[2]);
                    int64_t ix = a[0] + b0, iy = a[1] + b1, iz = a[2] + b2;
                    rphi += w * dense_get(&d, phi, ix, iy, iz);
                    if (grad3) {
                        if (in_box(&d, ix, iy, iz)) {
                            int64_t I = box_index(&d, ix, iy, iz);
                            for (int k = 0; k < 3; ++k) rg[k] += w * grad3[k * plane + I];
                        }
                    }
                }
            }
        }
        out_phi[p] = rphi;
        if (out_grad)
            for (int k = 0; k < 3; ++k) out_grad[3 * p + k] = rg[k];
    }
    return oob;
}

/* ------------------------------------------------------------ NEXT-2 --- */
/* SPH particle relaxation against the level set (force law and
 * bounding: reading R-21 = SPEC S:535-543 with the kernel-gradient integral G
 * as the surface force).  Per step, for every particle i inside the domain:
 *   S_i = sum_{j != i, |x_i - x_j| < 2h} V W'(|r|) r / |r|,   r = x_i - x_j,
 *   a_i = -2 (S_i - G(x_i)),   d_i = step dp^2 a_i, |d_i| clamped to max_d dp,
 *   x_i' = x_i + d_i;  then with (phi, grad phi) interpolated at x_i':
 *   if phi > -off dp: x_i' -= (phi + off dp) grad phi / |grad phi|.
 * All pairs are enumerated (brute force, small n).  Fields are the dense
 * phi, grad (3 planes) and G (3 planes) of the grid. */
static void interp_dense(const dense_ctx* d, const double* f3, int ncomp, int64_t plane,
                         const double x[3], double* out) {
    const or_grid* g = d->g;
    const double dx = data_spacing(g);
    int64_t a[3];
    double t[3];
    for (int k = 0; k < 3; ++k) {
        double u = (x[k] - g->lower[k]) / dx - 0.5;
        double fl = floor(u);
        a[k] = (int64_t)fl;
        t[k] = u - fl;
    }
    for (int c = 0; c < ncomp; ++c) out[c] = 0.0;
    for (int b = 0; b < 8; ++b) {
        int b0 = b & 1, b1 = (b >> 1) & 1, b2 = (b >> 2) & 1;
        double w = ((b0 ? t[0] : 1.0 - t[0]) * (b1 ? t[1] : 1.0 - t[1])) * (b2 ? t[2] : 1.0 - t[2]);
        int64_t ix = a[0] + b0, iy = a[1] + b1, iz = a[2] + b2;
        int in = in_box(d, ix, iy, iz);
        for (int c = 0; c < ncomp; ++c) {
            double v;
            if (ncomp == 1 && c == 0) v = dense_get(d, f3, ix, iy, iz);
            else v = in ? f3[c * plane + box_index(d, ix, iy, iz)] : 0.0;
            out[c] += w * v;
        }
    }
}

static int in_domain_pos(const or_grid* g, const double x[3], int64_t c[3]) {
    for (int k = 0; k < 3; ++k) {
        double upper = g->lower[k] + (double)g->n[k] * g->cell;
        if (!(x[k] >= g->lower[k] && x[k] < upper)) return 0;
        c[k] = (int64_t)floor((x[k] - g->lower[k]) / g->cell);
        if (c[k] > g->n[k] - 1) c[k] = g->n[k] - 1;
    }
    return 1;
}

void or_relax(const or_grid* g, const or_prim* prims, int32_t n_prims, const uint32_t* bg,
              const double* phi, const double* grad3, const double* G3, int64_t n, double* pos,
              double dp, double h_ratio, double step, double max_disp, double off, int32_t steps) {
    if (!full_domain(g)) return; /* whole-domain operation */
    dense_ctx d;
    dense_init(&d, g, prims, n_prims, bg);
    const int64_t plane = box_volume(&d);
    const double PI = 3.14159265358979323846;
    const double h = h_ratio * dp;
    const double sigma = 21.0 / (16.0 * PI * h * h * h);
    const double V = dp * dp * dp;
    double* moved = (double*)malloc(sizeof(double) * 3 * (size_t)n);
    for (int it = 0; it < steps; ++it) {
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            const double* xi = pos + 3 * i;
            int64_t c[3];
            for (int k = 0; k < 3; ++k) moved[3 * i + k] = xi[k];
            if (!in_domain_pos(g, xi, c)) continue;
            double S[3] = {0.0, 0.0, 0.0};
            for (int64_t j = 0; j < n; ++j) {
                if (j == i) continue;
                int64_t cj[3];
                if (!in_domain_pos(g, pos + 3 * j, cj)) continue;
                double r[3] = {xi[0] - pos[3 * j], xi[1] - pos[3 * j + 1], xi[2] - pos[3 * j + 2]};
                double rr = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
                if (!(rr > 0.0 && rr < 2.0 * h)) continue;
                double q = rr / h, a = 1.0 - 0.5 * q;
                double dW = -5.0 * sigma * q * a * a * a / h; /* W'(r) */
                for (int k = 0; k < 3; ++k) S[k] += V * dW * r[k] / rr;
            }
            double Gi[3] = {0.0, 0.0, 0.0};
            if (bg[lin_cell(g, c[0], c[1], c[2])] >= 2) interp_dense(&d, G3, 3, plane, xi, Gi);
            double dv[3], len = 0.0;
            for (int k = 0; k < 3; ++k) {
                dv[k] = step * dp * dp * (-2.0 * (S[k] - Gi[k]));
                len += dv[k] * dv[k];
            }
            len = sqrt(len);
            double mx = max_disp * dp;
            double sc = len > mx ? mx / len : 1.0;
            for (int k = 0; k < 3; ++k) moved[3 * i + k] = xi[k] + dv[k] * sc;
        }
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            double* x = moved + 3 * i;
            int64_t c[3];
            if (in_domain_pos(g, x, c)) {
                uint32_t b = bg[lin_cell(g, c[0], c[1], c[2])];
                double ph, gv[3] = {0.0, 0.0, 0.0};
                if (b >= 2) {
                    interp_dense(&d, phi, 1, plane, x, &ph);
                    interp_dense(&d, grad3, 3, plane, x, gv);
                } else {
                    ph = b == 0 ? -d.far : d.far;
                }
                if (ph > -off * dp) {
                    double m = sqrt(gv[0] * gv[0] + gv[1] * gv[1] + gv[2] * gv[2]);
                    if (m > 0.0)
                        for (int k = 0; k < 3; ++k) x[k] -= (ph + off * dp) * gv[k] / m;
                }
            }
            for (int k = 0; k < 3; ++k) pos[3 * i + k] = x[k];
        }
    }
    free(moved);
}

/* ------------------------------------------------------- layout helper -- */
/* ---------------------------------------------------------- NEXT-3 -- */
/* Sign-consistency correction ("only the sign of level set for
 * those data points very close to the surface is directly used, those at
 * other locations are obtained by a two-step diffusion process from the near
 * interface to the entire domain.  The first coarse step is on the mesh cells
 * and the second refined one is on the data packages."), reading R-22:
 *
 * Rule (both steps): synchronous sweeps; an unsigned site with at least one
 * signed face neighbour takes the sign held by more of its signed face
 * neighbours, a tie leaves it unsigned in that sweep; a step ends at the
 * first sweep that signs nothing (or after max_sweeps > 0 sweeps).
 *
 * Coarse step: sites = background cells, face neighbours inside the domain.
 * Core cells (cat 3) are signed by f at their centre, all others unsigned.
 * Then every inactive cell's table entry becomes 0 (negative) / 1, and every
 * singular neighbour-table entry of an in-domain cell is re-read from the
 * table.  cell_neg (optional, ncell bytes) receives the final cell signs
 * (cells never reached keep the sign of f at their centre).
 *
 * Refined step: sites = data points of active cells on the dense grid.
 * Points with |phi| < tau keep their sign; all other active points start
 * unsigned.  A neighbour point in an inactive in-domain cell is signed by the
 * table (0 negative); outside the domain by f at the virtual cell centre
 * (R-6).  Finally phi = -|phi| or +|phi| at every signed active point.
 * sweeps[0..1] = number of sweeps of each step that signed something. */
void or_sign_correct(const or_grid* g, const or_prim* prims, int32_t n_prims, const uint8_t* cat,
                     uint32_t* bg, const uint32_t* meta_cell, int64_t n_pkg, uint32_t* nb,
                     uint8_t* cell_neg, double* phi, double tau, int32_t max_sweeps,
                     int32_t* sweeps) {
    if (!full_domain(g)) return; /* whole-domain operation */
    const int64_t nx = g->n[0], ny = g->n[1], nz = g->n[2];
    const int64_t ncell = nx * ny * nz;
    static const int off[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};

    /* coarse step on the cells */
    uint8_t* known = (uint8_t*)malloc((size_t)ncell);
    uint8_t* neg = (uint8_t*)malloc((size_t)ncell);
    uint8_t* known2 = (uint8_t*)malloc((size_t)ncell);
    uint8_t* neg2 = (uint8_t*)malloc((size_t)ncell);
    for (int64_t cz = 0; cz < nz; ++cz)
        for (int64_t cy = 0; cy < ny; ++cy)
            for (int64_t cx = 0; cx < nx; ++cx) {
                int64_t L = lin_cell(g, cx, cy, cz);
                double x[3];
                cell_centre(g, cx, cy, cz, x);
                known[L] = cat[L] == 3;
                neg[L] = or_sdf(prims, n_prims, x) < 0.0;
            }
    int32_t sw = 0;
    for (;;) {
        if (max_sweeps > 0 && sw >= max_sweeps) break;
        int64_t signed_now = 0;
        for (int64_t cz = 0; cz < nz; ++cz)
            for (int64_t cy = 0; cy < ny; ++cy)
                for (int64_t cx = 0; cx < nx; ++cx) {
                    int64_t L = lin_cell(g, cx, cy, cz);
                    known2[L] = known[L];
                    neg2[L] = neg[L];
                    if (known[L]) continue;
                    int vn = 0, vp = 0;
                    for (int d = 0; d < 6; ++d) {
                        int64_t qx = cx + off[d][0], qy = cy + off[d][1], qz = cz + off[d][2];
                        if (!in_domain(g, qx, qy, qz)) continue;
                        int64_t Q = lin_cell(g, qx, qy, qz);
                        if (!known[Q]) continue;
                        if (neg[Q]) vn++;
                        else vp++;
                    }
                    if (vn != vp) {
                        known2[L] = 1;
                        neg2[L] = vn > vp;
                        signed_now++;
                    }
                }
        if (signed_now == 0) break;
        sw++;
        memcpy(known, known2, (size_t)ncell);
        memcpy(neg, neg2, (size_t)ncell);
    }
    sweeps[0] = sw;
    for (int64_t L = 0; L < ncell; ++L)
        if (bg[L] < 2) bg[L] = neg[L] ? 0u : 1u;
    for (int64_t id = 2; id < n_pkg; ++id) {
        int64_t L = meta_cell[id];
        int64_t cx = L % nx, cy = (L / nx) % ny, cz = L / (nx * ny);
        for (int s = 0; s < 27; ++s) {
            int64_t qx = cx + s % 3 - 1, qy = cy + (s / 3) % 3 - 1, qz = cz + s / 9 - 1;
            if (nb[id * 27 + s] < 2 && in_domain(g, qx, qy, qz))
                nb[id * 27 + s] = bg[lin_cell(g, qx, qy, qz)];
        }
    }
    if (cell_neg) memcpy(cell_neg, neg, (size_t)ncell);
    free(known);
    free(neg);
    free(known2);
    free(neg2);

    /* refined step on the data points of active cells */
    const int64_t mx = PKG * nx, my = PKG * ny, mz = PKG * nz;
    const int64_t np = mx * my * mz;
    known = (uint8_t*)calloc((size_t)np, 1);
    neg = (uint8_t*)calloc((size_t)np, 1);
    known2 = (uint8_t*)calloc((size_t)np, 1);
    neg2 = (uint8_t*)calloc((size_t)np, 1);
#define PIDX(ix, iy, iz) ((ix) + mx * ((iy) + my * (iz)))
#define ACTIVE(ix, iy, iz) (bg[lin_cell(g, (ix) / PKG, (iy) / PKG, (iz) / PKG)] >= 2)
    for (int64_t iz = 0; iz < mz; ++iz)
        for (int64_t iy = 0; iy < my; ++iy)
            for (int64_t ix = 0; ix < mx; ++ix) {
                if (!ACTIVE(ix, iy, iz)) continue;
                double v = phi[PIDX(ix, iy, iz)];
                known[PIDX(ix, iy, iz)] = fabs(v) < tau;
                neg[PIDX(ix, iy, iz)] = v < 0.0;
            }
    sw = 0;
    for (;;) {
        if (max_sweeps > 0 && sw >= max_sweeps) break;
        int64_t signed_now = 0;
        memcpy(known2, known, (size_t)np);
        memcpy(neg2, neg, (size_t)np);
        for (int64_t iz = 0; iz < mz; ++iz)
            for (int64_t iy = 0; iy < my; ++iy)
                for (int64_t ix = 0; ix < mx; ++ix) {
                    int64_t I = PIDX(ix, iy, iz);
                    if (!ACTIVE(ix, iy, iz) || known[I]) continue;
                    int vn = 0, vp = 0;
                    for (int d = 0; d < 6; ++d) {
                        int64_t jx = ix + off[d][0], jy = iy + off[d][1], jz = iz + off[d][2];
                        int kn, ng;
                        if (jx < 0 || jy < 0 || jz < 0 || jx >= mx || jy >= my || jz >= mz) {
                            kn = 1;
                            ng = far_pkg_virtual(g, prims, n_prims, fdiv4(jx), fdiv4(jy),
                                                 fdiv4(jz)) == 0;
                        } else if (!ACTIVE(jx, jy, jz)) {
                            kn = 1;
                            ng = bg[lin_cell(g, jx / PKG, jy / PKG, jz / PKG)] == 0;
                        } else {
                            kn = known[PIDX(jx, jy, jz)];
                            ng = neg[PIDX(jx, jy, jz)];
                        }
                        if (!kn) continue;
                        if (ng) vn++;
                        else vp++;
                    }
                    if (vn != vp) {
                        known2[I] = 1;
                        neg2[I] = vn > vp;
                        signed_now++;
                    }
                }
        if (signed_now == 0) break;
        sw++;
        memcpy(known, known2, (size_t)np);
        memcpy(neg, neg2, (size_t)np);
    }
    sweeps[1] = sw;
    for (int64_t iz = 0; iz < mz; ++iz)
        for (int64_t iy = 0; iy < my; ++iy)
            for (int64_t ix = 0; ix < mx; ++ix) {
                int64_t I = PIDX(ix, iy, iz);
                if (ACTIVE(ix, iy, iz)) {
                    if (known[I]) phi[I] = neg[I] ? -fabs(phi[I]) : fabs(phi[I]);
                } else { /* inactive point: far constant of the corrected cell sign */
                    phi[I] = bg[lin_cell(g, ix / PKG, iy / PKG, iz / PKG)] == 0 ? -fabs(phi[I])
                                                                               : fabs(phi[I]);
                }
            }
#undef PIDX
#undef ACTIVE
    free(known);
    free(neg);
    free(known2);
    free(neg2);
}

/* Small-feature cleaning ("we reimplemented the level-set
 * cleaning algorithms (only on the finest layer) in Ref. [yu2023level]"; the
 * criterion is reading R-23, the stand-in of SPEC S:476-484).  Per round:
 *   1. K = kernel integral of phi (or_kernel_dense, h = h_ratio dx);
 *      S = sum of the kernel weights;
 *   2. every active data point inside the body within dx of the surface
 *      (-dx < phi < 0) with K < threshold S is set to phi = +dx (points
 *      outside are already carved; raising them would change nothing of the
 *      geometry); modified[r] = their number; none -> stop;
 *   3. reinit_iters reinitialisation steps (or_reinit_dense).
 * At most max_rounds rounds; returns the number of rounds that raised
 * points.  phi is the dense field (in/out). */
int32_t or_clean(const or_grid* g, const or_prim* prims, int32_t n_prims, const uint32_t* bg,
                 double* phi, double h_ratio, double threshold, int32_t reinit_iters, double cfl,
                 int32_t max_rounds, int64_t* modified) {
    if (!full_domain(g)) return -1; /* whole-domain operation */
    dense_ctx d;
    dense_init(&d, g, prims, n_prims, bg);
    const double dx = data_spacing(g);
    const int64_t np = d.m[0] * d.m[1] * d.m[2];
    taps_t* t = (taps_t*)malloc(sizeof(taps_t));
    make_taps(h_ratio, dx, t);
    double S = 0.0;
    for (int k = 0; k < t->n; ++k) S += t->w[k];
    free(t);
    double* K = (double*)malloc(sizeof(double) * (size_t)np);
    double* tmp = (double*)malloc(sizeof(double) * (size_t)np);
    int32_t done = 0;
    for (int32_t r = 0; r < max_rounds; ++r) modified[r] = 0;
    for (int32_t r = 0; r < max_rounds; ++r) {
        or_kernel_dense(g, prims, n_prims, bg, phi, h_ratio, K, NULL);
        int64_t cnt = 0;
        for (int64_t iz = 0; iz < d.m[2]; ++iz)
            for (int64_t iy = 0; iy < d.m[1]; ++iy)
                for (int64_t ix = 0; ix < d.m[0]; ++ix) {
                    int64_t I = ix + d.m[0] * (iy + d.m[1] * iz);
                    if (!point_active(&d, ix, iy, iz)) continue;
                    if (phi[I] < 0.0 && fabs(phi[I]) < dx && K[I] < threshold * S) {
                        phi[I] = dx;
                        cnt++;
                    }
                }
        modified[r] = cnt;
        if (cnt == 0) break;
        done++;
        for (int32_t it = 0; it < reinit_iters; ++it) {
            or_reinit_dense(g, prims, n_prims, bg, phi, tmp, cfl);
            memcpy(phi, tmp, sizeof(double) * (size_t)np);
        }
    }
    free(K);
    free(tmp);
    return done;
}

/* Gather a dense scalar plane into package-major order using the oracle's
 * own meta table: out[id][i + 4 j + 16 k] = dense[4c + (i,j,k)] (R-9
 * canonical order).  Singular packages take `far_neg` / `far_pos`. */
void or_gather_packages(const or_grid* g, const double* dense, const uint32_t* meta_cell,
                        int64_t n_pkg, double far_neg, double far_pos, double* out) {
    if (!full_domain(g)) return; /* whole-domain operation */
    const int64_t nx = g->n[0], ny = g->n[1];
    const int64_t m0 = (int64_t)PKG * g->n[0], m1 = (int64_t)PKG * g->n[1];
    for (int d = 0; d < 64; ++d) {
        out[d] = far_neg;
        out[64 + d] = far_pos;
    }
#pragma omp parallel for schedule(static)
    for (int64_t id = 2; id < n_pkg; ++id) {
        int64_t L = meta_cell[id];
        int64_t cx = L % nx, cy = (L / nx) % ny, cz = L / (nx * ny);
        for (int k = 0; k < 4; ++k)
            for (int j = 0; j < 4; ++j)
                for (int i = 0; i < 4; ++i)
                    out[id * 64 + i + 4 * j + 16 * k] =
                        dense[(4 * cx + i) + m0 * ((4 * cy + j) + m1 * (4 * cz + k))];
    }
}

void or_set_threads(int32_t n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int32_t or_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
