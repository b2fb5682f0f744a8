// sdf.cuh -- fp64 analytic signed distance on the device.
//
// Only included by translation units compiled with -fmad=false: every
// operation below is a separately rounded IEEE double operation in the order
// written (no FMA contraction, IEEE sqrt/div), which makes the tagging
// decision |f(centre)| < l_c (reading R-2) reproducible bit for bit
// against any other IEEE evaluation with the same operation order.
#pragma once

#include "sg_internal.cuh"

namespace sg {

__device__ __forceinline__ double sd_len3(double ex, double ey, double ez) {
    return sqrt((ex * ex + ey * ey) + ez * ez);
}

// sqrt(a*a + b*b) for a, b >= 0 with the IEEE result: in binary floating
// point sqrt(fl(x*x)) == |x| when x*x neither overflows nor underflows, so a
// zero term (exactly representable: 0*0 = +0) lets the square root go
__device__ __forceinline__ double hyp2(double a, double b) {
    if (b == 0.0 && (a == 0.0 || (a > 1e-150 && a < 1e150))) return a;
    if (a == 0.0 && b > 1e-150 && b < 1e150) return b;
    return sqrt(a * a + b * b);
}

__device__ __forceinline__ double sd_prim(int kind, const double* p, double x, double y,
                                          double z) {
    switch (kind) {
    case SG_SPHERE:
        return sd_len3(x - p[0], y - p[1], z - p[2]) - p[3];
    case SG_SHELL: {
        const double rm = 0.5 * (p[3] + p[4]);
        const double hw = 0.5 * (p[4] - p[3]);
        return fabs(sd_len3(x - p[0], y - p[1], z - p[2]) - rm) - hw;
    }
    case SG_BOX: {
        const double qx = fabs(x - p[0]) - p[3];
        const double qy = fabs(y - p[1]) - p[4];
        const double qz = fabs(z - p[2]) - p[5];
        const double mx = fmax(qx, 0.0), my = fmax(qy, 0.0), mz = fmax(qz, 0.0);
        return sqrt((mx * mx + my * my) + mz * mz) + fmin(fmax(qx, fmax(qy, qz)), 0.0);
    }
    case SG_TORUS_X: {
        const double ex = x - p[0], ey = y - p[1], ez = z - p[2];
        const double t = sqrt(ey * ey + ez * ez) - p[3];
        return sqrt(t * t + ex * ex) - p[4];
    }
    case SG_TORUS_Y: {
        const double ex = x - p[0], ey = y - p[1], ez = z - p[2];
        const double t = sqrt(ex * ex + ez * ez) - p[3];
        return sqrt(t * t + ey * ey) - p[4];
    }
    case SG_TORUS_Z: {
        const double ex = x - p[0], ey = y - p[1], ez = z - p[2];
        const double t = sqrt(ex * ex + ey * ey) - p[3];
        return sqrt(t * t + ez * ez) - p[4];
    }
    case SG_TRIPRISM_Z: {
        // exact 2-D triangle distance: clamped point-segment distance per
        // edge; inside iff strictly left of every (ccw) edge
        double best = 0.0;
        bool inside = true;
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const int e1 = (e + 1) % 3;
            const double ux = p[2 * e1] - p[2 * e], uy = p[2 * e1 + 1] - p[2 * e + 1];
            const double wx = x - p[2 * e], wy = y - p[2 * e + 1];
            // t = clamp((w.u) / (u.u), 0, 1); the quotient is only needed
            // strictly inside (0, 1): w.u <= 0 gives t = 0 and w.u >= u.u
            // gives t = 1 for the correctly rounded quotient too, so the
            // skipped division changes no bit of the result
            const double wu = wx * ux + wy * uy, uu = ux * ux + uy * uy;
            const double t = wu <= 0.0 ? 0.0 : (wu >= uu ? 1.0 : wu / uu);
            const double hx = wx - ux * t, hy = wy - uy * t;
            const double d2 = hx * hx + hy * hy;
            best = (e == 0) ? d2 : fmin(best, d2);
            inside = inside && (ux * wy - uy * wx > 0.0);
        }
        const double dxy = inside ? -sqrt(best) : sqrt(best);
        const double zc = 0.5 * (p[6] + p[7]);
        const double hl = 0.5 * (p[7] - p[6]);
        const double qz = fabs(z - zc) - hl;
        const double a = fmax(dxy, 0.0), b = fmax(qz, 0.0);
        return fmin(fmax(dxy, qz), 0.0) + hyp2(a, b);
    }
    default:
        return __longlong_as_double(0x7ff8000000000000ULL);  // NaN
    }
}

// SG_LEAK post-operation (include/sg.h): f <- -f strictly inside any leak
// ball where |f| >= margin
__device__ __forceinline__ double sd_leak(const Geom& g, double x, double y, double z,
                                          double f) {
    bool flip = false;
    for (int i = 0; i < g.n_leak; ++i) {
        const double* l = g.leak[i];
        const double ex = x - l[0], ey = y - l[1], ez = z - l[2];
        flip = flip || (((ex * ex + ey * ey) + ez * ez < l[3] * l[3]) && fabs(f) >= l[4]);
    }
    return flip ? -f : f;
}

// union of the primitives = pointwise min, in order
__device__ __forceinline__ double sd_eval(const Geom& g, double x, double y, double z) {
    double f = sd_prim(g.kind[0], g.p[0], x, y, z);
    for (int i = 1; i < g.n; ++i) f = fmin(f, sd_prim(g.kind[i], g.p[i], x, y, z));
    return g.n_leak ? sd_leak(g, x, y, z, f) : f;
}

// f at NZ points sharing (x, y): the terms of each primitive that depend on
// x and y only are evaluated once per column; each f[k] is the operation
// sequence of sd_prim / sd_eval above (common-subexpression reuse only, so
// the result is bit-identical to NZ separate sd_eval calls).
template <int NZ>
__device__ __forceinline__ void sd_prim_col(int kind, const double* p, double x, double y,
                                            const double (&z)[NZ], double (&f)[NZ]) {
    switch (kind) {
    case SG_SPHERE:
    case SG_SHELL: {
        const double ex = x - p[0], ey = y - p[1];
        const double exy = ex * ex + ey * ey;
        const double rm = 0.5 * (p[3] + p[4]);
        const double hw = 0.5 * (p[4] - p[3]);
#pragma unroll
        for (int k = 0; k < NZ; ++k) {
            const double ez = z[k] - p[2];
            const double d = sqrt(exy + ez * ez);
            f[k] = kind == SG_SPHERE ? d - p[3] : fabs(d - rm) - hw;
        }
        return;
    }
    case SG_BOX: {
        const double qx = fabs(x - p[0]) - p[3];
        const double qy = fabs(y - p[1]) - p[4];
        const double mx = fmax(qx, 0.0), my = fmax(qy, 0.0);
        const double mxy = mx * mx + my * my;
#pragma unroll
        for (int k = 0; k < NZ; ++k) {
            const double qz = fabs(z[k] - p[2]) - p[5];
            const double mz = fmax(qz, 0.0);
            f[k] = sqrt(mxy + mz * mz) + fmin(fmax(qx, fmax(qy, qz)), 0.0);
        }
        return;
    }
    case SG_TORUS_Z: {
        const double ex = x - p[0], ey = y - p[1];
        const double t = sqrt(ex * ex + ey * ey) - p[3];
#pragma unroll
        for (int k = 0; k < NZ; ++k) {
            const double ez = z[k] - p[2];
            f[k] = sqrt(t * t + ez * ez) - p[4];
        }
        return;
    }
    case SG_TRIPRISM_Z: {
        double best = 0.0;
        bool inside = true;
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const int e1 = (e + 1) % 3;
            const double ux = p[2 * e1] - p[2 * e], uy = p[2 * e1 + 1] - p[2 * e + 1];
            const double wx = x - p[2 * e], wy = y - p[2 * e + 1];
            // t = clamp((w.u) / (u.u), 0, 1); the quotient is only needed
            // strictly inside (0, 1): w.u <= 0 gives t = 0 and w.u >= u.u
            // gives t = 1 for the correctly rounded quotient too, so the
            // skipped division changes no bit of the result
            const double wu = wx * ux + wy * uy, uu = ux * ux + uy * uy;
            const double t = wu <= 0.0 ? 0.0 : (wu >= uu ? 1.0 : wu / uu);
            const double hx = wx - ux * t, hy = wy - uy * t;
            const double d2 = hx * hx + hy * hy;
            best = (e == 0) ? d2 : fmin(best, d2);
            inside = inside && (ux * wy - uy * wx > 0.0);
        }
        const double dxy = inside ? -sqrt(best) : sqrt(best);
        const double zc = 0.5 * (p[6] + p[7]);
        const double hl = 0.5 * (p[7] - p[6]);
        const double a = fmax(dxy, 0.0);
#pragma unroll
        for (int k = 0; k < NZ; ++k) {
            const double qz = fabs(z[k] - zc) - hl;
            const double b = fmax(qz, 0.0);
            f[k] = fmin(fmax(dxy, qz), 0.0) + hyp2(a, b);
        }
        return;
    }
    default:  // torus x / y: no (x, y)-only term worth sharing
#pragma unroll
        for (int k = 0; k < NZ; ++k) f[k] = sd_prim(kind, p, x, y, z[k]);
        return;
    }
}

template <int NZ>
__device__ __forceinline__ void sd_eval_col(const Geom& g, double x, double y,
                                            const double (&z)[NZ], double (&f)[NZ]) {
    sd_prim_col<NZ>(g.kind[0], g.p[0], x, y, z, f);
    for (int i = 1; i < g.n; ++i) {
        double fi[NZ];
        sd_prim_col<NZ>(g.kind[i], g.p[i], x, y, z, fi);
#pragma unroll
        for (int k = 0; k < NZ; ++k) f[k] = fmin(f[k], fi[k]);
    }
    if (g.n_leak) {
#pragma unroll
        for (int k = 0; k < NZ; ++k) f[k] = sd_leak(g, x, y, z[k], f[k]);
    }
}

// the same min over the primitives selected by `mask` (bit i = primitive i);
// callers only drop primitives that provably exceed the minimum
template <int NZ>
__device__ __forceinline__ void sd_eval_col_mask(const Geom& g, uint32_t mask, double x, double y,
                                                 const double (&z)[NZ], double (&f)[NZ]) {
    bool first = true;
    // the selected primitives in ascending order (set bits only)
    for (uint32_t mm = mask; mm; mm &= mm - 1u) {
        const int i = __ffs(mm) - 1;
        double fi[NZ];
        sd_prim_col<NZ>(g.kind[i], g.p[i], x, y, z, fi);
#pragma unroll
        for (int k = 0; k < NZ; ++k) f[k] = first ? fi[k] : fmin(f[k], fi[k]);
        first = false;
    }
    if (g.n_leak) {
#pragma unroll
        for (int k = 0; k < NZ; ++k) f[k] = sd_leak(g, x, y, z[k], f[k]);
    }
}

// The same per-point values along a y-column (x, z shared): the torus about
// the y axis shares sqrt(ex^2 + ez^2) - R between the points, the box its x / z
// terms, the sphere / shell ex^2 and ez^2; the association of every sum is
// that of sd_prim, so each f[k] is bit-identical to sd_prim at (x, y[k], z).
template <int NY>
__device__ __forceinline__ void sd_prim_coly(int kind, const double* p, double x, double z,
                                             const double (&y)[NY], double (&f)[NY]) {
    switch (kind) {
    case SG_SPHERE:
    case SG_SHELL: {
        const double ex = x - p[0], ez = z - p[2];
        const double ex2 = ex * ex, ez2 = ez * ez;
        const double rm = 0.5 * (p[3] + p[4]);
        const double hw = 0.5 * (p[4] - p[3]);
#pragma unroll
        for (int k = 0; k < NY; ++k) {
            const double ey = y[k] - p[1];
            const double d = sqrt((ex2 + ey * ey) + ez2);
            f[k] = kind == SG_SPHERE ? d - p[3] : fabs(d - rm) - hw;
        }
        return;
    }
    case SG_BOX: {
        const double qx = fabs(x - p[0]) - p[3];
        const double qz = fabs(z - p[2]) - p[5];
        const double mx = fmax(qx, 0.0), mz = fmax(qz, 0.0);
        const double mx2 = mx * mx, mz2 = mz * mz;
#pragma unroll
        for (int k = 0; k < NY; ++k) {
            const double qy = fabs(y[k] - p[1]) - p[4];
            const double my = fmax(qy, 0.0);
            f[k] = sqrt((mx2 + my * my) + mz2) + fmin(fmax(qx, fmax(qy, qz)), 0.0);
        }
        return;
    }
    case SG_TORUS_Y: {
        const double ex = x - p[0], ez = z - p[2];
        const double t = sqrt(ex * ex + ez * ez) - p[3];
        const double t2 = t * t;
#pragma unroll
        for (int k = 0; k < NY; ++k) {
            const double ey = y[k] - p[1];
            f[k] = sqrt(t2 + ey * ey) - p[4];
        }
        return;
    }
    default:
#pragma unroll
        for (int k = 0; k < NY; ++k) f[k] = sd_prim(kind, p, x, y[k], z);
        return;
    }
}

template <int NY>
__device__ __forceinline__ void sd_eval_coly_mask(const Geom& g, uint32_t mask, double x, double z,
                                                  const double (&y)[NY], double (&f)[NY]) {
    bool first = true;
    for (uint32_t mm = mask; mm; mm &= mm - 1u) {
        const int i = __ffs(mm) - 1;
        double fi[NY];
        sd_prim_coly<NY>(g.kind[i], g.p[i], x, z, y, fi);
#pragma unroll
        for (int k = 0; k < NY; ++k) f[k] = first ? fi[k] : fmin(f[k], fi[k]);
        first = false;
    }
    if (g.n_leak) {
#pragma unroll
        for (int k = 0; k < NY; ++k) f[k] = sd_leak(g, x, y[k], z, f[k]);
    }
}

}  // namespace sg
