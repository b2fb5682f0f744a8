// sg_godunov.cuh -- the reinitialisation step (K5, O7 / reading R-12) at one
// data point and along one x-row of four points, shared by the single-sweep
// kernel (sg_stencil.cu k_sweep) and the two-sweep tile kernel
// (sg_tsweep.cu k_tsweep): both call the same inline code, so the two paths
// give bit-identical values (compiled with the same flags, -ftz=true).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sg {

template <class T>
struct StC {
    T inv_dx, dx2, cdx, inv_2dx;
};

// O7 (reading R-12): one Jacobi Godunov step at one data point, in the
// sign-folded form.  With sigma = sign(phi) the two upwind cases
//   phi > 0: g_k^2 = max(max(a,0)^2, min(b,0)^2)
//   phi < 0: g_k^2 = max(min(a,0)^2, max(b,0)^2),
// a = (phi - phi_{-e})/dx, b = (phi_{+e} - phi)/dx, are one expression:
//   g_k = max(sigma (phi - phi_{-e}), sigma (phi - phi_{+e}), 0) / dx.
// phi = 0 gives s = 0 and leaves the point unchanged, as the definition does.
// fp32: approximate rsqrt/sqrt (MUFU, ~2 ulp) -- well inside 1e-5 dx.
__device__ __forceinline__ float gd_axis(float ap, uint32_t sg, float m, float q) {
    const float sm = __uint_as_float(__float_as_uint(m) ^ sg);
    const float sq = __uint_as_float(__float_as_uint(q) ^ sg);
    return fmaxf(fmaxf(ap - sm, ap - sq), 0.f);
}
__device__ __forceinline__ float godunov(float p, float xm, float xp, float ym, float yp, float zm,
                                         float zp, const StC<float>& c) {
    const uint32_t sg = __float_as_uint(p) & 0x80000000u;
    const float ap = fabsf(p);
    const float wx = gd_axis(ap, sg, xm, xp);
    const float wy = gd_axis(ap, sg, ym, yp);
    const float wz = gd_axis(ap, sg, zm, zp);
    const float G = fmaf(wx, wx, fmaf(wy, wy, wz * wz));
    const float g = G > 0.f ? G * rsqrtf(G) : 0.f;  // |grad phi| dx
    const float s = p * rsqrtf(fmaf(p, p, c.dx2));
    return fmaf(-c.cdx * s, fmaf(g, c.inv_dx, -1.f), p);
}
__device__ __forceinline__ double gd_axis(double ap, double sg, double m, double q) {
    return fmax(fmax(ap - sg * m, ap - sg * q), 0.0);
}
__device__ __forceinline__ double godunov(double p, double xm, double xp, double ym, double yp,
                                          double zm, double zp, const StC<double>& c) {
    const double sg = p < 0.0 ? -1.0 : 1.0;
    const double ap = fabs(p);
    const double wx = gd_axis(ap, sg, xm, xp) * c.inv_dx;
    const double wy = gd_axis(ap, sg, ym, yp) * c.inv_dx;
    const double wz = gd_axis(ap, sg, zm, zp) * c.inv_dx;
    const double s = p / sqrt(p * p + c.dx2);
    return p - c.cdx * s * (sqrt(wx * wx + wy * wy + wz * wz) - 1.0);
}

// fp32 row form of the same sign-folded step, written for the Blackwell
// paired-FP32 pipe: with a_i = -sign(p_i)/dx and b_i = |p_i|/dx the two upwind
// differences of one axis are (a m + b, a q + b) / 1 and
// w = max(., ., 0) is one 3-input FMNMX.  The y / z neighbours of points
// i, i+1 sit in aligned register pairs of their float4 rows, so they (and
// |grad|^2, the sign factor and the update) go through FFMA2 / FMUL2; the x
// neighbours are not pair-aligned and stay scalar.  sqrt / rsqrt: MUFU
// (~2 ulp), inside the 1e-5 dx tolerance.  Same formula as godunov() above:
// out = p + cdx s (1 - |grad phi|), s = p / sqrt(p^2 + dx^2).
__device__ __forceinline__ float max3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void godunov_row(const float (&p)[4], float xm, float xp,
                                            const float (&ym)[4], const float (&yp)[4],
                                            const float (&zm)[4], const float (&zp)[4],
                                            const StC<float>& c, float (&o)[4]) {
    float a[4], b[4], wx[4];
    // a = -sign(p) / dx as one bit operation: the sign bit of p flips
    // -1/dx.  (p = -0 gets +1/dx where the select gave -1/dx; the step
    // returns p unchanged for p = +-0 either way: s = 0.)
    const uint32_t nid = __float_as_uint(-c.inv_dx);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a[i] = __uint_as_float((__float_as_uint(p[i]) & 0x80000000u) ^ nid);
        b[i] = fabsf(p[i]) * c.inv_dx;
        const float m = i > 0 ? p[i - 1] : xm, q = i < 3 ? p[i + 1] : xp;
        wx[i] = max3f(fmaf(a[i], m, b[i]), fmaf(a[i], q, b[i]), 0.f);
    }
    const float2 dx2 = make_float2(c.dx2, c.dx2), cdx = make_float2(c.cdx, c.cdx);
#pragma unroll
    for (int h = 0; h < 4; h += 2) {
        const float2 A = make_float2(a[h], a[h + 1]), B = make_float2(b[h], b[h + 1]);
        const float2 tym = __ffma2_rn(A, make_float2(ym[h], ym[h + 1]), B);
        const float2 typ = __ffma2_rn(A, make_float2(yp[h], yp[h + 1]), B);
        const float2 tzm = __ffma2_rn(A, make_float2(zm[h], zm[h + 1]), B);
        const float2 tzp = __ffma2_rn(A, make_float2(zp[h], zp[h + 1]), B);
        const float2 WX = make_float2(wx[h], wx[h + 1]);
        const float2 WY = make_float2(max3f(tym.x, typ.x, 0.f), max3f(tym.y, typ.y, 0.f));
        const float2 WZ = make_float2(max3f(tzm.x, tzp.x, 0.f), max3f(tzm.y, tzp.y, 0.f));
        const float2 G = __ffma2_rn(WX, WX, __ffma2_rn(WY, WY, __fmul2_rn(WZ, WZ)));
        const float2 t = make_float2(1.f - sqrt_approx(G.x), 1.f - sqrt_approx(G.y));
        const float2 P = make_float2(p[h], p[h + 1]);
        const float2 r2 = __ffma2_rn(P, P, dx2);
        const float2 cs = __fmul2_rn(__fmul2_rn(P, cdx), make_float2(rsqrtf(r2.x), rsqrtf(r2.y)));
        const float2 out = __ffma2_rn(cs, t, P);
        o[h] = out.x;
        o[h + 1] = out.y;
    }
}

}  // namespace sg
