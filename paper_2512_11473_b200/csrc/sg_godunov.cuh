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
    T ncfl;  // -cfl (the fp32 row form works in units of dx)
};

// O7 (reading R-12): one Jacobi Godunov step at one data point, in the
// sign-folded form.  With sigma = sign(phi) the two upwind cases
//   phi > 0: g_k^2 = max(max(a,0)^2, min(b,0)^2)
//   phi < 0: g_k^2 = max(min(a,0)^2, max(b,0)^2),
// a = (phi - phi_{-e})/dx, b = (phi_{+e} - phi)/dx, are one expression:
//   g_k = max(sigma (phi - phi_{-e}), sigma (phi - phi_{+e}), 0) / dx.
// phi = 0 gives s = 0 and leaves the point unchanged, as the definition does.
// The fp64 form below is the definition term by term (the C1 parity config);
// the fp32 path is the paired row form godunov_row further down.
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
// paired-FP32 pipe: per axis w = max(a m + |p|, a q + |p|, 0) with
// a = -sign(p) (in units of dx), one 3-input FMNMX.  The y / z neighbours of
// points i, i+1 sit in aligned register pairs of their float4 rows, so they
// (and |grad|^2, the sign factor and the update) go through FFMA2 / FMUL2;
// the x neighbours are not pair-aligned and stay scalar.  sqrt / rsqrt: MUFU
// (~2 ulp), inside the 1e-5 dx tolerance.  The formula of godunov() above:
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
    // In units of dx: with a = -sign(p) (one bit operation: the sign bit of
    // p flips -1; p = -0 gets +1, and the step returns p = +-0 unchanged
    // either way, s = 0) each upwind difference is a m + |p| -- one FMA with
    // the absolute value as a free operand modifier -- and
    // g = sqrt(sum of squares) = |grad phi| dx.  The update
    //   p + s cfl dx (1 - |grad phi|) = p + (p rsqrt(p^2 + dx^2)) (cdx - cfl g)
    // takes one FMA for (cdx - cfl g) and one for the result.
    float a[4], wx[4];
    const uint32_t m1 = __float_as_uint(-1.f);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a[i] = __uint_as_float((__float_as_uint(p[i]) & 0x80000000u) ^ m1);
        const float m = i > 0 ? p[i - 1] : xm, q = i < 3 ? p[i + 1] : xp;
        wx[i] = max3f(fmaf(a[i], m, fabsf(p[i])), fmaf(a[i], q, fabsf(p[i])), 0.f);
    }
    const float2 dx2 = make_float2(c.dx2, c.dx2), cdx = make_float2(c.cdx, c.cdx);
    const float2 ncfl = make_float2(c.ncfl, c.ncfl);
#pragma unroll
    for (int h = 0; h < 4; h += 2) {
        const float2 A = make_float2(a[h], a[h + 1]);
        const float2 B = make_float2(fabsf(p[h]), fabsf(p[h + 1]));
        const float2 tym = __ffma2_rn(A, make_float2(ym[h], ym[h + 1]), B);
        const float2 typ = __ffma2_rn(A, make_float2(yp[h], yp[h + 1]), B);
        const float2 tzm = __ffma2_rn(A, make_float2(zm[h], zm[h + 1]), B);
        const float2 tzp = __ffma2_rn(A, make_float2(zp[h], zp[h + 1]), B);
        const float2 WX = make_float2(wx[h], wx[h + 1]);
        const float2 WY = make_float2(max3f(tym.x, typ.x, 0.f), max3f(tym.y, typ.y, 0.f));
        const float2 WZ = make_float2(max3f(tzm.x, tzp.x, 0.f), max3f(tzm.y, tzp.y, 0.f));
        const float2 G = __ffma2_rn(WX, WX, __ffma2_rn(WY, WY, __fmul2_rn(WZ, WZ)));
        const float2 g = make_float2(sqrt_approx(G.x), sqrt_approx(G.y));
        const float2 t = __ffma2_rn(g, ncfl, cdx);  // cdx - cfl g
        const float2 P = make_float2(p[h], p[h + 1]);
        const float2 r2 = __ffma2_rn(P, P, dx2);
        const float2 sgn = __fmul2_rn(P, make_float2(rsqrtf(r2.x), rsqrtf(r2.y)));
        const float2 out = __ffma2_rn(sgn, t, P);
        o[h] = out.x;
        o[h + 1] = out.y;
    }
}

}  // namespace sg
