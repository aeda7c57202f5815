// collide.cuh -- the BGK collision shared by every sweep kernel, so that all
// sweep variants (SIMT, TMA; whole patch, shell, interior) produce bitwise
// identical results.
//
// eq:lbm with eq:feq, centred PDFs, rho0 = 1 (R4):
//   drho = sum p_i,  u = sum e_i p_i / rho0  (R7),
//   p_i <- p_i - omega (p_i - w_i [drho + 3 e_i.u + 4.5 (e_i.u)^2 - 1.5 u.u])  (R8)
// written as (1 - omega) p_i + omega w_i (...) and evaluated pairwise for
// opposite directions (e.u changes sign, the even part of f^eq is shared).
// The sums are balanced trees (short dependency chains for the latency-bound
// TMA consumer warps); the rounding differs from the oracle's left-to-right
// sums only at the 1e-16 level (R14).
#pragma once

#include "lbm_internal.h"

namespace lbm {

template <typename real>
__device__ __forceinline__ void collide_bgk(real (&p)[Q], real omega)
{
    const real a12 = p[1] + p[2], a34 = p[3] + p[4], a56 = p[5] + p[6];
    const real a78 = p[7] + p[8], a910 = p[9] + p[10], a1112 = p[11] + p[12];
    const real a1314 = p[13] + p[14], a1516 = p[15] + p[16], a1718 = p[17] + p[18];
    const real drho = ((p[0] + a12) + (a34 + a56)) + (((a78 + a910) + (a1112 + a1314)) + (a1516 + a1718));
    const real d12 = p[1] - p[2], d34 = p[3] - p[4], d56 = p[5] - p[6];
    const real d78 = p[7] - p[8], d910 = p[9] - p[10], d1112 = p[11] - p[12];
    const real d1314 = p[13] - p[14], d1516 = p[15] - p[16], d1718 = p[17] - p[18];
    const real ux = (d12 + (d78 + d910)) + (d1112 + d1314);
    const real uy = (d34 + (d78 - d910)) + (d1516 + d1718);
    const real uz = (d56 + (d1112 - d1314)) + (d1516 - d1718);
    const real c0 = real(1) - omega;
    const real base = drho - real(1.5) * ((ux * ux + uy * uy) + uz * uz);
    const real w0 = omega * real(1.0 / 3.0);
    const real w1 = omega * real(1.0 / 18.0);
    const real w2 = omega * real(1.0 / 36.0);
    p[0] = c0 * p[0] + w0 * base;
#define LBM_PAIR(a, b, eu, w)                       \
    {                                               \
        const real e_ = (eu);                       \
        const real t_ = base + real(4.5) * e_ * e_; \
        const real s_ = real(3) * e_;               \
        p[a] = c0 * p[a] + (w) * (t_ + s_);         \
        p[b] = c0 * p[b] + (w) * (t_ - s_);         \
    }
    LBM_PAIR(1, 2, ux, w1)
    LBM_PAIR(3, 4, uy, w1)
    LBM_PAIR(5, 6, uz, w1)
    LBM_PAIR(7, 8, ux + uy, w2)
    LBM_PAIR(9, 10, ux - uy, w2)
    LBM_PAIR(11, 12, ux + uz, w2)
    LBM_PAIR(13, 14, ux - uz, w2)
    LBM_PAIR(15, 16, uy + uz, w2)
    LBM_PAIR(17, 18, uy - uz, w2)
#undef LBM_PAIR
}

// The two cells of a thread (x2 sweeps).  fp64: collide_bgk twice.  fp32: the
// same update with packed f32x2 arithmetic (sm_100a FADD2 / FMUL2 / FFMA2),
// the two cells in the two halves of a register pair -- half the FP
// instructions, which shortens the compute phase between a warp's loads and
// stores (the fp32 sweep spends twice the arithmetic per byte of fp64).  Every
// operation is explicit (the fused multiply-adds are written out), so the
// result is one fixed rounding sequence for every kernel that uses it.
__device__ __forceinline__ unsigned long long f2u(float2 a) { return *reinterpret_cast<unsigned long long *>(&a); }
__device__ __forceinline__ float2 u2f(unsigned long long a) { return *reinterpret_cast<float2 *>(&a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b)
{
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b)
{
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b)
{
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c)
{
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(d);
}

__device__ __forceinline__ void collide_pair(double (&p0)[Q], double (&p1)[Q], double omega)
{
    collide_bgk<double>(p0, omega);
    collide_bgk<double>(p1, omega);
}

__device__ __forceinline__ void collide_pair(float (&p0)[Q], float (&p1)[Q], float omega)
{
    float2 p[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) p[i] = make_float2(p0[i], p1[i]);
    const float2 a12 = add2(p[1], p[2]), a34 = add2(p[3], p[4]), a56 = add2(p[5], p[6]);
    const float2 a78 = add2(p[7], p[8]), a910 = add2(p[9], p[10]), a1112 = add2(p[11], p[12]);
    const float2 a1314 = add2(p[13], p[14]), a1516 = add2(p[15], p[16]), a1718 = add2(p[17], p[18]);
    const float2 drho = add2(add2(add2(p[0], a12), add2(a34, a56)),
                             add2(add2(add2(a78, a910), add2(a1112, a1314)), add2(a1516, a1718)));
    const float2 d12 = sub2(p[1], p[2]), d34 = sub2(p[3], p[4]), d56 = sub2(p[5], p[6]);
    const float2 d78 = sub2(p[7], p[8]), d910 = sub2(p[9], p[10]), d1112 = sub2(p[11], p[12]);
    const float2 d1314 = sub2(p[13], p[14]), d1516 = sub2(p[15], p[16]), d1718 = sub2(p[17], p[18]);
    const float2 ux = add2(add2(d12, add2(d78, d910)), add2(d1112, d1314));
    const float2 uy = add2(add2(d34, sub2(d78, d910)), add2(d1516, d1718));
    const float2 uz = add2(add2(d56, sub2(d1112, d1314)), sub2(d1516, d1718));
    const float2 usq = fma2(uz, uz, fma2(uy, uy, mul2(ux, ux)));
    const float2 base = fma2(make_float2(-1.5f, -1.5f), usq, drho);
    const float2 c0 = make_float2(1.0f - omega, 1.0f - omega);
    const float w0s = omega * (1.0f / 3.0f), w1s = omega * (1.0f / 18.0f), w2s = omega * (1.0f / 36.0f);
    const float2 w0 = make_float2(w0s, w0s), w1 = make_float2(w1s, w1s), w2 = make_float2(w2s, w2s);
    const float2 k45 = make_float2(4.5f, 4.5f), k3 = make_float2(3.0f, 3.0f);
    p[0] = fma2(c0, p[0], mul2(w0, base));
#define LBM_PAIR2(a, b, eu, w)                            \
    {                                                     \
        const float2 e_ = (eu);                           \
        const float2 t_ = fma2(mul2(k45, e_), e_, base);  \
        const float2 s_ = mul2(k3, e_);                   \
        p[a] = fma2(c0, p[a], mul2(w, add2(t_, s_)));     \
        p[b] = fma2(c0, p[b], mul2(w, sub2(t_, s_)));     \
    }
    LBM_PAIR2(1, 2, ux, w1)
    LBM_PAIR2(3, 4, uy, w1)
    LBM_PAIR2(5, 6, uz, w1)
    LBM_PAIR2(7, 8, add2(ux, uy), w2)
    LBM_PAIR2(9, 10, sub2(ux, uy), w2)
    LBM_PAIR2(11, 12, add2(ux, uz), w2)
    LBM_PAIR2(13, 14, sub2(ux, uz), w2)
    LBM_PAIR2(15, 16, add2(uy, uz), w2)
    LBM_PAIR2(17, 18, sub2(uy, uz), w2)
#undef LBM_PAIR2
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        p0[i] = p[i].x;
        p1[i] = p[i].y;
    }
}

}  // namespace lbm
