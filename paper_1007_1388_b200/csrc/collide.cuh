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

}  // namespace lbm
