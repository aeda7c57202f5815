// sweep_common.cuh -- device helpers shared by the sweep kernels (sweep.cu,
// sweep_aa.cu) and the auxiliary kernels (aux_kernels.cu).
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace lbm {

__device__ __forceinline__ int64_t cell_index(const Geom &g, int x, int y, int z)
{
    return ((int64_t)(z + 1) * g.py + (y + 1)) * (int64_t)g.px + (x + g.xo);
}

template <typename real>
__device__ __forceinline__ real ld_stream(const real *p)
{
    return __ldg(p);
}

template <typename real, int STCS>
__device__ __forceinline__ void st_stream(real *p, real v)
{
    if (STCS)
        __stcs(p, v);  // evict-first: dst is not re-read in this sweep
    else
        *p = v;
}

// two cells per thread along x: the 2-vector type of the storage precision
template <typename real> struct Vec2;
template <> struct Vec2<float> { using T = float2; };
template <> struct Vec2<double> { using T = double2; };

}  // namespace lbm
