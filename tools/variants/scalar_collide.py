# fp32 pairs collided with the scalar collide_bgk (no packed f32x2)
PATCHES = [("collide.cuh", """__device__ __forceinline__ void collide_pair(float (&p0)[Q], float (&p1)[Q], float omega)
{
    float2 p[Q];""", """__device__ __forceinline__ void collide_pair(float (&p0)[Q], float (&p1)[Q], float omega)
{
    collide_bgk<float>(p0, omega);
    collide_bgk<float>(p1, omega);
}
__device__ __forceinline__ void collide_pair_unused(float (&p0)[Q], float (&p1)[Q], float omega)
{
    float2 p[Q];""")]
