// Conservative per-(splat, tile) cull shared by K2 (optional bit-31 flag)
// and K3/K4 (batch staging).
#pragma once

#include "ivr_common.cuh"

namespace ivr {

// Float32 lower bound of the splat's exponent over the pixel rectangle
// [px0,px1] x [py0,py1] (value at the clamped edge minimiser minus a rigorous
// rounding slack); the pair is culled iff the bound exceeds hi, i.e. the
// reference's float64 alpha is < 1/255 at every pixel of the tile.
__device__ __forceinline__ bool tile_cull32(const float4 r0, const float4 r1, int px0, int px1,
                                            int py0, int py1) {
    const float hi = r0.w;
    if (!(hi < 1e30f)) return false;
    const float ha = r1.x, b = r1.y, hc = r1.z;  // a/2, b, c/2
    const float det4 = 4.0f * ha * hc;
    if (!(ha > 0.0f && hc > 0.0f && det4 - b * b > 1e-4f * det4)) return false;
    // float subtraction of an exactly representable integer: one rounding of
    // the exact difference, as before in double
    const float ex0 = (float)px0 - r0.x, ex1 = (float)px1 - r0.x;
    const float ey0 = (float)py0 - r0.y, ey1 = (float)py1 - r0.y;
    if (ex0 <= 0.0f && ex1 >= 0.0f && ey0 <= 0.0f && ey1 >= 0.0f) return false;
    // approximate reciprocals only move the candidate minimiser on each edge
    // by <= |e| 2^-22 (e within the rectangle): a second-order change of the
    // quadratic, far below the slack below
    float i2a, i2c;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(i2a) : "f"(2.0f * ha));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(i2c) : "f"(2.0f * hc));
    float best = 3.0e38f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float dx, dy;
        if (k < 2) {
            dx = k ? ex1 : ex0;
            dy = fminf(fmaxf(-b * dx * i2c, ey0), ey1);
        } else {
            dy = (k & 1) ? ey1 : ey0;
            dx = fminf(fmaxf(-b * dy * i2a, ex0), ex1);
        }
        const float t1 = ha * dx * dx, t2 = b * dx * dy, t3 = hc * dy * dy;
        const float s = t1 + t2 + t3;
        const float lo = s - 2e-6f * (t1 + fabsf(t2) + t3) - 1e-4f;
        best = fminf(best, lo);
    }
    return best > hi;
}

}  // namespace ivr
