// dog_ego.cuh -- ego-motion compensation ("the ego movement of the test
// vehicle can be compensated in the grid map"; SPEC S:171-179 ego_scroll, A-32): the grid
// content and the particles move by a whole number of cells between cycles.
#pragma once
#include <cstdint>
#include "dog_common.cuh"

namespace dog {

// Particles (whole-grid context): one f32 addition per coordinate; leaving the grid -> sentinel (A-19);
// sentinel particles stay where they are.
__global__ __launch_bounds__(256) void k_ego_particles(float4* __restrict__ st, uint32_t nu, int32_t sx, int32_t sy,
                                                       int32_t W, int32_t H)
{
    const float fx = (float)sx, fy = (float)sy, Wf = (float)W, Hf = (float)H;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += gridDim.x * blockDim.x) {
        const float4 X = st[i];
        if (X.x == kSentinelPos && X.y == kSentinelPos) continue;
        const float xn = __fadd_rn(X.x, fx), yn = __fadd_rn(X.y, fy);
        const bool inside = xn >= 0.0f && xn < Wf && yn >= 0.0f && yn < Hf;
        st[i] = inside ? make_float4(xn, yn, X.z, X.w) : make_float4(kSentinelPos, kSentinelPos, 0.0f, 0.0f);
    }
}

// Grid: the content of cell (r, c) moves to (r + sy, c + sx); cells scrolled in are vacuous (m_F = 0).
__global__ __launch_bounds__(256) void k_ego_grid(const float* __restrict__ m_free, float* __restrict__ out,
                                                  int32_t sx, int32_t sy, int32_t W, int32_t H)
{
    const uint32_t C = (uint32_t)W * (uint32_t)H;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
        const int32_t r = (int32_t)(c / (uint32_t)W), col = (int32_t)(c % (uint32_t)W);
        const int32_t r0 = r - sy, c0 = col - sx;
        out[c] = (r0 >= 0 && r0 < H && c0 >= 0 && c0 < W) ? m_free[(uint32_t)r0 * (uint32_t)W + (uint32_t)c0] : 0.0f;
    }
}

}  // namespace dog
