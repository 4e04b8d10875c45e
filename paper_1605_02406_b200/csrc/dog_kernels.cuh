// dog_kernels.cuh -- the sm_100a kernels of one DS-PHD/MIB cycle (section VII).
//
// Stage map (paper -> kernel):
//   Alg. 1 predict              -> k_predict      (+ cell counts, radix histograms)
//   Alg. 2 sort + assign        -> dog_sort.cuh   (tile-local stable sort + per-cell run lists)
//   Alg. 3 occupancy predict/update           -> k_cells        (dog_cells.cuh)
//   Alg. 4 persistent update    -> implicit: weights are uniform per cell (A-8, A-23)
//   Alg. 5 slots + Alg. 7 joint CDF           -> k_list_scan    (dog_cells.cuh)
//   Alg. 5 births, Alg. 6 moments, Alg. 7     -> k_resample_tiles + k_births (dog_resample.cuh)
//
// Every floating-point expression on the parity path uses explicit round-to-nearest intrinsics in
// the operation order of DESIGN.md section 3 so the CPU oracle reproduces it bit for bit (A-21).
#pragma once
#include <cstdint>
#include "dog_common.cuh"
#include "dog_rng.cuh"

namespace dog {


// ------------------------------------------------------------------------------------------------
// Alg. 1 -- particle prediction.  One block advances one 4096-particle sort tile (state and predicted
// state are (x, y, vx, vy) float4 per particle: one 16-byte load and store each) and writes the new
// cell keys.
// ------------------------------------------------------------------------------------------------
constexpr int kPredThreads = 256;
constexpr int kSortTile = 4096;     // particles per sort tile (= one k_predict block)

__global__ __launch_bounds__(kPredThreads) void k_predict(const float4* __restrict__ st, float4* __restrict__ pst,
                                                          uint32_t* __restrict__ keys, DevScalars* __restrict__ sc,
                                                          FilterConst fc, StepArgs a)
{
    const float w_bar = sc->w_bar;
    const float w_pred = __fmul_rn(fc.p_s, w_bar);      // Eq. 39 (A-3): one scalar
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->w_pred = w_pred;
    const float Wf = (float)fc.W, Hf = (float)fc.H;
    const uint32_t i0 = blockIdx.x * kSortTile;

#pragma unroll 2
    for (int it = 0; it < kSortTile / kPredThreads; ++it) {
        const uint32_t i = i0 + it * kPredThreads + threadIdx.x;
        if (i >= fc.nu) break;
        const float4 S = st[i];
        const Philox4 r = draw(fc.seed, i, a.k, STAGE_PREDICT);
        float n0, n1, n2, n3;
        box_muller(r.r0, r.r1, n0, n1);
        box_muller(r.r2, r.r3, n2, n3);
        // p' = p + T v + xi_p with the OLD velocity (Eq. 14, A-2); v' = v + xi_v
        const float xn = __fmaf_rn(a.s_p, n0, __fmaf_rn(S.z, a.Tc, S.x));
        const float yn = __fmaf_rn(a.s_p, n1, __fmaf_rn(S.w, a.Tc, S.y));
        const float vxn = __fmaf_rn(a.s_v, n2, S.z);
        const float vyn = __fmaf_rn(a.s_v, n3, S.w);
        const bool inside = (xn >= 0.0f) && (xn < Wf) && (yn >= 0.0f) && (yn < Hf);
        keys[i] = inside ? (uint32_t)__float2int_rz(yn) * (uint32_t)fc.W + (uint32_t)__float2int_rz(xn)
                         : fc.C;                                    // A-4, A-5
        pst[i] = make_float4(xn, yn, vxn, vyn);
    }
}

}  // namespace dog
