// dog_eval.cuh -- evaluation workload on the filter's readouts (PAPER section VIII):
// per-cell Mahalanobis distance of the velocity estimate from v = 0 (Eq. 88 `eq:mahadist`), static /
// dynamic classification counts per threshold and the sums behind the cluster statistics
// (Eqs. 85-86).  Arithmetic in fp64 with the operation order of DESIGN.md A-33 (bit-identical m).
#pragma once
#include <cstdint>
#include "dog_common.cuh"

namespace dog {

constexpr int kEvalMaxThr = 64;
struct EvalThr { float v[kEvalMaxThr]; };

// valid_mode: 0 = valid[] (u8, NULL: mean or cov nonzero), 1 = the filter's moments-valid bitmask.
__global__ __launch_bounds__(256) void k_eval_cells(const float2* __restrict__ mean, const float* __restrict__ cov,
                                                    const uint8_t* __restrict__ valid, const uint32_t* __restrict__ vbits,
                                                    const uint8_t* __restrict__ labels, const uint8_t* __restrict__ mask,
                                                    EvalThr thr, int n_thr, float* __restrict__ m_out,
                                                    unsigned long long* __restrict__ counts, double* __restrict__ sums,
                                                    uint32_t C)
{
    __shared__ uint32_t s_cnt[kEvalMaxThr][4];
    __shared__ double s_sum[5];
    for (int i = threadIdx.x; i < kEvalMaxThr * 4; i += blockDim.x) (&s_cnt[0][0])[i] = 0u;
    if (threadIdx.x < 5) s_sum[threadIdx.x] = 0.0;
    __syncthreads();
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
        const float2 mv = mean[c];
        const double vx = mv.x, vy = mv.y;
        double pxx = cov[3 * (size_t)c], pyy = cov[3 * (size_t)c + 1];
        const double pxy = cov[3 * (size_t)c + 2];
        bool ok;
        if (vbits) ok = (vbits[c >> 5] >> (c & 31)) & 1u;
        else if (valid) ok = valid[c] != 0;
        else ok = vx != 0.0 || vy != 0.0 || pxx != 0.0 || pyy != 0.0 || pxy != 0.0;
        double m = 0.0;
        if (ok) {
            double det = __dsub_rn(__dmul_rn(pxx, pyy), __dmul_rn(pxy, pxy));
            if (det <= 1e-12) {                              // regularised (A-33)
                pxx = __dadd_rn(pxx, 1e-6);
                pyy = __dadd_rn(pyy, 1e-6);
                det = __dsub_rn(__dmul_rn(pxx, pyy), __dmul_rn(pxy, pxy));
            }
            const double a = __dmul_rn(__dmul_rn(vx, vx), pyy);
            const double b = __dmul_rn(__dmul_rn(__dmul_rn(2.0, vx), vy), pxy);
            const double e = __dmul_rn(__dmul_rn(vy, vy), pxx);
            m = __ddiv_rn(__dadd_rn(__dsub_rn(a, b), e), det);
        }
        const float mf = __double2float_rn(m);
        if (m_out) m_out[c] = mf;
        if (labels) {
            const uint8_t l = labels[c];
            if (l == 1 || l == 2)
                for (int t = 0; t < n_thr; ++t) {
                    const bool dyn_det = mf >= thr.v[t];
                    atomicAdd(&s_cnt[t][l == 2 ? (dyn_det ? 0 : 1) : (dyn_det ? 2 : 3)], 1u);
                }
        }
        if (mask && ok && mask[c]) {
            atomicAdd(&s_sum[0], 1.0);
            atomicAdd(&s_sum[1], vx);
            atomicAdd(&s_sum[2], __dadd_rn((double)cov[3 * (size_t)c], __dmul_rn(vx, vx)));
            atomicAdd(&s_sum[3], vy);
            atomicAdd(&s_sum[4], __dadd_rn((double)cov[3 * (size_t)c + 1], __dmul_rn(vy, vy)));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_thr * 4; i += blockDim.x)
        if ((&s_cnt[0][0])[i]) atomicAdd(&counts[i], (unsigned long long)(&s_cnt[0][0])[i]);
    if (threadIdx.x < 5 && s_sum[threadIdx.x] != 0.0) atomicAdd(&sums[threadIdx.x], s_sum[threadIdx.x]);
}

}  // namespace dog
