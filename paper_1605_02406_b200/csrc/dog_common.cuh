// dog_common.cuh -- shared device helpers and the per-step device scalar block.
#pragma once
#include <cstdint>

namespace dog {

typedef unsigned __int128 u128;

// Device-resident scalars of the filter (written and read by kernels, so a cycle needs no host sync).
struct DevScalars {
    float    w_bar;      // uniform particle weight of the current state S_k (Eq. 57)
    float    w_pred;     // p_S * w_bar of the cycle in flight (Eq. 39)
    uint32_t U;          // systematic-resampling offset of the cycle (A-24)
    uint32_t meas_bad;   // invalid measurement cells seen (sticky until reported)
    uint64_t W;          // total fixed-point joint weight (A-23)
    uint64_t A;          // total fixed-point born mass
    uint64_t n_in;       // particles inside the grid after predict (= offsets[C])
    uint64_t s_total;    // birth slots allocated (nu_b or 0)
};

// Per-step scalars computed on the host in fp64 and rounded once to f32.
struct StepArgs {
    float Tc;      // T / cell_size: cells moved per (m/s)
    float s_p;     // sigma_pos * T / cell_size: position noise SD in cells (A-1)
    float s_v;     // sigma_vel * T: velocity noise SD in m/s (A-1)
    float alpha;   // exp(-T / free_tau) (A-9)
    int64_t k;     // step counter of the state being advanced
};

struct FilterConst {
    int32_t W, H;
    uint32_t C;
    uint32_t nu, nu_b;
    float p_s, p_b, sigma_b, occ_max, v_max;
    uint64_t seed;
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v)
{
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed64(const uint64_t* p)
{
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Warp inclusive scan (add) of T via shuffles.
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane)
{
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        T o = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += o;
    }
    return v;
}

// Block exclusive scan for blockDim.x = 32*NW threads; returns exclusive prefix and block total.
template <typename T, int NW>
__device__ __forceinline__ T block_excl_scan(T v, T* s_warp /*[NW]*/, T& total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T incl = warp_incl_scan(v, lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        T w = lane < NW ? s_warp[lane] : T(0);
        T wi = warp_incl_scan(w, lane);
        if (lane < NW) s_warp[lane] = wi - w;   // exclusive warp offsets
        if (lane == NW - 1) s_warp[NW] = wi;    // total
    }
    __syncthreads();
    T res = s_warp[warp] + incl - v;
    total = s_warp[NW];
    __syncthreads();
    return res;
}

}  // namespace dog
