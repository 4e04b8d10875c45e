// dog_sort.cuh -- Alg. 2: stable sort of the predicted particles by cell key.
//
// LSD radix sort of (key, input index) with 8-bit digits, reduce-then-scan per pass (no look-back):
//   up   : per 4096-element tile, the digit histogram of the pass (pass 0: fused into k_predict)
//   scan : per digit, exclusive prefix over tiles + the digit's global base -> each tile's offsets
//   down : per tile, stable local ranking (warps own consecutive 512-element slices and rank in
//          order with match_any + running per-warp digit counters, A-6), then scatter.
// Sorting (key, index) pairs with a stable LSD sort orders ties by input index, exactly the
// oracle's stable sort.  The last pass writes only the permutation (cell-sorted slot -> index).
#pragma once
#include <cstdint>
#include "dog_common.cuh"
#include "dog_kernels.cuh"

namespace dog {

constexpr int kRsThreads = 256, kRsItems = 16, kRsWarps = 8;
static_assert(kRsThreads * kRsItems == kSortTile, "sort tile");

// Digit histogram of pass `shift` for every tile of the (already permuted) key array.
__global__ __launch_bounds__(kRsThreads) void k_rs_up(const uint32_t* __restrict__ kin, uint32_t n, int shift,
                                                      uint32_t* __restrict__ hist, uint32_t ntiles)
{
    __shared__ uint32_t s_h[kRsWarps][256];
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < kRsWarps * 256; i += kRsThreads) (&s_h[0][0])[i] = 0;
    __syncthreads();
    const uint32_t base = blockIdx.x * kSortTile;
#pragma unroll
    for (int i = 0; i < kRsItems / 4; ++i) {
        const uint32_t idx = base + (i * kRsThreads + tid) * 4;
        if (idx + 3 < n) {
            const uint4 k4 = *reinterpret_cast<const uint4*>(kin + idx);
            atomicAdd(&s_h[warp][(k4.x >> shift) & 255u], 1u);
            atomicAdd(&s_h[warp][(k4.y >> shift) & 255u], 1u);
            atomicAdd(&s_h[warp][(k4.z >> shift) & 255u], 1u);
            atomicAdd(&s_h[warp][(k4.w >> shift) & 255u], 1u);
        } else {
            for (uint32_t e = idx; e < n && e < idx + 4; ++e) atomicAdd(&s_h[warp][(kin[e] >> shift) & 255u], 1u);
        }
    }
    __syncthreads();
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) t += s_h[w][tid];
    hist[(size_t)tid * ntiles + blockIdx.x] = t;
}

// One block per digit d: hist[d][*] (counts per tile) -> global output offset of each tile's first
// element with digit d = (elements with smaller digits) + (digit-d elements of earlier tiles).
__global__ __launch_bounds__(256) void k_rs_scan(uint32_t* __restrict__ hist, const uint32_t* __restrict__ dhist,
                                                 uint32_t ntiles)
{
    __shared__ uint32_t s_scan[9];
    __shared__ uint32_t s_base;
    const int d = blockIdx.x, tid = threadIdx.x;
    uint32_t part = 0;
    for (int i = tid; i < d; i += 256) part += dhist[i];
    part = warp_sum(part);
    if ((tid & 31) == 0) s_scan[tid >> 5] = part;
    __syncthreads();
    if (tid == 0) {
        uint32_t b = 0;
        for (int w = 0; w < 8; ++w) b += s_scan[w];
        s_base = b;
    }
    __syncthreads();
    uint32_t carry = s_base;
    uint32_t* row = hist + (size_t)d * ntiles;
    for (uint32_t t0 = 0; t0 < ntiles; t0 += 256 * 8) {
        uint32_t v[8], sum = 0;
        const uint32_t b = t0 + tid * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) { v[i] = b + i < ntiles ? row[b + i] : 0u; sum += v[i]; }
        uint32_t tot;
        uint32_t run = carry + block_excl_scan<uint32_t, 8>(sum, s_scan, tot);
#pragma unroll
        for (int i = 0; i < 8; ++i) { if (b + i < ntiles) row[b + i] = run; run += v[i]; }
        carry += tot;
    }
}

template <bool FIRST, bool LAST>
__global__ __launch_bounds__(kRsThreads) void k_rs_down(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, uint32_t n, int shift, const uint32_t* __restrict__ offs, uint32_t ntiles)
{
    __shared__ uint32_t s_keys[kSortTile];
    __shared__ uint32_t s_vals[kSortTile];
    __shared__ uint32_t s_whist[kRsWarps][256];
    __shared__ uint32_t s_gofs[256];
    __shared__ uint32_t s_lstart[256];
    __shared__ uint32_t s_scan[kRsWarps + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < kRsWarps * 256; i += kRsThreads) (&s_whist[0][0])[i] = 0;
    const uint32_t tile = blockIdx.x;
    const uint32_t base = tile * kSortTile + warp * (kRsItems * 32);
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t goff = offs[(size_t)tid * ntiles + tile];      // this tile's offset for digit tid
    __syncthreads();

    uint32_t k[kRsItems], v[kRsItems], rk[kRsItems];
#pragma unroll
    for (int i = 0; i < kRsItems; ++i) {
        const uint32_t idx = base + i * 32 + lane;
        const bool ok = idx < n;
        k[i] = ok ? kin[idx] : 0u;
        v[i] = FIRST ? idx : (ok ? vin[idx] : 0u);
    }
#pragma unroll
    for (int i = 0; i < kRsItems; ++i) {
        const uint32_t idx = base + i * 32 + lane;
        const bool ok = idx < n;
        const uint32_t dig = ok ? ((k[i] >> shift) & 255u) : 0x100u;
        const uint32_t peers = __match_any_sync(0xffffffffu, dig);
        const uint32_t r = __popc(peers & lt);
        uint32_t prev = 0;
        if (ok) prev = s_whist[warp][dig];
        __syncwarp();
        if (ok && r == 0) s_whist[warp][dig] = prev + __popc(peers);
        __syncwarp();
        rk[i] = prev + r;
    }
    __syncthreads();
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
        const uint32_t c = s_whist[w][tid];
        s_whist[w][tid] = run;
        run += c;
    }
    uint32_t tot;
    const uint32_t lstart = block_excl_scan<uint32_t, kRsWarps>(run, s_scan, tot);
    s_lstart[tid] = lstart;
    s_gofs[tid] = goff - lstart;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRsItems; ++i) {
        const uint32_t idx = base + i * 32 + lane;
        if (idx < n) {
            const uint32_t dig = (k[i] >> shift) & 255u;
            const uint32_t pos = s_lstart[dig] + s_whist[warp][dig] + rk[i];
            s_keys[pos] = k[i];
            s_vals[pos] = v[i];
        }
    }
    __syncthreads();
    const uint32_t tile0 = tile * kSortTile;
    const uint32_t nvalid = n > tile0 ? min((uint32_t)kSortTile, n - tile0) : 0u;
    for (uint32_t p = tid; p < nvalid; p += kRsThreads) {
        const uint32_t key = s_keys[p];
        const uint32_t o = s_gofs[(key >> shift) & 255u] + p;
        if (!LAST || kout) kout[o] = key;
        vout[o] = s_vals[p];
    }
}

}  // namespace dog
