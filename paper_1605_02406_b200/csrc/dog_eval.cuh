// dog_eval.cuh -- evaluation workload on the filter's readouts (PAPER section VIII):
// per-cell Mahalanobis distance of the velocity estimate from v = 0 (Eq. 88 `eq:mahadist`), static /
// dynamic classification counts per threshold and the sums behind the cluster statistics
// (Eqs. 85-86).  Arithmetic in fp64 with the operation order of DESIGN.md A-33 (bit-identical m).
#pragma once
#include <cstdint>
#include "dog_common.cuh"

namespace dog {

constexpr int kEvalMaxThr = 64;
constexpr int kEvalBins = kEvalMaxThr + 1;          // rank of m among the sorted thresholds: 0..n
constexpr int kEvBucketBits = 12;                   // rank lookup: top 12 bits of the order-preserving key
constexpr int kEvBuckets = 1 << kEvBucketBits;
// Thresholds sorted ascending (NaN thresholds dropped: m >= NaN never holds; -0 stored as +0, which
// compares equal); pos[t] = sorted position of caller threshold t (-1 for NaN).  tab[b] = number of sorted
// thresholds whose order key is below bucket b's first key (tab[kEvBuckets] = n_sorted), so the rank of m
// -- #{sorted thresholds <= m} -- is tab[bucket(m)] plus a short scan inside that bucket.  Counts come
// from a rank histogram instead of one comparison per (cell, threshold).
struct EvalThr {
    float v[kEvalMaxThr];
    int8_t pos[kEvalMaxThr];
    uint8_t tab[kEvBuckets + 4];
};
struct EvalAcc { unsigned long long hist[2 * kEvalBins]; double sum[5]; unsigned int ticket; };

__host__ __device__ __forceinline__ uint32_t eval_key(float f)      // order-preserving u32 image of f
{
    uint32_t u;
    memcpy(&u, &f, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// m = v P^-1 v^T in fp64, A-33 operation order (bit-identical to orc_eval_cells)
__device__ __forceinline__ float eval_m(bool ok, double vx, double vy, double pxx, double pyy, double pxy)
{
    double m = 0.0;
    if (ok) {
        double det = __dsub_rn(__dmul_rn(pxx, pyy), __dmul_rn(pxy, pxy));
        if (det <= 1e-12) {                                  // regularised (A-33)
            pxx = __dadd_rn(pxx, 1e-6);
            pyy = __dadd_rn(pyy, 1e-6);
            det = __dsub_rn(__dmul_rn(pxx, pyy), __dmul_rn(pxy, pxy));
        }
        const double a = __dmul_rn(__dmul_rn(vx, vx), pyy);
        const double b = __dmul_rn(__dmul_rn(__dmul_rn(2.0, vx), vy), pxy);
        const double e = __dmul_rn(__dmul_rn(vy, vy), pxx);
        m = __ddiv_rn(__dadd_rn(__dsub_rn(a, b), e), det);
    }
    return __double2float_rn(m);
}

// #{sorted thresholds <= mf}; NaN mf -> 0
__device__ __forceinline__ int eval_rank(float mf, const uint8_t* s_tab, const float* s_thr)
{
    if (mf != mf) return 0;
    const uint32_t b = eval_key(mf == 0.f ? 0.f : mf) >> (32 - kEvBucketBits);
    int r = s_tab[b];
    const int hi = s_tab[b + 1];
    while (r < hi && s_thr[r] <= mf) ++r;
    return r;
}

// per-cell classification + cluster-sum accumulation; every lane of the warp calls it (l = 0 / ok = false
// for lanes without a cell) because the histogram update is warp-aggregated
__device__ __forceinline__ void eval_accum(float mf, uint8_t l, bool ok, uint8_t mk, float x, float y, float va,
                                           float vb, bool has_labels, bool has_mask, const uint8_t* s_tab,
                                           const float* s_thr, uint32_t* s_hist, int lane, double (&v)[5], bool& hit)
{
    if (has_labels) {
        const int key = (l == 1 || l == 2) ? (l == 2 ? kEvalBins : 0) + eval_rank(mf, s_tab, s_thr) : -1;
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        if (key >= 0 && lane == __ffs(peers) - 1) atomicAdd(&s_hist[key], (uint32_t)__popc(peers));
    }
    if (has_mask && ok && mk) {
        const double dx = x, dy = y;
        hit = true;
        v[0] += 1.0; v[1] += dx; v[3] += dy;
        v[2] += __dadd_rn((double)va, __dmul_rn(dx, dx));
        v[4] += __dadd_rn((double)vb, __dmul_rn(dy, dy));
    }
}

__device__ __forceinline__ void eval_flush_sums(bool has_mask, double (&v)[5], bool hit, int lane, double* s_sum)
{
    if (has_mask && __any_sync(0xffffffffu, hit)) {
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int i = 0; i < 5; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
        if (lane == 0)
#pragma unroll
            for (int i = 0; i < 5; ++i) atomicAdd(&s_sum[i], v[i]);
    }
#pragma unroll
    for (int i = 0; i < 5; ++i) v[i] = 0.0;
}

// block prologue: zero the block histogram / sums, stage thresholds and the rank table in shared memory
__device__ __forceinline__ void eval_prologue(const EvalThr& thr, uint32_t* s_hist, float* s_thr, uint8_t* s_tab,
                                              double* s_sum)
{
    for (int i = threadIdx.x; i < 2 * kEvalBins; i += blockDim.x) s_hist[i] = 0u;
    for (int i = threadIdx.x; i < kEvalMaxThr; i += blockDim.x) s_thr[i] = thr.v[i];
    for (int i = threadIdx.x; i < (kEvBuckets + 4) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(s_tab)[i] = reinterpret_cast<const uint32_t*>(thr.tab)[i];
    if (threadIdx.x < 5) s_sum[threadIdx.x] = 0.0;
}

// block epilogue; the last block to finish turns the rank histogram into (TP, FN, FP, TN) per caller
// threshold, writes the sums, and resets the accumulator (self-cleaning: no memset launches)
__device__ __forceinline__ void eval_finish(const uint32_t* s_hist, const double* s_sum, const EvalThr& thr, int n_thr,
                                            EvalAcc* acc, unsigned long long* counts, double* sums)
{
    __shared__ bool s_last;
    __shared__ unsigned long long s_suf[2][kEvalBins + 1];
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * kEvalBins; i += blockDim.x)
        if (s_hist[i]) atomicAdd(&acc->hist[i], (unsigned long long)s_hist[i]);
    if (threadIdx.x < 5 && s_sum[threadIdx.x] != 0.0) atomicAdd(&acc->sum[threadIdx.x], s_sum[threadIdx.x]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&acc->ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x < 2) {
        unsigned long long run = 0;
        s_suf[threadIdx.x][kEvalBins] = 0;
        for (int r = kEvalBins - 1; r >= 0; --r) {
            run += __ldcg(&acc->hist[threadIdx.x * kEvalBins + r]);
            s_suf[threadIdx.x][r] = run;                     // #cells of this label with rank >= r
        }
    }
    __syncthreads();
    if (threadIdx.x < n_thr) {
        const int p = thr.pos[threadIdx.x];
        // detected dynamic at sorted position p  <=>  rank > p  (NaN threshold: never)
        const unsigned long long dyn_det = p >= 0 ? s_suf[1][p + 1] : 0ull;
        const unsigned long long sta_det = p >= 0 ? s_suf[0][p + 1] : 0ull;
        counts[4 * threadIdx.x + 0] = dyn_det;
        counts[4 * threadIdx.x + 1] = s_suf[1][0] - dyn_det;
        counts[4 * threadIdx.x + 2] = sta_det;
        counts[4 * threadIdx.x + 3] = s_suf[0][0] - sta_det;
    }
    if (threadIdx.x < 5) sums[threadIdx.x] = __ldcg(&acc->sum[threadIdx.x]);
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * kEvalBins; i += blockDim.x) acc->hist[i] = 0ull;
    if (threadIdx.x < 5) acc->sum[threadIdx.x] = 0.0;
    if (threadIdx.x == 0) acc->ticket = 0u;
}

// one cell read straight from global memory (tails and unaligned inputs)
__device__ __forceinline__ void eval_load_direct(uint32_t c, uint32_t C, const float2* mean, const float* cov,
                                                 const uint8_t* valid, const uint32_t* vbits, const uint8_t* labels,
                                                 const uint8_t* mask, float& x, float& y, float& a, float& b,
                                                 float& cxy, uint8_t& l, uint8_t& mk, bool& ok)
{
    x = y = a = b = cxy = 0.f; l = mk = 0; ok = false;
    if (c >= C) return;
    const float2 mv = mean[c];
    x = mv.x; y = mv.y;
    a = cov[3 * (size_t)c]; b = cov[3 * (size_t)c + 1]; cxy = cov[3 * (size_t)c + 2];
    if (labels) l = labels[c];
    if (mask) mk = mask[c];
    if (vbits) ok = (vbits[c >> 5] >> (c & 31)) & 1u;
    else if (valid) ok = valid[c] != 0;
    else ok = x != 0.f || y != 0.f || a != 0.f || b != 0.f || cxy != 0.f;
}

// ---- direct variant (any alignment): one cell per thread per iteration, grid-stride -------------------
// valid_mode: vbits = the filter's moments-valid bitmask, else valid[] (u8), else "mean or cov nonzero".
__global__ __launch_bounds__(256) void k_eval_cells(const float2* __restrict__ mean, const float* __restrict__ cov,
                                                    const uint8_t* __restrict__ valid, const uint32_t* __restrict__ vbits,
                                                    const uint8_t* __restrict__ labels, const uint8_t* __restrict__ mask,
                                                    const __grid_constant__ EvalThr thr, int n_thr,
                                                    float* __restrict__ m_out, EvalAcc* __restrict__ acc,
                                                    unsigned long long* __restrict__ counts, double* __restrict__ sums,
                                                    uint32_t C)
{
    __shared__ uint32_t s_hist[2 * kEvalBins];
    __shared__ float s_thr[kEvalMaxThr];
    __shared__ __align__(4) uint8_t s_tab[kEvBuckets + 4];
    __shared__ double s_sum[5];
    const int lane = threadIdx.x & 31;
    eval_prologue(thr, s_hist, s_thr, s_tab, s_sum);
    __syncthreads();
    double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    bool hit = false;
    // warp-uniform trip count so every lane reaches the warp collectives
    for (uint32_t base = blockIdx.x * blockDim.x; base < C; base += gridDim.x * blockDim.x) {
        float x, y, a, b, cxy; uint8_t l, mk; bool ok;
        eval_load_direct(base + threadIdx.x, C, mean, cov, valid, vbits, labels, mask, x, y, a, b, cxy, l, mk, ok);
        const float mf = eval_m(ok, x, y, a, b, cxy);
        if (m_out && base + threadIdx.x < C) m_out[base + threadIdx.x] = mf;
        eval_accum(mf, l, ok, mk, x, y, a, b, labels != nullptr, mask != nullptr, s_tab, s_thr, s_hist, lane, v, hit);
    }
    eval_flush_sums(mask != nullptr, v, hit, lane, s_sum);
    eval_finish(s_hist, s_sum, thr, n_thr, acc, counts, sums);
}

// ---- staged variant (16-byte aligned inputs): whole tiles of kEvT cells arrive in shared memory by 1-D
// bulk copies (cp.async.bulk, completion counted on an mbarrier), kEvStages-deep ring, issued by one thread;
// the HBM stream then does not depend on how many warps are resident (the fp64 arithmetic keeps the
// register count -- and so occupancy -- high).  Ragged tail (C mod kEvT) read directly.
constexpr int kEvT = 1024;
constexpr int kEvStages = 4;
constexpr int kEvThreads = 512;
constexpr uint32_t kEvOffMean = 0, kEvOffCov = 8 * kEvT, kEvOffLab = 20 * kEvT, kEvOffMsk = 21 * kEvT,
                   kEvOffVal = 22 * kEvT, kEvStage = 23 * kEvT;
constexpr uint32_t kEvSmem = kEvStages * kEvStage;

__global__ __launch_bounds__(kEvThreads, 2) void k_eval_cells_tma(
    const float2* __restrict__ mean, const float* __restrict__ cov, const uint8_t* __restrict__ valid,
    const uint32_t* __restrict__ vbits, const uint8_t* __restrict__ labels, const uint8_t* __restrict__ mask,
    const __grid_constant__ EvalThr thr, int n_thr, float* __restrict__ m_out, EvalAcc* __restrict__ acc,
    unsigned long long* __restrict__ counts, double* __restrict__ sums, uint32_t C)
{
    extern __shared__ __align__(128) uint8_t ev_sm[];
    __shared__ __align__(8) uint64_t bar[kEvStages];
    __shared__ uint32_t s_hist[2 * kEvalBins];
    __shared__ float s_thr[kEvalMaxThr];
    __shared__ __align__(4) uint8_t s_tab[kEvBuckets + 4];
    __shared__ double s_sum[5];
    const int lane = threadIdx.x & 31;
    eval_prologue(thr, s_hist, s_thr, s_tab, s_sum);
    const uint32_t n_full = C / kEvT;
    const uint32_t tx = 20u * kEvT + (labels ? kEvT : 0u) + (mask ? kEvT : 0u) +
                        (vbits ? kEvT / 8u : valid ? kEvT : 0u);
    auto issue = [&](uint32_t tile, int s) {
        uint8_t* st = ev_sm + s * kEvStage;
        const size_t c0 = (size_t)tile * kEvT;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(tx) : "memory");
        bulk_g2s(st + kEvOffMean, mean + c0, 8u * kEvT, &bar[s]);
        bulk_g2s(st + kEvOffCov, cov + 3 * c0, 12u * kEvT, &bar[s]);
        if (labels) bulk_g2s(st + kEvOffLab, labels + c0, kEvT, &bar[s]);
        if (mask) bulk_g2s(st + kEvOffMsk, mask + c0, kEvT, &bar[s]);
        if (vbits) bulk_g2s(st + kEvOffVal, vbits + c0 / 32, kEvT / 8u, &bar[s]);
        else if (valid) bulk_g2s(st + kEvOffVal, valid + c0, kEvT, &bar[s]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kEvStages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < kEvStages; ++s)
            if (blockIdx.x + s * gridDim.x < n_full) issue(blockIdx.x + s * gridDim.x, s);
    }
    __syncthreads();
    double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    bool hit = false;
    uint32_t k = 0;
    for (uint32_t tile = blockIdx.x; tile < n_full; tile += gridDim.x, ++k) {
        const int s = k % kEvStages;
        mbar_wait(&bar[s], (k / kEvStages) & 1u);
        const uint8_t* st = ev_sm + s * kEvStage;
        const float2* sm_mean = reinterpret_cast<const float2*>(st + kEvOffMean);
        const float* sm_cov = reinterpret_cast<const float*>(st + kEvOffCov);
        const uint32_t c0 = tile * kEvT;
#pragma unroll 2
        for (int i = threadIdx.x; i < kEvT; i += kEvThreads) {
            const float2 mv = sm_mean[i];
            const float a = sm_cov[3 * i], b = sm_cov[3 * i + 1], cxy = sm_cov[3 * i + 2];
            const uint8_t l = labels ? st[kEvOffLab + i] : 0;
            const uint8_t mk = mask ? st[kEvOffMsk + i] : 0;
            bool ok;
            if (vbits) ok = (reinterpret_cast<const uint32_t*>(st + kEvOffVal)[i >> 5] >> (i & 31)) & 1u;
            else if (valid) ok = st[kEvOffVal + i] != 0;
            else ok = mv.x != 0.f || mv.y != 0.f || a != 0.f || b != 0.f || cxy != 0.f;
            const float mf = eval_m(ok, mv.x, mv.y, a, b, cxy);
            if (m_out) m_out[c0 + i] = mf;
            eval_accum(mf, l, ok, mk, mv.x, mv.y, a, b, labels != nullptr, mask != nullptr, s_tab, s_thr, s_hist,
                       lane, v, hit);
        }
        __syncthreads();                                     // stage s consumed by every thread
        if (threadIdx.x == 0 && tile + kEvStages * gridDim.x < n_full) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(tile + kEvStages * gridDim.x, s);
        }
    }
    for (uint32_t base = n_full * kEvT + blockIdx.x * blockDim.x; base < C; base += gridDim.x * blockDim.x) {
        float x, y, a, b, cxy; uint8_t l, mk; bool ok;
        eval_load_direct(base + threadIdx.x, C, mean, cov, valid, vbits, labels, mask, x, y, a, b, cxy, l, mk, ok);
        const float mf = eval_m(ok, x, y, a, b, cxy);
        if (m_out && base + threadIdx.x < C) m_out[base + threadIdx.x] = mf;
        eval_accum(mf, l, ok, mk, x, y, a, b, labels != nullptr, mask != nullptr, s_tab, s_thr, s_hist, lane, v, hit);
    }
    eval_flush_sums(mask != nullptr, v, hit, lane, s_sum);
    eval_finish(s_hist, s_sum, thr, n_thr, acc, counts, sums);
}

}  // namespace dog
