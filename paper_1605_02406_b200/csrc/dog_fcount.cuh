// dog_fcount.cuh -- systematic resampling in closed form (A-24): F(X) = #{i : t_i < X}.
#pragma once
#include <cstdint>
#include "dog_common.cuh"

namespace dog {

struct RsConst {
    uint64_t W;
    uint32_t U, nu;
    double nu_over_W;  // nu / W  (fp64)
    double U_frac;     // U 2^-32  (exact)
    u128 UW;           // U * W
    bool exact;        // skip the fp64 estimate (diagnostics: FilterConst::force_exact)
};

__device__ __forceinline__ RsConst make_rsconst(const DevScalars* sc, uint32_t nu, bool exact = false)
{
    RsConst r;
    r.exact = exact;
    r.W = scrd(sc->Wtot);            // joint weight over all shards (k_pair_sort)
    r.U = scrd(sc->U);
    r.nu = nu;
    r.nu_over_W = scrd(sc->nu_over_W);  // (double)nu / (double)W, divided once in k_pair_sort
    r.U_frac = (double)r.U * 0x1p-32;
    r.UW = (u128)r.U * (u128)r.W;
    return r;
}

// F(X) = number of systematic targets t_i below X = clamp(ceil(y), 0, nu) with
// y = (X nu 2^32 - U W) / (W 2^32) = X nu / W - U 2^-32.  The fp64 estimate of y is within 2^-20
// of y (|y| < 2^31, relative error < 2^-51); when it is further than 2^-16 from an integer its
// ceiling is exact, otherwise the ceiling is settled with exact 128-bit products.
__device__ __forceinline__ uint32_t fcount(uint64_t X, const RsConst& r)
{
    const double y = __fma_rn((double)X, r.nu_over_W, -r.U_frac);
    if (y <= -0.5) return 0u;
    if (y >= (double)r.nu) return r.nu;
    const double cy = ceil(y);
    const double d = cy - y;                       // in [0, 1)
    if (d > 0x1p-16 && d < 1.0 - 0x1p-16 && !r.exact) return (uint32_t)cy;
    const u128 num0 = ((u128)X * (u128)r.nu) << 32;
    if (num0 <= r.UW) return 0u;
    const u128 num = num0 - r.UW;
    const u128 E = ((u128)r.W) << 32;
    uint64_t q = (uint64_t)fmax(cy - 1.0, 0.0);
    while ((u128)q * E < num) ++q;                 // smallest q with q W 2^32 >= X nu 2^32 - U W
    while (q > 0 && (u128)(q - 1) * E >= num) --q;
    return (uint32_t)(q < r.nu ? q : r.nu);
}

}  // namespace dog
