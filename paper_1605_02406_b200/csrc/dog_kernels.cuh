// dog_kernels.cuh -- the sm_100a kernels of one DS-PHD/MIB cycle (section VII).
//
// Stage map (paper -> kernel):
//   Alg. 1 predict              -> k_predict_sort (dog_sort.cuh, fused with the tile sort)
//   Alg. 2 sort + assign        -> dog_sort.cuh   (tile-local stable sort + per-cell run lists)
//   NEXT rows: Doppler branch (dog_doppler.cuh), ego scroll (dog_ego.cuh), evaluation (dog_eval.cuh),
//              exact PHD/MIB cell update (k_cells<true>, grid-wide list scan in dog_cells.cuh)
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


constexpr int kSortTile = 4096;     // particles per tile (predict + tile sort, resampling)

}  // namespace dog
