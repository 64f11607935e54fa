// kernels.hpp -- host-side launchers of the sm_100a kernels (kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "device.hpp"

namespace jac {

enum TmaVariant { TMA_WIDE = 0 /* 64 x 16 tiles */, TMA_NARROW = 1 /* 32 x 16 tiles */ };
struct TileShape { int bx, by; };

TileShape tma_tile_shape(int variant);
cudaError_t prepare_sweep_tma(int variant);
int sweep_resident_ctas(int variant);         // SMs x resident CTAs of the TMA sweep (current device)  // sets the dynamic-smem attribute (current device)
cudaError_t launch_sweep_tma(const CUtensorMap &tm, const SweepArgs &a, int variant, cudaStream_t s);
cudaError_t launch_sweep_plain(const SweepArgs &a, cudaStream_t s);  // 64 x 8 tiles
cudaError_t launch_ghost_fill(const SweepArgs &a, int dst, cudaStream_t s);
cudaError_t launch_barrier(const BarrierArgs &ba, cudaStream_t s);
cudaError_t launch_hash_init(const SweepArgs &a, int64_t nx, int64_t ny, uint64_t seed, cudaStream_t s);

}  // namespace jac
