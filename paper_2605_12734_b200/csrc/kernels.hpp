// kernels.hpp -- host-side launchers of the sm_100a kernels (kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "device.hpp"

namespace jac {

enum TmaVariant {
    TMA_WIDE = 0,    /* 64 x 16 tiles, staged 68 wide (blocks wider than 64), 6-stage ring */
    TMA_WIDE4 = 5,   /* the same with a 4-stage ring (autotune candidate) */
    TMA_NARROW = 1,  /* 32 x 16 tiles, staged 36 wide (blocks 33..64 wide) */
    TMA_EXACT32 = 3, /* 32 x 16 tiles, staged 32 wide: one tile per block row (ex <= 32) */
    TMA_EXACT64 = 4, /* 64 x 16 tiles, staged 64 wide: one tile per block row (ex <= 64) */
    TMA_EXACT32_TALL = 12, /* 32 x 32 tiles: a whole 32^2 block face per item (ex <= 32) */
    TMA_EXACT32_6 = 13,    /* 32 x 16 tiles, 6-stage ring (ex <= 32) */
    TMA_EXACT64_6 = 14,    /* 64 x 16 tiles, 6-stage ring (ex <= 64) */
    TMA_WIDE_TALL = 15     /* 64 x 32 tiles staged 68 x 34, 4-stage ring, 2 CTAs / SM (experiment:
                              fewer shared-memory loads and less staging over-fetch per point) */
};
struct TileShape { int bx, by, w; };

TileShape tma_tile_shape(int variant);
cudaError_t prepare_sweep_tma(int variant);   // sets the dynamic-smem attribute (current device)
int sweep_resident_ctas(int variant);         // SMs x resident CTAs of the TMA sweep (current device)
// pdl: launch with programmatic stream serialization (the next sweep's CTAs may be
// scheduled during this one's tail; they wait for its completion before any access)
cudaError_t launch_sweep_tma(const CUtensorMap &tm, const SweepArgs &a, int variant, cudaStream_t s,
                             bool pdl = false);
cudaError_t launch_sweep2d_tma(const CUtensorMap &tm, const SweepArgs &a, int variant, cudaStream_t s,
                               bool pdl = false);
cudaError_t prepare_sweep2d_tma(int variant);
cudaError_t launch_sweep_plain(const SweepArgs &a, cudaStream_t s);  // 64 x 8 tiles
cudaError_t launch_sweep_plain_one(const SweepArgs &a, cudaStream_t s);  // a.blocks = one block
cudaError_t launch_ghost_fill(const SweepArgs &a, int dst, cudaStream_t s);
cudaError_t launch_barrier(const BarrierArgs &ba, cudaStream_t s);
// n copies of the device list (virtual-partition transport); maxcount = largest count
cudaError_t launch_face_copy(const FaceCopy *list, int n, int64_t maxcount, cudaStream_t s);
cudaError_t launch_pack_face(const SweepArgs &a, int slot, int f, int buf, int par, cudaStream_t s);
cudaError_t launch_unpack_face(const SweepArgs &a, int slot, int nslot, int f, int buf, int par, cudaStream_t s);
cudaError_t launch_xghost_extract(const SweepArgs &a, cudaStream_t s);
cudaError_t launch_hash_init(const SweepArgs &a, int64_t nx, int64_t ny, uint64_t seed, cudaStream_t s);
// Staged host transfers (jac_set_init_box / jac_get_field_box): one slab of the local
// box sits in device staging memory, x fastest; the kernels move it into / out of the
// blocks listed in list[0..nlist) (indices into a.blocks).
struct StageBox {
    int64_t o[3];  // padded global coordinates of the first staged cell
    int64_t n[3];  // staged extents (x, y, z)
    int64_t pitch; // doubles per staged row (>= n[0])
};
// every ghost-inclusive cell of a listed block inside the stage box -> both buffers
// (dense rows: x ghosts -> both x-ghost arrays), as hash_init does with hash values
cudaError_t launch_stage_scatter(const SweepArgs &a, const int32_t *list, int32_t nlist, int64_t rows,
                                 const double *st, const StageBox &sb, cudaStream_t s);
// every interior cell of a listed block inside the stage box, buffer `buf` -> staging
cudaError_t launch_stage_gather(const SweepArgs &a, const int32_t *list, int32_t nlist, int64_t rows, double *st,
                                const StageBox &sb, int buf, cudaStream_t s);

}  // namespace jac
