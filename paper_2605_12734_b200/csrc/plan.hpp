// plan.hpp -- host planner: GPU grid, uniform block grid, block->partition map and
// face kinds (the analog of Charm++'s pre-filled location table, and
// of transport selection by source/destination placement).
// Pure host code: unit-testable without a GPU through jac_plan / jac_plan_face.
#pragma once
#include <cstdint>
#include <string>

#include "device.hpp"

namespace jac {

struct Plan {
    int64_t n[3];   // interior points per dim (x, y, z) -- reading R7
    int32_t b[3];   // global blocks per dim
    int32_t g[3];   // GPU (partition) grid
    int32_t n_gpus;
    int64_t e[3];   // block extent (interior points) per dim
    int32_t lb[3];  // blocks per partition per dim = b / g

    int32_t blocks_total() const { return b[0] * b[1] * b[2]; }
    int32_t blocks_per_part() const { return lb[0] * lb[1] * lb[2]; }
    int32_t odf() const { return blocks_total() / n_gpus; }

    // partition owning block (ix,iy,iz); partitions are contiguous sub-boxes of
    // the block grid, id = (pz*gy + py)*gx + px (SPEC.md:259-265 contiguous map).
    int32_t owner(int32_t ix, int32_t iy, int32_t iz) const {
        const int32_t px = ix / lb[0], py = iy / lb[1], pz = iz / lb[2];
        return (pz * g[1] + py) * g[0] + px;
    }
    // slot of a block inside its owner's arena (local coords, x fastest)
    int32_t local_slot(int32_t ix, int32_t iy, int32_t iz) const {
        const int32_t lx = ix % lb[0], ly = iy % lb[1], lz = iz % lb[2];
        return (lz * lb[1] + ly) * lb[0] + lx;
    }
    void block_of(int32_t part, int32_t slot, int32_t out[3]) const {
        const int32_t px = part % g[0], py = (part / g[0]) % g[1], pz = part / (g[0] * g[1]);
        const int32_t lx = slot % lb[0], ly = (slot / lb[0]) % lb[1], lz = slot / (lb[0] * lb[1]);
        out[0] = px * lb[0] + lx;
        out[1] = py * lb[1] + ly;
        out[2] = pz * lb[2] + lz;
    }
    // neighbour of block across face f; false at the global boundary
    bool neighbor(const int32_t blk[3], int f, int32_t nb[3]) const {
        nb[0] = blk[0]; nb[1] = blk[1]; nb[2] = blk[2];
        const int d = f >> 1;
        nb[d] += (f & 1) ? 1 : -1;
        return nb[d] >= 0 && nb[d] < b[d];
    }
};

// Validates and fills *out.  Returns 0 (JAC_OK), -1 (EINVAL) or -2 (EDECOMP);
// *err names the offending argument.  gpu_grid == nullptr selects the GPU grid by
// reading R10: minimum total inter-GPU face area, ties prefer splitting z, then y.
int make_plan(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz,
              int32_t n_gpus, const int32_t *gpu_grid, Plan *out, std::string *err);

}  // namespace jac
