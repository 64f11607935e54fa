// plan.cpp -- see plan.hpp.  Error conventions follow SPEC.md's Jacobi interface:
// "tiling mismatch -> configuration error", integral ODF and
// divisibility preconditions, zero counts rejected.
#include "plan.hpp"

#include <limits>

namespace jac {

int make_plan(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz,
              int32_t n_gpus, const int32_t *gpu_grid, Plan *out, std::string *err)
{
    const int64_t n[3] = {nx, ny, nz};
    const int32_t b[3] = {bx, by, bz};
    static const char *nn[3] = {"nx", "ny", "nz"}, *bn[3] = {"bx", "by", "bz"};
    for (int d = 0; d < 3; ++d) {
        if (n[d] < 1) { *err = std::string(nn[d]) + " must be >= 1"; return -1; }
        if (b[d] < 1) { *err = std::string(bn[d]) + " must be >= 1"; return -1; }
    }
    if (n_gpus < 1) { *err = "n_gpus must be >= 1"; return -1; }
    // keep every index below 2^31 blocks and the padded grid below 2^40 cells (R11 key)
    if ((int64_t)bx * by * bz > (int64_t)1 << 30) { *err = "bx*by*bz too large"; return -1; }
    if ((double)(nx + 2) * (double)(ny + 2) * (double)(nz + 2) >= 1099511627776.0) {
        *err = "padded grid must have < 2^40 cells (R11 hash key)"; return -1;
    }
    for (int d = 0; d < 3; ++d)
        if (n[d] % b[d] != 0) {
            *err = std::string(nn[d]) + " % " + bn[d] + " != 0 (blocks must tile the grid evenly)";
            return -2;
        }
    const int64_t nblk = (int64_t)bx * by * bz;
    if (nblk % n_gpus != 0) {
        *err = "(bx*by*bz) % n_gpus != 0 (ODF must be integral)";
        return -2;
    }
    int32_t g[3];
    if (gpu_grid) {
        for (int d = 0; d < 3; ++d) {
            g[d] = gpu_grid[d];
            if (g[d] < 1) { *err = "gpu_grid entries must be >= 1"; return -1; }
        }
        if ((int64_t)g[0] * g[1] * g[2] != n_gpus) { *err = "gpu_grid product != n_gpus"; return -2; }
        for (int d = 0; d < 3; ++d)
            if (b[d] % g[d] != 0) {
                *err = std::string(bn[d]) + " % gpu_grid[" + std::to_string(d) + "] != 0";
                return -2;
            }
    } else {
        // R10: minimise (gx-1)*ny*nz + (gy-1)*nx*nz + (gz-1)*nx*ny over divisible
        // factorisations; ties prefer more splits in z, then in y.
        double best = std::numeric_limits<double>::infinity();
        int32_t bg[3] = {0, 0, 0};
        for (int32_t gx = 1; gx <= n_gpus; ++gx) {
            if (n_gpus % gx || bx % gx) continue;
            for (int32_t gy = 1; gy <= n_gpus / gx; ++gy) {
                if ((n_gpus / gx) % gy || by % gy) continue;
                const int32_t gz = n_gpus / gx / gy;
                if (bz % gz) continue;
                const double area = (double)(gx - 1) * ny * nz + (double)(gy - 1) * nx * nz +
                                    (double)(gz - 1) * nx * ny;
                bool better = area < best;
                if (area == best) better = (gz > bg[2]) || (gz == bg[2] && gy > bg[1]);
                if (better) { best = area; bg[0] = gx; bg[1] = gy; bg[2] = gz; }
            }
        }
        if (bg[0] == 0) { *err = "no GPU grid divides the block grid (bx,by,bz) for n_gpus"; return -2; }
        g[0] = bg[0]; g[1] = bg[1]; g[2] = bg[2];
    }
    for (int d = 0; d < 3; ++d) {
        out->n[d] = n[d];
        out->b[d] = b[d];
        out->g[d] = g[d];
        out->e[d] = n[d] / b[d];
        out->lb[d] = b[d] / g[d];
    }
    out->n_gpus = n_gpus;
    return 0;
}

}  // namespace jac
