"""Is the Jacobi2D wide-row penalty a property of the memory system?  A plain tiled copy
(no TMA, no stencil): each CTA copies a 64-double x ROWS tile, tiles x-fastest, for the
same bytes laid out as 131072-wide vs 32768-wide rows.  JIT-built with
torch.utils.cpp_extension (probe only, not part of the library)."""
import os, torch
from torch.utils.cpp_extension import load_inline

src = r"""
#include <torch/extension.h>
__global__ void tile_copy(const double* __restrict__ s, double* __restrict__ d, long pitch, int ntx, int rows, int nrows) {
    const int tx = blockIdx.x % ntx, band = blockIdx.x / ntx;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;          // 8 warps
    for (int r = w; r < rows; r += 8) {
        const long row = (long)band * rows + r;
        if (row >= nrows) break;
        const double2 v = reinterpret_cast<const double2*>(s + row * pitch + tx * 64)[lane];
        reinterpret_cast<double2*>(d + row * pitch + tx * 64)[lane] = v;
    }
}
void run(torch::Tensor s, torch::Tensor d, int rows) {
    const long pitch = s.size(1); const int nrows = s.size(0); const int ntx = pitch / 64;
    const int nb = (nrows + rows - 1) / rows;
    tile_copy<<<ntx * nb, 256>>>(s.data_ptr<double>(), d.data_ptr<double>(), pitch, ntx, rows, nrows);
}
"""
m = load_inline("pitch_copy_probe", cpp_sources="void run(torch::Tensor s, torch::Tensor d, int rows);",
                cuda_sources=src, functions=["run"], extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                verbose=False)
for total, rows in ((1 << 29, 16), (1 << 29, 128), (1 << 27, 16), (1 << 27, 128)):  # doubles per array: 4 GiB, 1 GiB
    res = {}
    for width in (32768, 131072, 32768, 131072):
        s = torch.rand((total // width, width), dtype=torch.float64, device="cuda")
        d = torch.empty_like(s)
        for _ in range(3): m.run(s, d, rows)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): m.run(s, d, rows)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res.setdefault(width, []).append(ms)
        del s, d
    print(f"{total * 8 >> 30} GiB arrays, tile rows {rows}: " + "  ".join(f"width {w}: {min(v):.3f} ms ({2 * total * 8 / (min(v) * 1e-3) / 1e12:.2f} TB/s)"
                                           for w, v in res.items()), flush=True)
