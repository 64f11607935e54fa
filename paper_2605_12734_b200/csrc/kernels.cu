// kernels.cu -- sm_100a kernels of the overdecomposed Jacobi3D hot path.
//
//  sweep_tma_kernel   north-star subsystem (2): ONE batched launch per GPU per
//                     iteration walks every local block through the descriptor
//                     table.  Each CTA owns a BX x BY column tile of one block and
//                     marches a z-chunk; z-planes (with x/y halo) are staged into a
//                     ring of shared-memory buffers by TMA (cp.async.bulk.tensor,
//                     mbarrier complete_tx), the z-neighbours ride in registers.
//                     The epilogue stores the new interior AND, for boundary layers,
//                     the same values straight into the neighbour block's ghost
//                     cells of the output buffer (fused pack + ghost copy; peer
//                     blocks on other GPUs are written over NVLink through IPC
//                     pointers), so ODF costs no extra launch and no extra pass.
//  sweep_plain_kernel JAC_F_NO_TMA ablation: per-point global loads (L1/L2 reuse).
//  ghost_fill_kernel  north-star subsystem (3) as the JAC_F_UNFUSED_PACK path: the
//                     sweep packs faces into an outbox, this batched kernel copies
//                     every block's neighbour outboxes into its ghosts (PAPER.md:90
//                     pack/unpack kernels; PAPER.md:269 intra-process D2D copy).
//  barrier_kernel     cross-rank neighbour barrier on device flags (st.release.sys /
//                     ld.acquire.sys over NVLink), replacing the paper's IPC event
//                     pool.
//  hash_init_kernel   R11 synthetic initial field (input generation, not the method).
//
// The update (PAPER.md:281 Jacobi, 3-D lift R1; readings R2-R4 in DESIGN.md):
//     u' = ((((((c + x-) + x+) + y-) + y+) + z-) + z+) * fl(1/7)
// computed with __dadd_rn/__dmul_rn (no contraction, no reassociation; built with
// -fmad=false), so every ODF and GPU count reproduces the oracle bit for bit.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>

#include "device.hpp"
#include "kernels.hpp"

namespace jac {

__device__ __forceinline__ double stencil7(double c, double xm, double xp, double ym, double yp,
                                           double zm, double zp)
{
    constexpr double K = 0x1.2492492492492p-3;  // fl(1/7), reading R3
    double s = __dadd_rn(c, xm);
    s = __dadd_rn(s, xp);
    s = __dadd_rn(s, ym);
    s = __dadd_rn(s, yp);
    s = __dadd_rn(s, zm);
    s = __dadd_rn(s, zp);
    return __dmul_rn(s, K);
}

__device__ __forceinline__ void st_pair(double *p, double2 v, bool both)
{
    if (both) *reinterpret_cast<double2 *>(p) = v;
    else p[0] = v.x;
}

// Stores the new values of points (i, j, k) and (i+1, j, k) of block `blk` into
// buffer `dst`, plus the face traffic of the chosen mode.  Caller guarantees
// j < ey and 0 <= k < ez; i may be past the ragged x edge.
__device__ __forceinline__ void emit_pair(const SweepArgs &a, const DevBlock &blk, int dst,
                                          int i, int j, int k, double2 v)
{
    const Geom &g = a.g;
    if (i >= g.ex) return;
    const bool both = (i + 1) < g.ex;
    const int64_t row = (int64_t)(j + 1) * g.P + g.A + i;
    const int64_t off = (int64_t)(k + 1) * g.Q + row;
    double *own = a.arena + (int64_t)(dst * g.nslots + blk.slot) * g.bstride;
    st_pair(own + off, v, both);
    if (a.mode == MODE_NOEXCHANGE) return;
    if (a.mode == MODE_FUSED) {
        // direct-to-ghost: the neighbour's ghost layer of the OUTPUT buffer is not
        // read by anyone during this sweep, so writing it here is race-free.
        if (k == 0) {
            double *p = blk.nb[ZM][dst];
            if (p) st_pair(p + (int64_t)(g.ez + 1) * g.Q + row, v, both);
        }
        if (k == g.ez - 1) {
            double *p = blk.nb[ZP][dst];
            if (p) st_pair(p + row, v, both);
        }
        if (j == 0) {
            double *p = blk.nb[YM][dst];
            if (p) st_pair(p + (int64_t)(k + 1) * g.Q + (int64_t)(g.ey + 1) * g.P + g.A + i, v, both);
        }
        if (j == g.ey - 1) {
            double *p = blk.nb[YP][dst];
            if (p) st_pair(p + (int64_t)(k + 1) * g.Q + g.A + i, v, both);
        }
        // x-faces: the ghost column is strided (one value per row).  Write the
        // whole 32-byte sector holding it (the rest is row padding) so L2 never
        // has to fetch a partially written sector from DRAM.
        if (i == 0) {
            double *p = blk.nb[XM][dst];
            if (p) {
                double *q = p + (off - i + g.ex);  // neighbour's ghost column i = ex (col A+ex)
                if (((g.A + g.ex) & 3) == 0) {  // ghost alone in its sector
                    *reinterpret_cast<double2 *>(q) = make_double2(v.x, 0.0);
                    *reinterpret_cast<double2 *>(q + 2) = make_double2(0.0, 0.0);
                } else {
                    *q = v.x;
                }
            }
        }
        const bool last_x = (i == g.ex - 1) || (both && i + 1 == g.ex - 1);
        if (last_x) {
            double *p = blk.nb[XP][dst];
            if (p) {
                const double val = (i == g.ex - 1) ? v.x : v.y;
                double *q = p + (off - i - 1);     // neighbour's ghost column i = -1 (col A-1)
                if ((g.A & 3) == 0) {                // ghost is the last word of its sector
                    *reinterpret_cast<double2 *>(q - 3) = make_double2(0.0, 0.0);
                    *reinterpret_cast<double2 *>(q - 1) = make_double2(0.0, val);
                } else {
                    *q = val;
                }
            }
        }
    } else {  // MODE_PACK: contiguous outbox faces, layouts x:[k][j] y:[k][i] z:[j][i]
        double *ob = a.outbox + (int64_t)blk.slot * g.ostride;
        if (k == 0 && blk.nb[ZM][0]) {
            double *p = ob + g.ooff[ZM] + (int64_t)j * g.ex + i;
            p[0] = v.x; if (both) p[1] = v.y;
        }
        if (k == g.ez - 1 && blk.nb[ZP][0]) {
            double *p = ob + g.ooff[ZP] + (int64_t)j * g.ex + i;
            p[0] = v.x; if (both) p[1] = v.y;
        }
        if (j == 0 && blk.nb[YM][0]) {
            double *p = ob + g.ooff[YM] + (int64_t)k * g.ex + i;
            p[0] = v.x; if (both) p[1] = v.y;
        }
        if (j == g.ey - 1 && blk.nb[YP][0]) {
            double *p = ob + g.ooff[YP] + (int64_t)k * g.ex + i;
            p[0] = v.x; if (both) p[1] = v.y;
        }
        if (i == 0 && blk.nb[XM][0]) ob[g.ooff[XM] + (int64_t)k * g.ey + j] = v.x;
        if (i == g.ex - 1 && blk.nb[XP][0]) ob[g.ooff[XP] + (int64_t)k * g.ey + j] = v.x;
        else if (both && i + 1 == g.ex - 1 && blk.nb[XP][0])
            ob[g.ooff[XP] + (int64_t)k * g.ey + j] = v.y;
    }
}

// ------------------------------------------------------------------ TMA / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_fence_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Watchdog: a wait that cannot complete (a TMA that never lands, a peer rank that
// never signals) traps after ~kSpinLimitNs instead of hanging the GPU.
constexpr uint64_t kSpinLimitNs = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ uint64_t globaltimer_ns()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ bool mbar_try(uint32_t b, uint32_t parity)
{
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
    return done != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    const uint32_t b = smem_u32(bar);
    if (mbar_try(b, parity)) return;
    const uint64_t t0 = globaltimer_ns();
    while (!mbar_try(b, parity))
        if (globaltimer_ns() - t0 > kSpinLimitNs) __trap();
}

__device__ __forceinline__ void tma_plane(const CUtensorMap *tm, double *dst, uint64_t *bar,
                                          uint32_t bytes, int c0, int c1, int c2, int c3)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar))
        : "memory");
}

constexpr size_t tma_smem_bytes(int BX, int BY, int NS)
{
    return (size_t)NS * (((BX + 4) * (BY + 2) + 15) / 16 * 16) * sizeof(double) + NS * sizeof(uint64_t);
}

struct TileItem {
    int b, x0, y0, zs, ze;
};

template <int BX, int BY>
__device__ __forceinline__ TileItem decode_item(const SweepArgs &a, int item)
{
    TileItem t;
    const int grp = item / (a.gcols * a.nzc);
    const int r = item - grp * a.gcols * a.nzc;
    const int gsize = min(a.gcols, a.ncols - grp * a.gcols);
    const int zi = r / gsize;
    int col = grp * a.gcols + (r - zi * gsize);
    const int tx = col % a.ntx; col /= a.ntx;
    const int ty = col % a.nty;
    t.b = col / a.nty;
    t.x0 = tx * BX;
    t.y0 = ty * BY;
    t.zs = (int)(((int64_t)zi * a.g.ez) / a.nzc);
    t.ze = (int)(((int64_t)(zi + 1) * a.g.ez) / a.nzc);
    return t;
}

// Producer state (thread 0 only): walks this CTA's items and their planes in order,
// keeping up to NS plane loads in flight across item boundaries.
template <int BX, int BY, int NS>
struct Producer {
    int item;    // current item index (global)
    int p;       // plane offset within the item's load sequence (0 .. ze-zs+1)
    uint32_t l;  // loads issued so far
    TileItem t;
    int c3;

    __device__ __forceinline__ void start(const SweepArgs &a)
    {
        item = blockIdx.x;
        p = 0;
        l = 0;
        if (item < a.nitems) {
            t = decode_item<BX, BY>(a, item);
            c3 = a.src * a.g.nslots + a.blocks[t.b].slot;
        }
    }
    __device__ __forceinline__ void issue(const SweepArgs &a, const CUtensorMap *tm, double *stage,
                                          uint64_t *bars, int stage_doubles, uint32_t bytes)
    {
        if (item >= a.nitems) return;
        const int s = (int)(l % NS);
        // plane k = zs - 1 + p  ->  tensor z index k + 1 = zs + p
        tma_plane(tm, stage + s * stage_doubles, &bars[s], bytes, a.g.A - 2 + t.x0, t.y0, t.zs + p, c3);
        ++l;
        if (++p == t.ze - t.zs + 2) {
            p = 0;
            item += gridDim.x;
            if (item < a.nitems) {
                t = decode_item<BX, BY>(a, item);
                c3 = a.src * a.g.nslots + a.blocks[t.b].slot;
            }
        }
    }
};

// Persistent TMA z-march.  BX x BY column tile per work item, NT threads, NS-deep
// plane ring.  Each thread owns a pair of x-points (double2) in RY rows; the
// z-neighbours ride in registers, x/y neighbours come from the staged plane.
template <int BX, int BY, int NT, int NS>
__global__ void __launch_bounds__(NT, 4) sweep_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                       const SweepArgs a)
{
    constexpr int TXL = BX / 2;    // threads along x
    constexpr int NRG = NT / TXL;  // row groups
    constexpr int RY = BY / NRG;   // rows per thread
    static_assert(RY >= 1 && RY * NRG == BY, "tile shape");
    constexpr int W = BX + 4;      // staged width: x0-2 .. x0+BX+1
    constexpr int H = BY + 2;      // staged height: y0-1 .. y0+BY
    constexpr uint32_t STAGE_BYTES = W * H * sizeof(double);  // TMA transaction bytes
    constexpr int STAGE = (W * H + 15) / 16 * 16;  // ring stride: TMA needs 128-byte aligned smem
    static_assert(NS >= 3, "ring must hold planes k, k+1 and prefetch");

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stage = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + NS * STAGE * sizeof(double));

    const Geom &g = a.g;
    __shared__ Producer<BX, BY, NS> prod;  // touched by thread 0 only; kept out of registers
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
        mbar_fence_init();
        prod.start(a);
        for (int s = 0; s < NS; ++s) prod.issue(a, &tmap, stage, bars, STAGE, STAGE_BYTES);
    }
    __syncthreads();

    const int lane = threadIdx.x % TXL;
    const int rg = threadIdx.x / TXL;
    const int col = 2 * lane + 2;  // staged column of point i = x0 + 2*lane
    const int dst = 1 - a.src;
    uint32_t l = 0;                // loads consumed

    // release(): every thread is done with the oldest unreleased stage -> refill it
    auto release = [&]() {
        __syncthreads();
        if (threadIdx.x == 0) prod.issue(a, &tmap, stage, bars, STAGE, STAGE_BYTES);
    };
    auto plane = [&](uint32_t li) { return stage + (li % NS) * STAGE; };
    auto wait = [&](uint32_t li) { mbar_wait(&bars[li % NS], (li / NS) & 1); };

    for (int item = blockIdx.x; item < a.nitems; item += gridDim.x) {
        const TileItem t = decode_item<BX, BY>(a, item);
        const DevBlock &blk = a.blocks[t.b];
        const int i = t.x0 + 2 * lane;
        double2 zm[RY], c[RY], zp[RY];
        wait(l);
#pragma unroll
        for (int r = 0; r < RY; ++r)
            zm[r] = *reinterpret_cast<const double2 *>(plane(l) + (rg * RY + r + 1) * W + col);
        release();  // plane zs-1 only feeds zm
        ++l;
        wait(l);
#pragma unroll
        for (int r = 0; r < RY; ++r)
            c[r] = *reinterpret_cast<const double2 *>(plane(l) + (rg * RY + r + 1) * W + col);

        for (int k = t.zs; k < t.ze; ++k) {
            const double *Sn = plane(l + 1);
            wait(l + 1);
#pragma unroll
            for (int r = 0; r < RY; ++r)
                zp[r] = *reinterpret_cast<const double2 *>(Sn + (rg * RY + r + 1) * W + col);
            const double *S = plane(l);
#pragma unroll
            for (int r = 0; r < RY; ++r) {
                const int jl = rg * RY + r;
                const double *row = S + (jl + 1) * W + col;
                const double xm = row[-1];
                const double xp = row[2];
                const double2 ym = (r == 0) ? *reinterpret_cast<const double2 *>(row - W) : c[r - 1];
                const double2 yp = (r == RY - 1) ? *reinterpret_cast<const double2 *>(row + W) : c[r + 1];
                double2 v;
                v.x = stencil7(c[r].x, xm, c[r].y, ym.x, yp.x, zm[r].x, zp[r].x);
                v.y = stencil7(c[r].y, c[r].x, xp, ym.y, yp.y, zm[r].y, zp[r].y);
                const int j = t.y0 + jl;
                if (j < g.ey) emit_pair(a, blk, dst, i, j, k, v);
            }
            release();  // centre plane k is done
            ++l;
#pragma unroll
            for (int r = 0; r < RY; ++r) { zm[r] = c[r]; c[r] = zp[r]; }
        }
        release();  // plane ze only fed zp
        ++l;
    }
}

// ------------------------------------------------------------------ plain sweep
// JAC_F_NO_TMA: each thread reads its 7 neighbours from global memory (L1/L2 serve
// the reuse).  Tile 64 x 8 points, z-chunk of a.zc planes.
__global__ void __launch_bounds__(256) sweep_plain_kernel(const SweepArgs a)
{
    const Geom &g = a.g;
    int t = blockIdx.x;
    const int tx = t % a.ntx; t /= a.ntx;
    const int ty = t % a.nty; t /= a.nty;
    const int tz = t % a.ntz;
    const int b = t / a.ntz;
    const DevBlock &blk = a.blocks[b];
    const int i = tx * 64 + 2 * (threadIdx.x & 31);
    const int j = ty * 8 + (threadIdx.x >> 5);
    if (i >= g.ex || j >= g.ey) return;
    const int z0 = tz * a.zc, z1 = min(g.ez, z0 + a.zc);
    const double *s = a.arena + (int64_t)(a.src * g.nslots + blk.slot) * g.bstride;
    const int dst = 1 - a.src;
    for (int k = z0; k < z1; ++k) {
        const int64_t o = (int64_t)(k + 1) * g.Q + (int64_t)(j + 1) * g.P + g.A + i;
        const double2 cc = *reinterpret_cast<const double2 *>(s + o);
        const double xm = s[o - 1], xp = s[o + 2];
        const double2 ym = *reinterpret_cast<const double2 *>(s + o - g.P);
        const double2 yp = *reinterpret_cast<const double2 *>(s + o + g.P);
        const double2 zm = *reinterpret_cast<const double2 *>(s + o - g.Q);
        const double2 zp = *reinterpret_cast<const double2 *>(s + o + g.Q);
        double2 v;
        v.x = stencil7(cc.x, xm, cc.y, ym.x, yp.x, zm.x, zp.x);
        v.y = stencil7(cc.y, cc.x, xp, ym.y, yp.y, zm.y, zp.y);
        emit_pair(a, blk, dst, i, j, k, v);
    }
}

// ------------------------------------------------------------------ ghost fill
// One CTA row per (slot, face); grid.y strides over the face.  dst = the buffer the
// preceding sweep wrote (its ghosts are read by the next sweep).
__global__ void __launch_bounds__(256) ghost_fill_kernel(const SweepArgs a, int dst)
{
    const Geom &g = a.g;
    const int slot_face = blockIdx.x;
    const int b = slot_face / 6, f = slot_face % 6;
    const DevBlock &blk = a.blocks[b];
    const double *src = blk.nb_out[f];
    if (!src) return;
    double *base = a.arena + (int64_t)(dst * g.nslots + blk.slot) * g.bstride;
    const int d = f >> 1;
    const int64_t n = (d == 0) ? (int64_t)g.ey * g.ez : (d == 1) ? (int64_t)g.ex * g.ez : (int64_t)g.ex * g.ey;
    for (int64_t e = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.y * blockDim.x) {
        int64_t off;
        if (d == 0) {
            const int64_t k = e / g.ey, j = e % g.ey;
            off = (k + 1) * g.Q + (j + 1) * g.P + g.A + ((f == XM) ? -1 : g.ex);
        } else if (d == 1) {
            const int64_t k = e / g.ex, i = e % g.ex;
            off = (k + 1) * g.Q + ((f == YM) ? 0 : (int64_t)(g.ey + 1) * g.P) + g.A + i;
        } else {
            const int64_t j = e / g.ex, i = e % g.ex;
            off = ((f == ZM) ? 0 : (int64_t)(g.ez + 1) * g.Q) + (j + 1) * g.P + g.A + i;
        }
        base[off] = src[e];
    }
}

// ------------------------------------------------------------------ neighbour barrier
__global__ void barrier_kernel(const BarrierArgs ba)
{
    if (threadIdx.x != 0) return;
    __threadfence_system();  // the preceding phase's stores (incl. peer stores) first
    const uint64_t e = ba.ctrl[0] + 1;
    ba.ctrl[0] = e;
    for (int n = 0; n < ba.npeers; ++n)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(ba.peer_slot[n]), "l"(e) : "memory");
    for (int n = 0; n < ba.npeers; ++n) {
        const uint64_t *f = ba.ctrl + 1 + ba.peer_id[n];
        uint64_t v;
        const uint64_t t0 = globaltimer_ns();
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
            if (v >= e) break;
            if (globaltimer_ns() - t0 > kSpinLimitNs) __trap();
            __nanosleep(64);
        }
    }
    __threadfence_system();
}

// ------------------------------------------------------------------ R11 hash init
__device__ __forceinline__ double r11_value(uint64_t seed, uint64_t p)
{
    uint64_t z = (seed << 40) + p;
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * 0x1.0p-53;
}

__global__ void hash_init_kernel(const SweepArgs a, int64_t nx, int64_t ny, uint64_t seed)
{
    const Geom &g = a.g;
    const DevBlock &blk = a.blocks[blockIdx.y];
    const int64_t sx = g.ex + 2, sy = g.ey + 2;
    const int64_t n = sx * sy * (g.ez + 2);
    double *b0 = a.arena + (int64_t)blk.slot * g.bstride;
    double *b1 = a.arena + (int64_t)(g.nslots + blk.slot) * g.bstride;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ii = e % sx, jj = (e / sx) % sy, kk = e / (sx * sy);  // ghost-inclusive
        const uint64_t px = blk.org[0] + ii, py = blk.org[1] + jj, pz = blk.org[2] + kk;
        const uint64_t p = (pz * (uint64_t)(ny + 2) + py) * (uint64_t)(nx + 2) + px;
        const double v = r11_value(seed, p);
        const int64_t off = kk * g.Q + jj * g.P + (g.A - 1) + ii;
        b0[off] = v;
        b1[off] = v;
    }
}

// ------------------------------------------------------------------ host launchers
template <int BX, int BY, int NT, int NS>
static int resident_tma_t()
{
    static int resident = 0;  // SMs x CTAs per SM (per process; one device per process)
    if (!resident) {
        constexpr size_t smem = tma_smem_bytes(BX, BY, NS);
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_tma_kernel<BX, BY, NT, NS>, NT, smem);
        resident = std::max(1, sms * std::max(1, per_sm));
    }
    return resident;
}

template <int BX, int BY, int NT, int NS>
static cudaError_t launch_tma_t(const CUtensorMap &tm, const SweepArgs &a, cudaStream_t s)
{
    constexpr size_t smem = tma_smem_bytes(BX, BY, NS);
    // One CTA per item by default: the hardware launches CTAs in index order as slots
    // free up, which keeps x/y-adjacent tiles (and successive z-chunks of a column)
    // temporally close, so their shared halo planes are L2 hits.  A persistent grid
    // with static striding lets CTAs drift apart and turns halos into DRAM re-reads
    // (measured 359 -> 454 us per 512^3 sweep).  JAC_GRID=<n> caps the grid (tuning).
    static int grid_cap = -1;
    if (grid_cap < 0) {
        const char *e = getenv("JAC_GRID");
        grid_cap = e ? std::max(0, atoi(e)) : 0;
    }
    const int grid = grid_cap > 0 ? std::min(a.nitems, grid_cap) : a.nitems;
    sweep_tma_kernel<BX, BY, NT, NS><<<(unsigned)grid, NT, smem, s>>>(tm, a);
    return cudaGetLastError();
}

template <int BX, int BY, int NT, int NS>
static cudaError_t prepare_tma_t()
{
    constexpr size_t smem = tma_smem_bytes(BX, BY, NS);
    return cudaFuncSetAttribute(sweep_tma_kernel<BX, BY, NT, NS>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t prepare_sweep_tma(int variant)
{
    if (variant == TMA_NARROW) return prepare_tma_t<32, 16, 256, 4>();
    return prepare_tma_t<64, 16, 256, 4>();
}

int sweep_resident_ctas(int variant)
{
    if (variant == TMA_NARROW) return resident_tma_t<32, 16, 256, 4>();
    return resident_tma_t<64, 16, 256, 4>();
}

TileShape tma_tile_shape(int variant)
{
    if (variant == TMA_NARROW) return {32, 16};
    return {64, 16};
}

cudaError_t launch_sweep_tma(const CUtensorMap &tm, const SweepArgs &a, int variant, cudaStream_t s)
{
    if (variant == TMA_NARROW) return launch_tma_t<32, 16, 256, 4>(tm, a, s);
    return launch_tma_t<64, 16, 256, 4>(tm, a, s);
}

cudaError_t launch_sweep_plain(const SweepArgs &a, cudaStream_t s)
{
    const int64_t grid = (int64_t)a.g.nslots * a.ntx * a.nty * a.ntz;
    sweep_plain_kernel<<<(unsigned)grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_ghost_fill(const SweepArgs &a, int dst, cudaStream_t s)
{
    const int64_t maxface = std::max((int64_t)a.g.ey * a.g.ez,
                                     std::max((int64_t)a.g.ex * a.g.ez, (int64_t)a.g.ex * a.g.ey));
    const int64_t gy = std::min<int64_t>(64, (maxface + 255) / 256);
    ghost_fill_kernel<<<dim3((unsigned)(a.g.nslots * 6), (unsigned)gy), 256, 0, s>>>(a, dst);
    return cudaGetLastError();
}

cudaError_t launch_barrier(const BarrierArgs &ba, cudaStream_t s)
{
    barrier_kernel<<<1, 32, 0, s>>>(ba);
    return cudaGetLastError();
}

cudaError_t launch_hash_init(const SweepArgs &a, int64_t nx, int64_t ny, uint64_t seed, cudaStream_t s)
{
    hash_init_kernel<<<dim3(64, (unsigned)a.g.nslots), 256, 0, s>>>(a, nx, ny, seed);
    return cudaGetLastError();
}

}  // namespace jac
