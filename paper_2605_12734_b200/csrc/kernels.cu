// kernels.cu -- sm_100a kernels of the overdecomposed Jacobi3D hot path.
//
//  sweep_tma_kernel   north-star subsystem (2): ONE batched launch per GPU per
//                     iteration walks every local block through the descriptor
//                     table.  Each CTA owns one (block, BX x BY column tile, z-chunk)
//                     work item and marches it in z; z-planes (with the in-block
//                     x/y halo) are staged into a ring of shared-memory buffers by
//                     TMA (cp.async.bulk.tensor + mbarrier complete_tx), the
//                     block-edge x ghosts by a 1-D bulk copy into the same stage, the
//                     z-neighbours ride in registers.  The epilogue stores the new
//                     interior AND, for boundary layers, the same values straight into
//                     the neighbour block's ghost cells of the output buffer (fused
//                     pack + ghost copy; blocks on other GPUs are written over NVLink
//                     through IPC pointers), so ODF costs no extra launch or pass.
//  sweep_plain_kernel JAC_F_NO_TMA ablation: per-point global loads (L1/L2 reuse).
//  ghost_fill_kernel  north-star subsystem (3) as the JAC_F_UNFUSED_PACK path: the
//                     sweep packs faces into an outbox, this batched kernel copies
//                     every block's neighbour outboxes into its ghosts (PAPER.md:90
//                     pack/unpack kernels; PAPER.md:269 intra-process D2D copy).
//  barrier_kernel     cross-rank neighbour barrier on device flags (st.release.sys /
//                     ld.acquire.sys over NVLink), replacing the paper's IPC event
//                     pool.
//  xghost_extract_kernel / hash_init_kernel / stage_kernel<scatter|gather>
//                     cold-path init and host-transfer helpers.
//
// The update (PAPER.md:281 Jacobi, 3-D lift R1; readings R2-R4 in DESIGN.md):
//     u' = ((((((c + x-) + x+) + y-) + y+) + z-) + z+) * fl(1/7)
// computed with __dadd_rn/__dmul_rn (no contraction, no reassociation; built with
// -fmad=false), so every ODF and GPU count reproduces the oracle bit for bit.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

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

// ------------------------------------------------------------------ checked stores
// Production build: plain stores.  -DJAC_CHECKED (libjacobi3d_checked.so): every store
// is range- and alignment-checked against CheckArgs (device.hpp) and skipped on a
// violation, which is recorded with its source line and address.
#ifdef JAC_CHECKED
__device__ __noinline__ void check_fail(const CheckArgs &c, uint32_t code, int line, const void *p)
{
    if (!c.status) return;
    atomicOr(c.status, code);
    if (atomicCAS(c.status + 1, 0u, (unsigned)line) == 0u) {
        c.status[2] = (uint32_t)(uintptr_t)p;
        c.status[3] = (uint32_t)((unsigned long long)(uintptr_t)p >> 32);
    }
    __threadfence_system();
}
__device__ __noinline__ bool check_ptr(const CheckArgs &c, const void *p, int bytes, int line)
{
    const unsigned long long u = (unsigned long long)(uintptr_t)p;
    if (u % (unsigned)bytes) { check_fail(c, kStatusMisaligned, line, p); return false; }
    for (int r = 0; r < c.nranges; ++r)
        if (u >= c.ranges[r].lo && u + bytes <= c.ranges[r].hi) return true;
    check_fail(c, kStatusOutOfRange, line, p);
    return false;
}
#define JAC_OK_PTR(a, p, bytes) check_ptr((a).chk, (p), (bytes), __LINE__)
#define JAC_ASSERT(a, cond) do { if (!(cond)) check_fail((a).chk, kStatusAssert, __LINE__, nullptr); } while (0)
#else
#define JAC_OK_PTR(a, p, bytes) true
#define JAC_ASSERT(a, cond) ((void)0)
#endif
#define ST8(a, p, v) do { double *p_ = (p); if (JAC_OK_PTR(a, p_, 8)) *p_ = (v); } while (0)
#define ST16(a, p, v) do { double *p_ = (p); if (JAC_OK_PTR(a, p_, 16)) *reinterpret_cast<double2 *>(p_) = (v); } while (0)

__device__ __forceinline__ void st_pair(const SweepArgs &a, double *p, double2 v, bool both)
{
    if (both) ST16(a, p, v);
    else ST8(a, p, v.x);
}

// Does face f of `blk` have a store target in this sweep's mode (neighbour ghosts of
// output buffer dst in the fused mode, the outbox in the pack mode)?
__device__ __forceinline__ bool has_target(const SweepArgs &a, const DevBlock &blk, int dst, int f)
{
    return (a.mode == MODE_FUSED ? blk.nb[f][dst] : blk.nb[f][0]) != nullptr;
}

// Stores the new values of points (i, j, k) and (i+1, j, k) of block `blk` into the
// output buffer `dst` (own_plane = the block's output array + (k+1)*Q, rowoff =
// (j+1)*P + A + i), plus the face traffic of the chosen mode.  Caller guarantees
// j < ey and 0 <= k < ez; i may be past the ragged x edge.  `blk` should live in
// shared memory or registers: global stores would otherwise force the compiler to
// re-load it after every store.
template <bool HAS_Z = true>
__device__ __forceinline__ void emit_pair(const SweepArgs &a, const DevBlock &blk, int dst, double *own_plane,
                                          int64_t rowoff, int i, int j, int k, double2 v)
{
    const Geom &g = a.g;
    if (i >= g.ex) return;
    const bool both = (i + 1) < g.ex;
    st_pair(a, own_plane + rowoff, v, both);
    if (a.mode == MODE_NOEXCHANGE) return;
    const bool zface = HAS_Z && ((k == 0) || (k == g.ez - 1));
    const bool yface = (j == 0) || (j == g.ey - 1);
    const bool last_x = (i == g.ex - 1) || (both && i + 1 == g.ex - 1);
    const bool xface = (i == 0) || last_x;
    if (!(zface || yface || xface)) return;  // interior point: done
    const double last_v = (i == g.ex - 1) ? v.x : v.y;
    const int64_t xgi = (int64_t)k * g.eyp + j;
    if (a.mode == MODE_FUSED) {
        // direct-to-ghost: the neighbour's ghost layer of the OUTPUT buffer is not
        // read by anyone during this sweep, so writing it here is race-free.
        // (pack_mask faces -- JAC_F_NCCL -- go to a contiguous send buffer instead.)
        auto packed = [&](double *p, int64_t idx) { ST8(a, p + idx, v.x); if (both) ST8(a, p + idx + 1, v.y); };
        if (zface) {
            if (k == 0) {
                double *p = blk.nb[ZM][dst];
                if (p) {
                    if (blk.pack_mask & (1u << ZM)) packed(p, (int64_t)j * g.ex + i);
                    else st_pair(a, p + (int64_t)(g.ez + 1) * g.Q + rowoff, v, both);
                }
            }
            if (k == g.ez - 1) {
                double *p = blk.nb[ZP][dst];
                if (p) {
                    if (blk.pack_mask & (1u << ZP)) packed(p, (int64_t)j * g.ex + i);
                    else st_pair(a, p + rowoff, v, both);
                }
            }
        }
        if (yface) {
            if (j == 0) {
                double *p = blk.nb[YM][dst];
                if (p) {
                    if (blk.pack_mask & (1u << YM)) packed(p, (int64_t)k * g.ex + i);
                    else st_pair(a, p + (int64_t)(k + g.zg) * g.Q + (int64_t)(g.ey + 1) * g.P + g.A + i, v, both);
                }
            }
            if (j == g.ey - 1) {
                double *p = blk.nb[YP][dst];
                if (p) {
                    if (blk.pack_mask & (1u << YP)) packed(p, (int64_t)k * g.ex + i);
                    else st_pair(a, p + (int64_t)(k + g.zg) * g.Q + g.A + i, v, both);
                }
            }
        }
        // x faces: into the neighbour's contiguous x-ghost array; the 16 rows of a
        // tile write one 128-byte run per plane (merged in L2 into full sectors).
        if (i == 0) {
            double *p = blk.nb[XM][dst];
            if (p) ST8(a, p + xgi, v.x);
        }
        if (last_x) {
            double *p = blk.nb[XP][dst];
            if (p) ST8(a, p + xgi, last_v);
        }
    } else {  // MODE_PACK: contiguous outbox faces, layouts x:[k][j] y:[k][i] z:[j][i]
        double *ob = a.outbox + (int64_t)blk.slot * g.ostride;
        if (k == 0 && blk.nb[ZM][0]) {
            double *p = ob + g.ooff[ZM] + (int64_t)j * g.ex + i;
            ST8(a, p, v.x); if (both) ST8(a, p + 1, v.y);
        }
        if (k == g.ez - 1 && blk.nb[ZP][0]) {
            double *p = ob + g.ooff[ZP] + (int64_t)j * g.ex + i;
            ST8(a, p, v.x); if (both) ST8(a, p + 1, v.y);
        }
        if (j == 0 && blk.nb[YM][0]) {
            double *p = ob + g.ooff[YM] + (int64_t)k * g.ex + i;
            ST8(a, p, v.x); if (both) ST8(a, p + 1, v.y);
        }
        if (j == g.ey - 1 && blk.nb[YP][0]) {
            double *p = ob + g.ooff[YP] + (int64_t)k * g.ex + i;
            ST8(a, p, v.x); if (both) ST8(a, p + 1, v.y);
        }
        if (i == 0 && blk.nb[XM][0]) ST8(a, ob + g.ooff[XM] + (int64_t)k * g.ey + j, v.x);
        if (last_x && blk.nb[XP][0]) ST8(a, ob + g.ooff[XP] + (int64_t)k * g.ey + j, last_v);
    }
}

// ------------------------------------------------------------------ programmatic dependent launch
// Sweeps are launched with programmatic stream serialization: every CTA lets the
// next sweep be scheduled early (its CTAs fill SMs freed during this sweep's last
// wave) and then waits, before touching any buffer, until the previous grid has
// completed and its memory is visible.  Only the read-only descriptor table and the
// kernel parameters are read before the wait, so the result is that of serialized
// launches.  Without the launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_launch_dependents_then_wait()
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Kernel span on the device clock for jac_profile_sweep (a.span set): first CTA start
// after the dependency wait, last CTA end -- under programmatic dependent launch,
// where event-record nodes between sweeps would break the launch overlap.
__device__ __forceinline__ void span_begin(unsigned long long *span)
{
    if (span && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMin(&span[0], t);
    }
}
__device__ __forceinline__ void span_end(unsigned long long *span)
{
    if (span) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            atomicMax(&span[1], t);
        }
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

// Watchdog of the shared-memory ring: a TMA that never lands (a kernel bug, not a
// timing condition) traps after ~kSpinLimitNs instead of hanging the GPU.  Waits on
// other partitions use the softer, configurable Watchdog of device.hpp instead.
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
#ifdef JAC_MBAR_HINT  // experiment build: an explicit suspend-time hint (ns) for the wait
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(b), "r"(parity), "n"(JAC_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
#endif
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

__device__ __forceinline__ void mbar_expect(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_box(const CUtensorMap *tm, double *dst, uint64_t *bar, int c0, int c1,
                                        int c2, int c3)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_copy(double *dst, const double *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Ring stage: the W x (BY+2) staged plane, then 2 x BY x-ghost values (side 0, 1).
template <int BX, int BY, int W>
struct StageLayout {
    static constexpr int H = BY + 2;
    static constexpr uint32_t BOX_BYTES = W * H * sizeof(double);
    static constexpr int XG_OFF = W * H;  // doubles; 16-byte aligned since W*H is even
    static constexpr uint32_t XG_BYTES = BY * sizeof(double);
    static constexpr int STRIDE = ((W * H + 2 * BY) + 15) / 16 * 16;  // 128-byte aligned stages
};

constexpr size_t tma_smem_bytes(int BX, int BY, int W, int NS)
{
    return (size_t)NS * (((W * (BY + 2) + 2 * BY) + 15) / 16 * 16) * sizeof(double) + NS * sizeof(uint64_t);
}

template <int BX, int BY>
__device__ __forceinline__ TileItem decode_item(const SweepArgs &a, int item)
{
    return decode_item3d(a, item, BX, BY);
}

// ---- fused cross-partition ordering (see SweepArgs, PartSync) -------------------
// Spins until every neighbour partition of `ps` has stored an epoch >= e into its flag
// word here.  Watchdog: after wd.spin_limit_ns it records kStatusPeerTimeout in the
// mapped host status word and gives up (the engine turns that into JAC_ECUDA) instead
// of trapping, so a skewed or dead peer does not poison this CUDA context.
__device__ __forceinline__ void wait_flags(const PartSync &ps, uint64_t e, const Watchdog &wd)
{
    for (int n = 0; n < ps.npeers; ++n) {
        const uint64_t *f = ps.ctrl + 1 + ps.peer_id[n];
        uint64_t v;
        const uint64_t t0 = globaltimer_ns();
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
            if (v >= e) break;
            if (wd.spin_limit_ns && globaltimer_ns() - t0 > wd.spin_limit_ns) {
                if (wd.status) {
                    *reinterpret_cast<volatile uint32_t *>(wd.status) = kStatusPeerTimeout;
                    __threadfence_system();
                }
                return;
            }
            __nanosleep(100);
        }
    }
    // The peers' ghost stores were generic-proxy writes; this CTA reads them next with
    // TMA / bulk copies (async proxy).  The acquire orders them for the generic proxy;
    // this fence extends the order to the async proxy (PTX memory model, proxies).
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Thread 0 of a remote-touching item, before its first staging copy: wait for the
// neighbours' signal of the phase this partition completed last.
__device__ __forceinline__ void wait_peers(const SweepArgs &a, const PartSync &ps)
{
    const uint64_t e = *reinterpret_cast<volatile const uint64_t *>(ps.ctrl);  // phases completed here
    wait_flags(ps, e, a.wd);
}

// wait_peers, timed under jac_profile_sweep: span[2] += wait ns, span[3] = max(wait ns)
__device__ __forceinline__ void timed_wait_peers(const SweepArgs &a, const PartSync &ps)
{
    if (!a.span) {
        wait_peers(a, ps);
        return;
    }
    const uint64_t w0 = globaltimer_ns();
    wait_peers(a, ps);
    const unsigned long long w = globaltimer_ns() - w0;
    atomicAdd(&a.span[2], w);
    atomicMax(&a.span[3], w);
}

// All threads of a remote-touching item: after the CTA's last store.  The last such
// CTA of its partition in this launch bumps the partition's epoch and releases it to
// every neighbour partition.
__device__ __forceinline__ void signal_done(const PartSync &ps, int32_t exp_bits = 0)
{
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (!(exp_bits & kExpNoCtaSysFence))
        __threadfence_system();  // this CTA's stores (peer stores included) before the count
    if (atomicAdd(ps.count, 1ull) == (unsigned long long)ps.nremote - 1) {
        *reinterpret_cast<volatile unsigned long long *>(ps.count) = 0;
        __threadfence_system();
        const uint64_t e = ps.ctrl[0] + 1;
        *reinterpret_cast<volatile uint64_t *>(ps.ctrl) = e;
        for (int n = 0; n < ps.npeers; ++n)
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(ps.peer_slot[n]), "l"(e) : "memory");
    }
}

// Copies a block descriptor into shared memory, 16 bytes per thread (threads 0..10).
// The caller's first __syncthreads publishes it.
static_assert(sizeof(DevBlock) % 16 == 0, "DevBlock is copied in 16-byte pieces");
__device__ __forceinline__ void load_descriptor(DevBlock *dst, const DevBlock *src)
{
    constexpr int kPieces = (int)(sizeof(DevBlock) / 16);
    if ((int)threadIdx.x < kPieces)
        reinterpret_cast<int4 *>(dst)[threadIdx.x] = __ldg(reinterpret_cast<const int4 *>(src) + threadIdx.x);
}

// Staged column of the tile's first point i = x0.  Interior tiles stage x0-2 ..
// x0+BX+1 (soff = 2).  The box never reads the inline x-ghost sectors (x ghosts come
// from the x-ghost arrays): the first tile starts at the interior (soff = 0) and the
// last tile is pulled back by two columns (soff = 4) so a full last tile ends exactly
// at the interior's end.  W == BX (single-tile blocks) stages the interior only.
template <int BX, int W>
__device__ __forceinline__ int tile_soff(const Geom &g, int x0)
{
    if (W == BX || x0 == 0) return 0;
    return (x0 + BX >= g.ex) ? 4 : 2;
}

// Persistent-free TMA z-march: one CTA per work item.  BX x BY column tile, NT
// threads, NS-deep plane ring, staged width W (BX + 4 with in-block x halo, or BX
// for single-tile blocks).  Each thread owns a pair of x-points (double2) in RY rows.
constexpr int min_ctas_per_sm(int NT, int NS, int BX = 64, int BY = 16)
{
    // 64 x 32 tiles (4 rows per thread) need > 80 registers: 2 CTAs per SM
    return (BX >= 64 && BY >= 32) ? 2 : NT >= 512 ? 2 : NT <= 128 ? 8 : (NS >= 8 ? 2 : (NS >= 6 ? 3 : 4));
}

template <int BX, int BY, int W, int NT, int NS>
__global__ void __launch_bounds__(NT, min_ctas_per_sm(NT, NS, BX, BY))
    sweep_tma_kernel(const __grid_constant__ CUtensorMap tmap, const SweepArgs a)
{
    using L = StageLayout<BX, BY, W>;
    constexpr int TXL = BX / 2;    // threads along x
    constexpr int NRG = NT / TXL;  // row groups
    constexpr int RY = BY / NRG;   // rows per thread
    static_assert(RY >= 1 && RY * NRG == BY, "tile shape");
    static_assert(W == BX || W == BX + 4, "staged width");
    static_assert(NS >= 3, "ring must hold planes k, k+1 and prefetch");
    // A ring of NSL = NS stages with NS - 1 planes in flight: the refill after plane q
    // overwrites the stage of plane q-1, whose values were all consumed (in registers)
    // one plane earlier -- see refill below.
    constexpr int NSL = NS;
    constexpr int NIF = NS - 1;  // planes in flight

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stage = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + NSL * L::STRIDE * sizeof(double));

    const Geom &g = a.g;
    const int code = a.item_map ? a.item_map[blockIdx.x] : (int)blockIdx.x;  // ~item: remote-touching
    const TileItem t = decode_item<BX, BY>(a, code < 0 ? ~code : code);
    const bool remote = a.fused_sync && code < 0;
    // The work list enumerates the table's slots in order, so the staging copies need
    // no descriptor: thread 0 issues them without waiting for the table read.  The
    // descriptor (store targets, for the epilogue) is copied to shared memory 16 bytes
    // per thread in parallel (a measured 12% of the small-block sweep's stall samples
    // sat at the prologue barrier while thread 0 serially read it first).
    const int slot = a.slot_base + t.b;
    __shared__ __align__(16) DevBlock blk;
    load_descriptor(&blk, a.blocks + t.b);
    pdl_launch_dependents_then_wait();
    span_begin(a.span);
    const int soff = tile_soff<BX, W>(g, t.x0);  // staged column of point i = x0 (0, 2 or 4)
    const int c0 = g.A + t.x0 - soff;
    const bool xlo = (t.x0 == 0);                 // tile touches the x- block face
    const bool xhi = (t.x0 + BX >= g.ex);         // tile touches the x+ block face
    const int nq = t.ze - t.zs + 2;               // planes zs-1 .. ze
    // producer-only state (thread 0): source block coordinates for TMA / bulk copies
    int c3 = 0;
    const double *xg0 = nullptr, *xg1 = nullptr;

    // plane q of the item = interior plane k = zs - 1 + q; x-ghosts only for k in [zs, ze)
    auto issue = [&](int q) {
        double *st = stage + (q % NSL) * L::STRIDE;
        uint64_t *bar = &bars[q % NSL];
        const bool mid = (q >= 1) && (q <= nq - 2);
        const uint32_t bytes = L::BOX_BYTES + (mid ? ((xlo ? L::XG_BYTES : 0) + (xhi ? L::XG_BYTES : 0)) : 0);
        JAC_ASSERT(a, c0 >= 0 && c0 < g.P && t.y0 >= 0 && t.y0 < g.ey && t.zs + q >= 0 &&
                          t.zs + q < g.ez + 2 * g.zg && c3 >= 0 && c3 < 2 * g.nslots && q < nq);
        mbar_expect(bar, bytes);
        tma_box(&tmap, st, bar, c0, t.y0, t.zs + q, c3);
        if (mid) {
            const int64_t ko = (int64_t)(t.zs - 1 + q) * g.eyp;
            JAC_ASSERT(a, ko + t.y0 + BY <= g.xgstride);
            if (xlo) bulk_copy(st + L::XG_OFF, xg0 + ko, L::XG_BYTES, bar);
            if (xhi) bulk_copy(st + L::XG_OFF + BY, xg1 + ko, L::XG_BYTES, bar);
        }
    };

    if (threadIdx.x == 0) {
        if (remote) timed_wait_peers(a, a.sync[a.blocks[t.b].part]);
        c3 = a.src * g.nslots + slot;
        xg0 = xg_array(a.xg, g, a.src, slot, 0) + t.y0;
        xg1 = xg_array(a.xg, g, a.src, slot, 1) + t.y0;
        for (int s = 0; s < NSL; ++s) mbar_init(&bars[s], 1);  // producer arrive + TMA bytes
        mbar_fence_init();
        for (int q = 0; q < NIF && q < nq; ++q) issue(q);
    }
    __syncthreads();

    const int lane = threadIdx.x % TXL;
    const int rg = threadIdx.x / TXL;
    const int col = soff + 2 * lane;  // staged column of point i = x0 + 2*lane
    const int i = t.x0 + 2 * lane;
    const int dst = 1 - a.src;
    const bool ilo = (i == 0);                     // element 0 is the first interior point
    const bool ihi0 = (i == g.ex - 1);             // element 0 is the last interior point
    const bool ihi1 = (i + 1 == g.ex - 1);         // element 1 is the last interior point
    const int jl0 = rg * RY;                       // tile row of this thread's row 0
    const int sb = (jl0 + 1) * W + col;            // stage index of (row 0, element 0)
    const int xg = L::XG_OFF + jl0;                // stage index of row 0's x- ghost (+BY: x+)
    double *const own = a.arena + (int64_t)(dst * g.nslots + blk.slot) * g.bstride;  // (slot here spills at 64 regs)
    auto plane = [&](int q) { return stage + (q % NSL) * L::STRIDE; };
    auto wait = [&](int q) { mbar_wait(&bars[q % NSL], (q / NSL) & 1); };
    // Plane q is done -> the producer issues plane q + NIF into the stage of plane q-1.
    // A stage may be overwritten only once every value read from it has reached
    // registers: the barrier orders the threads' shared-memory loads before the refill,
    // but a load whose result is not yet used can still be in flight when the TMA (async
    // proxy) overwrites the stage.  Plane q-1's loads were all consumed by the stencil of
    // plane q-1 or q -- including plane 0's, which only feed zm for plane 1 -- whereas
    // plane q's own stage may still hold values in flight.  (The first version refilled
    // plane q's stage, and plane 0's straight after loading zm: a rare write-after-read
    // race -- a few stale 32-point row segments in one run out of dozens, and in every run
    // of a build whose scheduling delayed those loads.)  (Per-warp "empty" mbarriers
    // instead of this CTA barrier were measured: no robust gain, and slower for the
    // small-block tiles.)
    auto refill = [&](int q) {
        __syncthreads();
        if (threadIdx.x == 0 && q + NIF < nq) issue(q + NIF);
    };

    double2 zm[RY], c[RY], zp[RY];
    wait(0);
#pragma unroll
    for (int r = 0; r < RY; ++r) zm[r] = *reinterpret_cast<const double2 *>(plane(0) + sb + r * W);
    refill(0);  // plane NIF into the spare stage (plane -1's): plane 0's stage stays intact
    wait(1);
#pragma unroll
    for (int r = 0; r < RY; ++r) c[r] = *reinterpret_cast<const double2 *>(plane(1) + sb + r * W);

    // One z-plane of the march: wait for plane q+1, update centre plane q (k), store.
    auto update = [&](int q, double2 (&v)[RY]) {
        wait(q + 1);
        const double *Sn = plane(q + 1);
#pragma unroll
        for (int r = 0; r < RY; ++r) zp[r] = *reinterpret_cast<const double2 *>(Sn + sb + r * W);
        const double *S = plane(q);
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            const double xm = ilo ? S[xg + r] : S[sb + r * W - 1];
            const double xp1 = ihi1 ? S[xg + BY + r] : S[sb + r * W + 2];
            const double xp0 = ihi0 ? S[xg + BY + r] : c[r].y;
            const double2 ym = (r == 0) ? *reinterpret_cast<const double2 *>(S + sb - W) : c[r - 1];
            const double2 yp = (r == RY - 1) ? *reinterpret_cast<const double2 *>(S + sb + RY * W) : c[r + 1];
            v[r].x = stencil7(c[r].x, xm, xp0, ym.x, yp.x, zm[r].x, zp[r].x);
            v[r].y = stencil7(c[r].y, c[r].x, xp1, ym.y, yp.y, zm[r].y, zp[r].y);
        }
    };
    auto advance = [&](int q) {
        refill(q);  // centre plane k is done
#pragma unroll
        for (int r = 0; r < RY; ++r) { zm[r] = c[r]; c[r] = zp[r]; }
    };
    // General plane: every store through emit_pair (ragged edges, y faces, z faces,
    // every exchange mode).
    auto plane_general = [&](int q) {
        const int k = t.zs - 1 + q;
        double2 v[RY];
        update(q, v);
        double *const own_k = own + (int64_t)(k + 1) * g.Q;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            const int j = t.y0 + jl0 + r;
            if (j < g.ey) emit_pair(a, blk, dst, own_k, (int64_t)(j + 1) * g.P + g.A + i, i, j, k, v[r]);
        }
        advance(q);
    };

    // Lean planes (the z-march is issue-bound once the power cap lowers the clock, so
    // instructions per point count): a CTA-uniform choice for full tiles -- every lane
    // holds two interior points, every row is interior -- away from the block's
    // first and last plane.  They store the pair with one 16-byte
    // store, x-face lanes the boundary value into the neighbour's x-ghost array (or
    // outbox), element (j, k) at xf + k*xs + j, and y-face rows the pair into the
    // neighbour's ghost row (or send buffer / outbox) at yf + k*ys.  XE = edge tile
    // (x-ghost reads, face stores); interior tiles address every operand as one
    // per-plane base + immediate.  The loop is unrolled by 3 with rotated register
    // names (no moves), and the ring slot / parity advance incrementally.
    const bool exch = (a.mode != MODE_NOEXCHANGE);
    const bool lean = (t.x0 + BX <= g.ex) && (t.y0 + BY <= g.ey) && g.ex > 2;
    int q = 1;
    const int qlast = nq - 2;
    if (exch && t.zs == 0) plane_general(q++);  // z- face plane
    const int qlean_end = (exch && t.ze == g.ez) ? qlast - 1 : qlast;
    if (lean && q <= qlean_end) {
        // edge instantiation: x-ghost lanes, or a y-face row with a target
        auto has = [&](int f) { return has_target(a, blk, dst, f); };
        const bool edge = (t.x0 == 0) || (t.x0 + BX >= g.ex) ||
                          (exch && ((t.y0 == 0 && has(YM)) || (t.y0 + BY >= g.ey && has(YP))));
        // x faces: the face lanes (first / last lane of every row group) put their values
        // in shared memory; after the plane's barrier the first BY threads store each
        // side's BY rows, two per thread, as one contiguous run per instruction (full
        // 32-byte sectors: over NVLink a partly written sector travels as its own
        // transfer -- the face lanes storing their own rows sent 1.75x the face bytes).
        auto xtarget = [&](int f, int64_t &stride) -> double * {
            double *p = nullptr;
            stride = 0;
            if (a.mode == MODE_FUSED) {
                p = blk.nb[f][dst];
                stride = g.eyp;
            } else if (blk.nb[f][0]) {
                p = a.outbox + (int64_t)slot * g.ostride + g.ooff[f];
                stride = g.ey;
            }
            return p;
        };
        int64_t xs = 0;
        const bool xput = exch && (ilo || ihi1) && xtarget(ilo ? XM : XP, xs) != nullptr;  // holds face values
        const int xside = ilo ? 0 : 1;
        double *xf = nullptr;  // this thread's store target (threads < BY): rows 2l, 2l+1 of one side
        if (exch && (int)threadIdx.x < BY) {
            const int side = (int)threadIdx.x / (BY / 2);
            if (side == 0 ? t.x0 == 0 : t.x0 + BX >= g.ex) {
                xf = xtarget(side ? XP : XM, xs);
                if (xf) xf += t.y0 + 2 * ((int)threadIdx.x % (BY / 2)) + (int64_t)(t.zs - 1 + q) * xs;
            }
        }
        // y-face target of this thread (row 0 if yf_lo, else row RY-1; a full tile has
        // ey >= BY, so no thread holds both): the neighbour's ghost row (plane stride
        // Q), or a packed send buffer / outbox row [k][ex] (stride ex).
        double *yf = nullptr;
        int64_t ys = 0;
        bool yf_lo = false;
        if (exch) {
            int f = -1;
            if (t.y0 + jl0 == 0) { f = YM; yf_lo = true; }
            else if (t.y0 + jl0 + RY - 1 == g.ey - 1) f = YP;
            if (f >= 0) {
                if (a.mode == MODE_FUSED) {
                    if (double *p = blk.nb[f][dst]) {
                        if (blk.pack_mask & (1u << f)) { yf = p + i; ys = g.ex; }
                        else {
                            yf = p + (int64_t)g.zg * g.Q + (f == YM ? (int64_t)(g.ey + 1) * g.P : 0) + g.A + i;
                            ys = g.Q;
                        }
                    }
                } else if (blk.nb[f][0]) {
                    yf = a.outbox + (int64_t)slot * g.ostride + g.ooff[f] + i;
                    ys = g.ex;
                }
                if (yf) yf += (int64_t)(t.zs - 1 + q) * ys;
            }
        }
        const bool yv = (ys & 1) == 0;  // y-face rows 16-byte aligned (ghost rows; packed, even ex)
        const bool xv2 = (xs & 1) == 0;  // x-face row pairs 16-byte aligned (pitch eyp; outbox: even ey)
        __shared__ __align__(16) double xface[2][2][BY];  // [plane parity][side][row]
        double *op = own + (int64_t)(t.zs + q) * g.Q + (int64_t)(t.y0 + jl0 + 1) * g.P + g.A + i;
        const int64_t P = g.P, Qs = g.Q;
        int sn = (q + 1) % NSL;               // ring slot of plane q+1
        uint32_t pn = ((q + 1) / NSL) & 1u;   // its mbarrier parity
        const double *Sc = plane(q);
        auto step = [&](const bool XE, const double2 (&A)[RY], const double2 (&B)[RY], double2 (&C)[RY]) {
            mbar_wait(&bars[sn], pn);
            const double *Sn = stage + sn * L::STRIDE;
            const double *Sb = Sc + sb;
#pragma unroll
            for (int r = 0; r < RY; ++r) C[r] = *reinterpret_cast<const double2 *>(Sn + sb + r * W);
#pragma unroll
            for (int r = 0; r < RY; ++r) {
                double xm = Sb[r * W - 1], xp1 = Sb[r * W + 2];
                if (XE) {
                    if (ilo) xm = Sc[xg + r];
                    if (ihi1) xp1 = Sc[xg + BY + r];
                }
                const double2 ym = (r == 0) ? *reinterpret_cast<const double2 *>(Sb - W) : B[r - 1];
                const double2 yp = (r == RY - 1) ? *reinterpret_cast<const double2 *>(Sb + RY * W) : B[r + 1];
                double2 v;
                v.x = stencil7(B[r].x, xm, B[r].y, ym.x, yp.x, A[r].x, C[r].x);
                v.y = stencil7(B[r].y, B[r].x, xp1, ym.y, yp.y, A[r].y, C[r].y);
                ST16(a, op + r * P, v);
                if (XE && xput) xface[q & 1][xside][jl0 + r] = ilo ? v.x : v.y;
                if (XE && yf && ((r == 0 && yf_lo) || (r == RY - 1 && !yf_lo))) {
                    // one 16-byte store (NVLink sends a half-written 32-byte sector as its own
                    // transfer); packed rows of odd width ex are only 8-byte aligned
                    if (yv) ST16(a, yf, v);
                    else { ST8(a, yf, v.x); ST8(a, yf + 1, v.y); }
                }
            }
            op += Qs;
            if (XE && yf) yf += ys;
            refill(q);  // centre plane done; its x-face values are in shared memory
            if (XE && xf) {
                const double2 pv = *reinterpret_cast<const double2 *>(
                    &xface[q & 1][(int)threadIdx.x / (BY / 2)][2 * ((int)threadIdx.x % (BY / 2))]);
                if (xv2) ST16(a, xf, pv);
                else { ST8(a, xf, pv.x); ST8(a, xf + 1, pv.y); }
                xf += xs;
            }
            ++q;
            Sc = Sn;
            if (++sn == NSL) { sn = 0; pn ^= 1u; }
        };
        auto run = [&](const bool xe) {
            while (q + 2 <= qlean_end) {
                step(xe, zm, c, zp);
                step(xe, c, zp, zm);
                step(xe, zp, zm, c);
            }
            if (q <= qlean_end) {  // 1 or 2 more planes; restore the canonical names
                step(xe, zm, c, zp);
                if (q <= qlean_end) {
                    step(xe, c, zp, zm);
#pragma unroll
                    for (int r = 0; r < RY; ++r) { const double2 t0 = zm[r]; zm[r] = zp[r]; zp[r] = c[r]; c[r] = t0; }
                } else {
#pragma unroll
                    for (int r = 0; r < RY; ++r) { const double2 t0 = zm[r]; zm[r] = c[r]; c[r] = zp[r]; zp[r] = t0; }
                }
            }
        };
        if (edge) run(true);
        else run(false);
    } else {
        for (; q <= qlean_end; ++q) plane_general(q);
    }
    if (q <= qlast) plane_general(q);  // z+ face plane
    if (remote) signal_done(a.sync[blk.part], a.exp_bits);
    span_end(a.span);
}

// ------------------------------------------------------------------ Jacobi2D sweep
// NEXT-1 (JAC_F_2D): u' = ((((c + x-) + x+) + y-) + y+) * fl(1/5) on one plane.
// Work item = (block, 64-wide x tile, chunk of 16-row y tiles), x tile fastest.  The
// CTA marches its chunk in y: one staged box per y tile (rows y0-1 .. y0+16, i.e. the
// y halo or the block's ghost rows, plus the in-block x halo), the block-edge x ghosts
// by bulk copy, a 4-deep TMA ring of tiles in flight.  Same fused direct-to-ghost
// epilogue as the 3-D sweep (no z faces).
__device__ __forceinline__ double stencil5(double c, double xm, double xp, double ym, double yp)
{
    constexpr double K5 = 0x1.999999999999ap-3;  // fl(1/5)
    double s = __dadd_rn(c, xm);
    s = __dadd_rn(s, xp);
    s = __dadd_rn(s, ym);
    s = __dadd_rn(s, yp);
    return __dmul_rn(s, K5);
}

template <int BX, int BY, int W, int NT, int NS>
__global__ void __launch_bounds__(NT, 4) sweep2d_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                            const SweepArgs a)
{
    using L = StageLayout<BX, BY, W>;
    constexpr int TXL = BX / 2;
    constexpr int NRG = NT / TXL;
    constexpr int RY = BY / NRG;
    static_assert(RY >= 1 && RY * NRG == BY, "tile shape");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stage = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + NS * L::STRIDE * sizeof(double));

    const Geom &g = a.g;
    const int code = a.item_map ? a.item_map[blockIdx.x] : (int)blockIdx.x;  // ~item: remote-touching
    const TileItem t = decode_item2d(a, code < 0 ? ~code : code, BX, BY);
    const bool remote = a.fused_sync && code < 0;
    const int b = t.b;
    const int slot = a.slot_base + b;  // see the 3-D sweep
    const int ty0 = t.zs;
    const int nq = max(0, t.ze - t.zs);
    const int x0 = t.x0;
    __shared__ __align__(16) DevBlock blk;
    load_descriptor(&blk, a.blocks + b);
    pdl_launch_dependents_then_wait();
    span_begin(a.span);
    const int soff = tile_soff<BX, W>(g, x0);
    const int c0 = g.A + x0 - soff;
    const bool xlo = (x0 == 0), xhi = (x0 + BX >= g.ex);
    int c3 = 0;
    const double *xg0 = nullptr, *xg1 = nullptr;
    auto issue = [&](int q) {
        double *st = stage + (q % NS) * L::STRIDE;
        uint64_t *bar = &bars[q % NS];
        const int y0 = (ty0 + q) * BY;
        JAC_ASSERT(a, c0 >= 0 && c0 < g.P && y0 >= 0 && y0 < g.ey && c3 >= 0 && c3 < 2 * g.nslots &&
                          y0 + BY <= g.xgstride);
        mbar_expect(bar, L::BOX_BYTES + (xlo ? L::XG_BYTES : 0) + (xhi ? L::XG_BYTES : 0));
        tma_box(&tmap, st, bar, c0, y0, 0, c3);
        if (xlo) bulk_copy(st + L::XG_OFF, xg0 + y0, L::XG_BYTES, bar);
        if (xhi) bulk_copy(st + L::XG_OFF + BY, xg1 + y0, L::XG_BYTES, bar);
    };
    if (threadIdx.x == 0) {
        if (remote) timed_wait_peers(a, a.sync[a.blocks[b].part]);
        c3 = a.src * g.nslots + slot;
        xg0 = xg_array(a.xg, g, a.src, slot, 0);
        xg1 = xg_array(a.xg, g, a.src, slot, 1);
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
        mbar_fence_init();
        for (int q = 0; q < NS && q < nq; ++q) issue(q);
    }
    __syncthreads();

    const int lane = threadIdx.x % TXL;
    const int rg = threadIdx.x / TXL;
    const int col = soff + 2 * lane;
    const int i = x0 + 2 * lane;
    const int dst = 1 - a.src;
    const bool ilo = (i == 0), ihi0 = (i == g.ex - 1), ihi1 = (i + 1 == g.ex - 1);
    double *own = a.arena + (int64_t)(dst * g.nslots + slot) * g.bstride;  // plane k = 0 (zg = 0)
    // Lean y tiles (as in the 3-D sweep): full in x and y, no y-face row -> one 16-byte
    // store per pair (+ the x-face value on x-edge lanes), rows shared between a
    // thread's RY rows instead of reloaded.  Other tiles take emit_pair.
    const bool exch = (a.mode != MODE_NOEXCHANGE);
    auto has = [&](int f) { return has_target(a, blk, dst, f); };
    const bool xfull = (x0 + BX <= g.ex) && g.ex > 2;
    const bool xedge = xlo || xhi;
    const bool ym_face = exch && has(YM), yp_face = exch && has(YP);  // loop-invariant
    const int jl0 = rg * RY;
    const int sb = (jl0 + 1) * W + col;
    const int xg = L::XG_OFF + jl0;
    // x faces as in the 3-D sweep: the face lanes put their values in shared memory, and
    // after the tile's barrier the first BY threads store each side's rows, two per
    // thread, as one contiguous run per instruction.
    auto xtarget = [&](int f) -> double * {  // element j at p + j (plane k = 0)
        if (a.mode == MODE_FUSED) return blk.nb[f][dst];
        return blk.nb[f][0] ? a.outbox + (int64_t)slot * g.ostride + g.ooff[f] : nullptr;
    };
    const bool xput = xfull && exch && (ilo || ihi1) && xtarget(ilo ? XM : XP) != nullptr;
    const int xside = ilo ? 0 : 1;
    double *xst = nullptr;  // threads < BY: rows 2l, 2l+1 of one side
    if (xfull && exch && (int)threadIdx.x < BY) {
        const int side = (int)threadIdx.x / (BY / 2);
        if (side == 0 ? xlo : xhi) {
            xst = xtarget(side ? XP : XM);
            if (xst) xst += 2 * ((int)threadIdx.x % (BY / 2));
        }
    }
    __shared__ __align__(16) double xface[2][2][BY];  // [tile parity][side][row]
    // general y tile: every store through emit_pair
    auto tile_general = [&](int q) {
        mbar_wait(&bars[q % NS], (q / NS) & 1);
        const double *S = stage + (q % NS) * L::STRIDE;
        const int y0 = (ty0 + q) * BY;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            const int jl = rg * RY + r;
            const double *row = S + (jl + 1) * W + col;
            const double2 c = *reinterpret_cast<const double2 *>(row);
            const double xm = ilo ? S[L::XG_OFF + jl] : row[-1];
            const double xp1 = ihi1 ? S[L::XG_OFF + BY + jl] : row[2];
            const double xp0 = ihi0 ? S[L::XG_OFF + BY + jl] : c.y;
            const double2 ym = *reinterpret_cast<const double2 *>(row - W);
            const double2 yp = *reinterpret_cast<const double2 *>(row + W);
            double2 v;
            v.x = stencil5(c.x, xm, xp0, ym.x, yp.x);
            v.y = stencil5(c.y, c.x, xp1, ym.y, yp.y);
            const int j = y0 + jl;
            if (j < g.ey) emit_pair<false>(a, blk, dst, own, (int64_t)(j + 1) * g.P + g.A + i, i, j, 0, v);
        }
        __syncthreads();
        if (threadIdx.x == 0 && q + NS < nq) issue(q + NS);
    };
    auto lean_ok = [&](int q) {
        const int y0 = (ty0 + q) * BY;
        return xfull && (y0 + BY <= g.ey) && !((y0 == 0 && ym_face) || (y0 + BY == g.ey && yp_face));
    };
    // The block's first and last y tile (y faces, ragged rows) take the general path;
    // the tiles between are lean whenever the tile is full in x.
    int q = 0;
    if (q < nq && !lean_ok(q)) tile_general(q++);
    const int qend = (nq > q && !lean_ok(nq - 1)) ? nq - 1 : nq;
    if (xfull && q < qend) {
        int sl = q % NS;                    // ring slot of tile q
        uint32_t ph = (q / NS) & 1u;        // its mbarrier parity
        double *op = own + (int64_t)((ty0 + q) * BY + jl0 + 1) * g.P + g.A + i;
        double *xfp = xst ? xst + (int64_t)(ty0 + q) * BY : nullptr;
        const int64_t P = g.P, TP = (int64_t)BY * g.P;
        auto run = [&](const bool XE) {
            for (; q < qend; ++q) {
                mbar_wait(&bars[sl], ph);
                const double *S = stage + sl * L::STRIDE;
                const double *Sb = S + sb;
                double2 rw[RY + 2];  // rows jl0-1 .. jl0+RY
#pragma unroll
                for (int r = 0; r < RY + 2; ++r) rw[r] = *reinterpret_cast<const double2 *>(Sb + (r - 1) * W);
#pragma unroll
                for (int r = 0; r < RY; ++r) {
                    double xm = Sb[r * W - 1], xp1 = Sb[r * W + 2];
                    if (XE) {
                        if (ilo) xm = S[xg + r];
                        if (ihi1) xp1 = S[xg + BY + r];
                    }
                    const double2 c = rw[r + 1];
                    double2 v;
                    v.x = stencil5(c.x, xm, c.y, rw[r].x, rw[r + 2].x);
                    v.y = stencil5(c.y, c.x, xp1, rw[r].y, rw[r + 2].y);
                    ST16(a, op + r * P, v);
                    if (XE && xput) xface[q & 1][xside][jl0 + r] = ilo ? v.x : v.y;
                }
                op += TP;
                __syncthreads();
                if (threadIdx.x == 0 && q + NS < nq) issue(q + NS);
                if (XE && xfp) {  // row pairs of the x-ghost array (element j at xfp + j; even offsets)
                    ST16(a, xfp, *reinterpret_cast<const double2 *>(
                                     &xface[q & 1][(int)threadIdx.x / (BY / 2)][2 * ((int)threadIdx.x % (BY / 2))]));
                    xfp += BY;
                }
                if (++sl == NS) { sl = 0; ph ^= 1u; }
            }
        };
        if (xedge) run(true);
        else run(false);
    } else {
        for (; q < qend; ++q) tile_general(q);
    }
    if (q < nq) tile_general(q);
    if (remote) signal_done(a.sync[blk.part], a.exp_bits);
    span_end(a.span);
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
    const DevBlock blk = a.blocks[b];  // register copy (see emit_pair)
    const int i = tx * 64 + 2 * (threadIdx.x & 31);
    const int j = ty * 8 + (threadIdx.x >> 5);
    if (i >= g.ex || j >= g.ey) return;
    const int z0 = tz * a.zc, z1 = min(g.ez, z0 + a.zc);
    const double *s = a.arena + (int64_t)(a.src * g.nslots + blk.slot) * g.bstride;
    const double *xg0 = xg_array(a.xg, g, a.src, blk.slot, 0);
    const double *xg1 = xg_array(a.xg, g, a.src, blk.slot, 1);
    const int dst = 1 - a.src;
    double *own = a.arena + (int64_t)(dst * g.nslots + blk.slot) * g.bstride;
    for (int k = z0; k < z1; ++k) {
        const int64_t o = (int64_t)(k + 1) * g.Q + (int64_t)(j + 1) * g.P + g.A + i;
        const int64_t xo = (int64_t)k * g.eyp + j;
        const double2 cc = *reinterpret_cast<const double2 *>(s + o);
        const double xm = (i == 0) ? xg0[xo] : s[o - 1];
        const double xp0 = (i == g.ex - 1) ? xg1[xo] : cc.y;
        const double xp1 = (i + 1 == g.ex - 1) ? xg1[xo] : s[o + 2];
        const double2 ym = *reinterpret_cast<const double2 *>(s + o - g.P);
        const double2 yp = *reinterpret_cast<const double2 *>(s + o + g.P);
        const double2 zm = *reinterpret_cast<const double2 *>(s + o - g.Q);
        const double2 zp = *reinterpret_cast<const double2 *>(s + o + g.Q);
        double2 v;
        v.x = stencil7(cc.x, xm, xp0, ym.x, yp.x, zm.x, zp.x);
        v.y = stencil7(cc.y, cc.x, xp1, ym.y, yp.y, zm.y, zp.y);
        emit_pair(a, blk, dst, own + (int64_t)(k + 1) * g.Q, (int64_t)(j + 1) * g.P + g.A + i, i, j, k, v);
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
    double *xg = (d == 0) ? xg_array(a.xg, g, dst, blk.slot, f & 1) : nullptr;
    for (int64_t e = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.y * blockDim.x) {
        if (d == 0) {
            const int64_t k = e / g.ey, j = e % g.ey;
            // JAC_F_NCCL inboxes keep the x-ghost layout (pitch eyp); outboxes [k][ey]
            ST8(a, xg + k * g.eyp + j, (blk.pack_mask & (1u << f)) ? src[k * g.eyp + j] : src[e]);
            continue;
        }
        int64_t off;
        if (d == 1) {
            const int64_t k = e / g.ex, i = e % g.ex;
            off = (k + g.zg) * g.Q + ((f == YM) ? 0 : (int64_t)(g.ey + 1) * g.P) + g.A + i;
        } else {
            const int64_t j = e / g.ex, i = e % g.ex;
            off = ((f == ZM) ? 0 : (int64_t)(g.ez + 1) * g.Q) + (j + 1) * g.P + g.A + i;
        }
        ST8(a, base + off, src[e]);
    }
}

// ------------------------------------------------------------------ paper-style pack / unpack
// JAC_F_PER_BLOCK (NEXT-2): one pack and one unpack launch per face per block, on
// the block's own stream, as in the paper's Charm++ Jacobi (PAPER.md:90, SPEC.md:474:
// "packs 4 boundary strips (pack kernel per face on its own stream) ... on receiving
// all 4 runs unpack kernels then the stencil kernel").
// pack: boundary layer of face f of block `slot`, buffer `buf` -> outbox[par][slot][f]
__global__ void __launch_bounds__(256) pack_face_kernel(const SweepArgs a, int slot, int f, int buf, int par)
{
    const Geom &g = a.g;
    const double *base = a.arena + (int64_t)(buf * g.nslots + slot) * g.bstride;
    double *ob = a.outbox + ((int64_t)par * g.nslots + slot) * g.ostride + g.ooff[f];
    const int d = f >> 1;
    const int64_t n = (d == 0) ? (int64_t)g.ey * g.ez : (d == 1) ? (int64_t)g.ex * g.ez : (int64_t)g.ex * g.ey;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t off;
        if (d == 0) {
            const int64_t k = e / g.ey, j = e % g.ey;
            off = (k + g.zg) * g.Q + (j + 1) * g.P + g.A + ((f == XM) ? 0 : g.ex - 1);
        } else if (d == 1) {
            const int64_t k = e / g.ex, i = e % g.ex;
            off = (k + g.zg) * g.Q + ((f == YM) ? 1 : (int64_t)g.ey) * g.P + g.A + i;
        } else {
            const int64_t j = e / g.ex, i = e % g.ex;
            off = ((f == ZM) ? 1 : (int64_t)g.ez) * g.Q + (j + 1) * g.P + g.A + i;
        }
        ST8(a, ob + e, base[off]);
    }
}

// unpack: outbox[par][nslot][opposite(f)] of the neighbour -> ghost face f of block
// `slot` in buffer `buf` (x ghosts into the x-ghost arrays).
__global__ void __launch_bounds__(256) unpack_face_kernel(const SweepArgs a, int slot, int nslot, int f, int buf, int par)
{
    const Geom &g = a.g;
    const double *src = a.outbox + ((int64_t)par * g.nslots + nslot) * g.ostride + g.ooff[opposite(f)];
    double *base = a.arena + (int64_t)(buf * g.nslots + slot) * g.bstride;
    const int d = f >> 1;
    const int64_t n = (d == 0) ? (int64_t)g.ey * g.ez : (d == 1) ? (int64_t)g.ex * g.ez : (int64_t)g.ex * g.ey;
    double *xg = (d == 0) ? xg_array(a.xg, g, buf, slot, f & 1) : nullptr;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        if (d == 0) {
            const int64_t k = e / g.ey, j = e % g.ey;
            ST8(a, xg + k * g.eyp + j, src[e]);
            continue;
        }
        int64_t off;
        if (d == 1) {
            const int64_t k = e / g.ex, i = e % g.ex;
            off = (k + g.zg) * g.Q + ((f == YM) ? 0 : (int64_t)(g.ey + 1) * g.P) + g.A + i;
        } else {
            const int64_t j = e / g.ex, i = e % g.ex;
            off = ((f == ZM) ? 0 : (int64_t)(g.ez + 1) * g.Q) + (j + 1) * g.P + g.A + i;
        }
        ST8(a, base + off, src[e]);
    }
}

static unsigned face_grid(const Geom &g, int f)
{
    const int d = f >> 1;
    const int64_t n = (d == 0) ? (int64_t)g.ey * g.ez : (d == 1) ? (int64_t)g.ex * g.ez : (int64_t)g.ex * g.ey;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(1184, (n + 255) / 256));
}

cudaError_t launch_pack_face(const SweepArgs &a, int slot, int f, int buf, int par, cudaStream_t s)
{
    pack_face_kernel<<<face_grid(a.g, f), 256, 0, s>>>(a, slot, f, buf, par);
    return cudaGetLastError();
}

cudaError_t launch_unpack_face(const SweepArgs &a, int slot, int nslot, int f, int buf, int par, cudaStream_t s)
{
    unpack_face_kernel<<<face_grid(a.g, f), 256, 0, s>>>(a, slot, nslot, f, buf, par);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ neighbour barrier
__global__ void barrier_kernel(const BarrierArgs ba)
{
    if (threadIdx.x != 0) return;
    __threadfence_system();  // the preceding phase's stores (incl. peer stores) first
    for (int p = 0; p < ba.nparts; ++p) {
        const PartSync &ps = ba.sync[p];
        const uint64_t e = ps.ctrl[0] + 1;
        *reinterpret_cast<volatile uint64_t *>(ps.ctrl) = e;
        for (int n = 0; n < ps.npeers; ++n)
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(ps.peer_slot[n]), "l"(e) : "memory");
    }
    for (int p = 0; p < ba.nparts; ++p) {
        const PartSync &ps = ba.sync[p];
        wait_flags(ps, ps.ctrl[0], ba.wd);
    }
    __threadfence_system();
}

// ------------------------------------------------------------------ virtual transport
// JAC_F_VIRTUAL_GPUS | JAC_F_NCCL: the packed REMOTE faces move from each partition's
// send buffer into its neighbour's receive buffer (one list entry per face, the pair
// an ncclSend / ncclRecv would move); the batched ghost kernel then unpacks them.
__global__ void __launch_bounds__(256) face_copy_kernel(const FaceCopy *list)
{
    const FaceCopy fc = list[blockIdx.y];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < fc.count;
         e += (int64_t)gridDim.x * blockDim.x)
        fc.dst[e] = fc.src[e];
}

// ------------------------------------------------------------------ init helpers
// Copies the inline ghost columns i = -1 / ex of buffer 0 (filled by the init copy)
// into both buffers' x-ghost arrays.
__global__ void xghost_extract_kernel(const SweepArgs a)
{
    const Geom &g = a.g;
    const DevBlock &blk = a.blocks[blockIdx.y];
    const double *b0 = a.arena + (int64_t)blk.slot * g.bstride;
    const int64_t n = (int64_t)g.ey * g.ez;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / g.ey, j = e % g.ey;
        const int64_t row = (k + g.zg) * g.Q + (j + 1) * g.P + g.A;
        const double lo = b0[row - 1], hi = b0[row + g.ex];
        for (int buf = 0; buf < 2; ++buf) {
            ST8(a, xg_array(a.xg, g, buf, blk.slot, 0) + k * g.eyp + j, lo);
            ST8(a, xg_array(a.xg, g, buf, blk.slot, 1) + k * g.eyp + j, hi);
        }
    }
}

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
    const int64_t n = sx * sy * (g.ez + 2 * g.zg);
    double *b0 = a.arena + (int64_t)blk.slot * g.bstride;
    double *b1 = a.arena + (int64_t)(g.nslots + blk.slot) * g.bstride;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ii = e % sx, jj = (e / sx) % sy, kk = e / (sx * sy);  // ghost-inclusive
        const uint64_t px = blk.org[0] + ii, py = blk.org[1] + jj, pz = blk.org[2] + kk;
        const uint64_t p = (pz * (uint64_t)(ny + 2) + py) * (uint64_t)(nx + 2) + px;
        const double v = r11_value(seed, p);
        if (g.A == 0 && (ii == 0 || ii == sx - 1)) {  // dense rows: x ghosts -> x-ghost arrays
            if (jj >= 1 && jj <= g.ey && kk >= g.zg && kk < g.ez + g.zg) {
                const int64_t xi = (kk - g.zg) * g.eyp + (jj - 1);
                ST8(a, xg_array(a.xg, g, 0, blk.slot, ii ? 1 : 0) + xi, v);
                ST8(a, xg_array(a.xg, g, 1, blk.slot, ii ? 1 : 0) + xi, v);
            }
            continue;
        }
        const int64_t off = kk * g.Q + jj * g.P + (g.A - 1) + ii;
        ST8(a, b0 + off, v);
        ST8(a, b1 + off, v);
    }
}

// ------------------------------------------------------------------ staged host transfers
// The intersection of a block's cell range [lo0, lo0 + n) (block-relative, per dim) with
// the stage box, as block-relative [lo, hi).
__device__ __forceinline__ bool stage_clip(const DevBlock &blk, const StageBox &sb, const int64_t lo0[3],
                                           const int64_t n[3], int64_t lo[3], int64_t hi[3])
{
    bool any = true;
    for (int k = 0; k < 3; ++k) {
        lo[k] = max(lo0[k], sb.o[k] - blk.org[k]);
        hi[k] = min(lo0[k] + n[k], sb.o[k] + sb.n[k] - blk.org[k]);
        any &= lo[k] < hi[k];
    }
    return any;
}

// One warp per row of the clipped range (x along the lanes, rows spread over the grid):
// coalesced on both sides, one division per row.  SCATTER: staging -> every
// ghost-inclusive cell of the block in both buffers (dense rows: x ghosts -> both
// x-ghost arrays, as hash_init_kernel); else interior cells of buffer `buf` -> staging.
template <bool SCATTER>
__global__ void __launch_bounds__(256) stage_kernel(const SweepArgs a, const int32_t *__restrict__ list, int32_t nlist,
                                                   double *__restrict__ st, const StageBox sb, int buf)
{
    const Geom &g = a.g;
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int64_t lo0[3] = {SCATTER ? 0 : 1, SCATTER ? 0 : 1, SCATTER ? 0 : g.zg};
    const int64_t n[3] = {SCATTER ? g.ex + 2 : g.ex, SCATTER ? g.ey + 2 : g.ey,
                          SCATTER ? g.ez + 2 * g.zg : g.ez};
    for (int32_t li = blockIdx.y; li < nlist; li += gridDim.y) {
        const DevBlock &blk = a.blocks[list[li]];
        int64_t lo[3], hi[3];
        if (!stage_clip(blk, sb, lo0, n, lo, hi)) continue;
        const int ny = (int)(hi[1] - lo[1]), nrows = ny * (int)(hi[2] - lo[2]);
        const int i0 = (int)lo[0], i1 = (int)hi[0];
        double *b0 = a.arena + (int64_t)((SCATTER ? 0 : buf) * g.nslots + blk.slot) * g.bstride;
        double *b1 = a.arena + (int64_t)(g.nslots + blk.slot) * g.bstride;
        for (int r = blockIdx.x * nw + (threadIdx.x >> 5); r < nrows; r += gridDim.x * nw) {
            const int64_t jj = lo[1] + r % ny, kk = lo[2] + r / ny;
            double *srow = st + ((blk.org[2] + kk - sb.o[2]) * sb.n[1] + (blk.org[1] + jj - sb.o[1])) * sb.pitch +
                           (blk.org[0] - sb.o[0]);  // element ii of the block row
            const int64_t roff = kk * g.Q + jj * g.P + (g.A - 1);
            if (SCATTER) {
                const bool xgrow = g.A == 0 && jj >= 1 && jj <= g.ey && kk >= g.zg && kk < g.ez + g.zg;
#pragma unroll 4
                for (int ii = i0 + lane; ii < i1; ii += 32) {
                    const double v = srow[ii];
                    if (g.A == 0 && (ii == 0 || ii == n[0] - 1)) {  // dense rows: x ghosts
                        if (xgrow) {
                            const int64_t xi = (kk - g.zg) * g.eyp + (jj - 1);
                            ST8(a, xg_array(a.xg, g, 0, blk.slot, ii ? 1 : 0) + xi, v);
                            ST8(a, xg_array(a.xg, g, 1, blk.slot, ii ? 1 : 0) + xi, v);
                        }
                        continue;
                    }
                    ST8(a, b0 + roff + ii, v);
                    ST8(a, b1 + roff + ii, v);
                }
            } else {
#pragma unroll 4
                for (int ii = i0 + lane; ii < i1; ii += 32) ST8(a, srow + ii, b0[roff + ii]);
            }
        }
    }
}

// ------------------------------------------------------------------ host launchers
template <int BX, int BY, int W, int NT, int NS>
static int resident_tma_t()
{
    static int resident = 0;  // SMs x CTAs per SM (per process; one device per process)
    if (!resident) {
        constexpr size_t smem = tma_smem_bytes(BX, BY, W, NS);  // NS stages, NS - 1 planes in flight
        // the occupancy query needs the kernel's dynamic shared-memory limit raised
        // first (above 48 KB it would report 0 CTAs per SM)
        cudaFuncSetAttribute(sweep_tma_kernel<BX, BY, W, NT, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_tma_kernel<BX, BY, W, NT, NS>, NT, smem);
        resident = std::max(1, sms * std::max(1, per_sm));
    }
    return resident;
}

template <int BX, int BY, int W, int NT, int NS>
static cudaError_t prepare_tma_t()
{
    constexpr size_t smem = tma_smem_bytes(BX, BY, W, NS);
    return cudaFuncSetAttribute(sweep_tma_kernel<BX, BY, W, NT, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem);
}

// <<<grid, block, smem, s>>>(args...) with programmatic stream serialization when pdl
template <typename... Args>
static cudaError_t launch_maybe_pdl(void (*kernel)(Args...), unsigned grid, unsigned block, size_t smem,
                                    cudaStream_t s, bool pdl, const Args &...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int BX, int BY, int W, int NT, int NS>
static cudaError_t launch_tma_t(const CUtensorMap &tm, const SweepArgs &a, cudaStream_t s, bool pdl)
{
    constexpr size_t smem = tma_smem_bytes(BX, BY, W, NS);
    // One CTA per item: the hardware launches CTAs in index order as slots free up,
    // which keeps x/y-adjacent tiles (and successive z-chunks of a column) temporally
    // close, so their shared halo planes are L2 hits.  A persistent grid with static
    // striding lets CTAs drift apart and turns halos into DRAM re-reads (measured
    // 359 -> 454 us per 512^3 sweep).
    return launch_maybe_pdl(sweep_tma_kernel<BX, BY, W, NT, NS>, (unsigned)a.nitems, NT, smem, s, pdl, tm, a);
}

// Ring depth, measured on several B200 boxes: for the wide tile a 6-stage ring (3 CTAs
// / SM at 79 registers) gave 355 us per 512^3 ODF-1 sweep on every box, a 4-stage
// ring (4 CTAs / SM) 348 us on some and 385 us on others, so jac_create times both
// (engine.cu: autotune) -- also for the 2-D kernel (32768^2: 2.53 ms at 4 stages vs
// 2.91 ms at 6 on one box).  5 stages (spills), 7-8 stages (2 CTAs / SM) and 64 x 8
// tiles were slower everywhere.  The narrow / exact tiles (small blocks) keep 4
// stages (6 stages: 32^3 blocks 582 -> 655 us).  128 x 16 tiles (256 threads: spills;
// 512 threads: 2 CTAs / SM) were 1-8% slower than 64 x 16.  32-wide blocks
// take a whole 32 x 32 face per item (C5's 32^3 blocks: 583 -> 475 us per 512^3);
// 64 x 32 tiles spill at 64 registers and lose.
#define JAC_TMA_VARIANTS(X)               \
    X(TMA_WIDE, 64, 16, 68, 256, 6)       \
    X(TMA_WIDE4, 64, 16, 68, 256, 4)      \
    X(TMA_NARROW, 32, 16, 36, 256, 4)     \
    X(TMA_EXACT32, 32, 16, 32, 256, 5)    \
    X(TMA_EXACT64, 64, 16, 64, 256, 4)    \
    X(TMA_EXACT32_TALL, 32, 32, 32, 256, 4) \
    X(TMA_EXACT32_6, 32, 16, 32, 256, 6)    \
    X(TMA_EXACT64_6, 64, 16, 64, 256, 6)    \
    X(TMA_WIDE_TALL, 64, 32, 68, 256, 4)

int sweep_resident_ctas(int variant)
{
#define X(V, BX, BY, W, NT, NS) \
    if (variant == V) return resident_tma_t<BX, BY, W, NT, NS>();
    JAC_TMA_VARIANTS(X)
#undef X
    return 148;
}

TileShape tma_tile_shape(int variant)
{
#define X(V, BX, BY, W, NT, NS) \
    if (variant == V) return {BX, BY, W};
    JAC_TMA_VARIANTS(X)
#undef X
    return {0, 0, 0};
}

cudaError_t prepare_sweep_tma(int variant)
{
#define X(V, BX, BY, W, NT, NS) \
    if (variant == V) return prepare_tma_t<BX, BY, W, NT, NS>();
    JAC_TMA_VARIANTS(X)
#undef X
    return cudaErrorInvalidValue;
}

cudaError_t launch_sweep_tma(const CUtensorMap &tm, const SweepArgs &a, int variant, cudaStream_t s, bool pdl)
{
#define X(V, BX, BY, W, NT, NS) \
    if (variant == V) return launch_tma_t<BX, BY, W, NT, NS>(tm, a, s, pdl);
    JAC_TMA_VARIANTS(X)
#undef X
    return cudaErrorInvalidValue;
}

template <int BX, int BY, int W, int NT, int NS>
static cudaError_t launch2d_t(const CUtensorMap &tm, const SweepArgs &a, cudaStream_t s, bool prepare_only,
                              bool pdl = false)
{
    constexpr size_t smem = tma_smem_bytes(BX, BY, W, NS);
    if (prepare_only)
        return cudaFuncSetAttribute(sweep2d_tma_kernel<BX, BY, W, NT, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem);
    return launch_maybe_pdl(sweep2d_tma_kernel<BX, BY, W, NT, NS>, (unsigned)a.nitems, NT, smem, s, pdl, tm, a);
}

cudaError_t launch_sweep2d_tma(const CUtensorMap &tm, const SweepArgs &a, int variant, cudaStream_t s, bool pdl)
{
#define X(V, BX, BY, W, NT, NS) \
    if (variant == V) return launch2d_t<BX, BY, W, NT, NS>(tm, a, s, false, pdl);
    JAC_TMA_VARIANTS(X)
#undef X
    return cudaErrorInvalidValue;
}

cudaError_t prepare_sweep2d_tma(int variant)
{
    static const CUtensorMap none{};  // not read: prepare_only sets the attribute only
    SweepArgs dummy{};
#define X(V, BX, BY, W, NT, NS) \
    if (variant == V) return launch2d_t<BX, BY, W, NT, NS>(none, dummy, nullptr, true);
    JAC_TMA_VARIANTS(X)
#undef X
    return cudaErrorInvalidValue;
}

cudaError_t launch_sweep_plain(const SweepArgs &a, cudaStream_t s)
{
    const int64_t grid = (int64_t)a.g.nslots * a.ntx * a.nty * a.ntz;
    sweep_plain_kernel<<<(unsigned)grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_sweep_plain_one(const SweepArgs &a, cudaStream_t s)
{
    const int64_t grid = (int64_t)a.ntx * a.nty * a.ntz;  // a.blocks points at the one block
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

cudaError_t launch_face_copy(const FaceCopy *list, int n, int64_t maxcount, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    const int64_t gx = std::max<int64_t>(1, std::min<int64_t>(64, (maxcount + 255) / 256));
    face_copy_kernel<<<dim3((unsigned)gx, (unsigned)n), 256, 0, s>>>(list);
    return cudaGetLastError();
}

cudaError_t launch_hash_init(const SweepArgs &a, int64_t nx, int64_t ny, uint64_t seed, cudaStream_t s)
{
    hash_init_kernel<<<dim3(64, (unsigned)a.g.nslots), 256, 0, s>>>(a, nx, ny, seed);
    return cudaGetLastError();
}

// rows: an upper bound on one listed block's rows inside the slab (8 rows per CTA)
static dim3 stage_grid(int32_t nlist, int64_t rows)
{
    const int64_t gx = std::min<int64_t>(std::max<int64_t>(1, 4096 / std::max(1, nlist)),
                                         std::max<int64_t>(1, (rows + 7) / 8));
    return dim3((unsigned)gx, (unsigned)std::max(1, std::min(nlist, 65535)));
}

cudaError_t launch_stage_scatter(const SweepArgs &a, const int32_t *list, int32_t nlist, int64_t rows,
                                 const double *st, const StageBox &sb, cudaStream_t s)
{
    if (nlist <= 0) return cudaSuccess;
    stage_kernel<true><<<stage_grid(nlist, rows), 256, 0, s>>>(a, list, nlist, const_cast<double *>(st), sb, 0);
    return cudaGetLastError();
}

cudaError_t launch_stage_gather(const SweepArgs &a, const int32_t *list, int32_t nlist, int64_t rows, double *st,
                                const StageBox &sb, int buf, cudaStream_t s)
{
    if (nlist <= 0) return cudaSuccess;
    stage_kernel<false><<<stage_grid(nlist, rows), 256, 0, s>>>(a, list, nlist, st, sb, buf);
    return cudaGetLastError();
}

cudaError_t launch_xghost_extract(const SweepArgs &a, cudaStream_t s)
{
    xghost_extract_kernel<<<dim3(16, (unsigned)a.g.nslots), 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace jac
