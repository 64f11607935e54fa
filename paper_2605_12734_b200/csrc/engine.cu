// engine.cu -- host engine + C ABI (include/jacobi3d.h).
//
// Owns, per context (one CUDA device; one process per GPU for multi-GPU runs):
//   * the block-descriptor table (north-star subsystem 1), built once from the
//     planner and copied to the device; REMOTE faces carry IPC-mapped peer pointers
//     (the paper's pre-filled location table + transport selection, PAPER.md:230,
//     266-275, resolved once instead of per message);
//   * one arena holding both ghosted buffers of every local block, one 4-D TMA
//     tensor map over it, optional outbox (JAC_F_UNFUSED_PACK), control words;
//   * one stream, CUDA graphs of the iteration (north-star subsystem 5; PAPER.md:86
//     "CUDA Graphs to amortize kernel launch overhead"), timing events.
// Nothing is allocated inside jac_step (persistent views and
// preallocated scratch instead of allocations that imply fences).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without a tool attached

#include <algorithm>
#include <climits>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <tuple>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/jacobi3d.h"
#include "device.hpp"
#include "kernels.hpp"
#include "plan.hpp"

namespace {

thread_local std::string g_err;

// NVTX range over one C-ABI call (jac_step, init, profile, create), for timelines
// taken with a tracing tool (nsys is not in this image; the ranges are inert without one)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                             \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(e_ == cudaErrorMemoryAllocation ? JAC_ENOMEM : JAC_ECUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                  \
    } while (0)

constexpr uint32_t kIpcMagic = 0x4A414334u;  // "JAC4"
constexpr int kPlain = 2;  // variant id of the JAC_F_NO_TMA sweep

struct IpcRecord {
    uint32_t magic;
    int32_t rank;
    uint64_t fingerprint;
    uint64_t arena_off, outbox_off, ctrl_off, xg_off;
    uint64_t alloc_bytes;  // size of the mapped allocation (checked build: store ranges)
    cudaIpcMemHandle_t handle;
    unsigned char pad_[256 - 56 - sizeof(cudaIpcMemHandle_t)];
};
static_assert(sizeof(IpcRecord) == 256, "IPC record size");

// NCCL, loaded at run time (JAC_F_NCCL only): no link-time dependency, and the
// process's already-loaded libnccl.so.2 (torch's) is the one resolved.
struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId *);
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*commDestroy)(ncclComm_t);
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*groupStart)();
    ncclResult_t (*groupEnd)();
    const char *(*errorString)(ncclResult_t);
};

const NcclApi *nccl_api()
{
    static NcclApi api;
    static int state = 0;  // 0 untried, 1 ok, -1 failed
    if (state == 0) {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        state = -1;
        if (h) {
            api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
            api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
            api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
            api.send = (decltype(api.send))dlsym(h, "ncclSend");
            api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
            api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
            api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
            api.errorString = (decltype(api.errorString))dlsym(h, "ncclGetErrorString");
            if (api.getUniqueId && api.commInitRank && api.commDestroy && api.send && api.recv && api.groupStart &&
                api.groupEnd && api.errorString)
                state = 1;
        }
    }
    return state == 1 ? &api : nullptr;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                    const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

namespace jac {
// for the microbenchmarks (microbench.cu): same thread-local error slot
void set_last_error(int code, const char *msg)
{
    (void)code;
    g_err = msg;
}
}  // namespace jac

struct NcclFace {
    int32_t peer;
    int64_t key;    // min(global block ids) * 3 + axis: identical on both ranks
    int64_t count;  // doubles
    double *send, *recv;
};

struct jac_ctx {
    jac::Plan plan{};
    uint32_t flags = 0;
    bool rank_mode = false;
    bool virtual_parts = false;  // JAC_F_VIRTUAL_GPUS: every partition on one device, one kernel
    int32_t rank = 0;         // partition owned in rank mode
    int device = 0;
    std::vector<int32_t> parts;  // partitions hosted by this context
    int32_t nslots = 0;

    // group context (jac_create with n_gpus > 1): one rank-mode sub-context per device,
    // connected by plain peer pointers; every call fans out to them
    bool group = false;
    std::vector<jac_ctx *> subs;
    bool in_group = false;  // a group's sub-context

    jac::Geom geom{};
    char *alloc = nullptr;    // single allocation: [ctrl][arena][x ghosts][outbox]
    size_t alloc_bytes = 0, ctrl_off = 0, arena_off = 0, xg_off = 0, outbox_off = 0;
    uint64_t *ctrl = nullptr;
    int64_t ctrl_stride = 0;  // control words per hosted partition (PartSync)
    double *arena = nullptr, *xg = nullptr, *outbox = nullptr;
    std::vector<jac::DevBlock> hblocks;
    jac::DevBlock *dblocks = nullptr;

    int variant = 0;          // jac::TmaVariant, or kPlain
    CUtensorMap tmap{};
    int ntx = 1, nty = 1, ntz = 1, zc = 1;
    int nzc = 1, ncols = 1, nitems = 1, gcols = 1;
    float tuned_ms[2] = {0.f, 0.f};  // autotune: sweep ms for the 6- and 4-stage wide tiles
    double last_gap_ms = -1.0;       // jac_profile_sweep: median gap between consecutive sweeps
    int64_t last_wait_sum_ns = 0, last_wait_max_ns = 0;  // jac_profile_sweep: remote CTAs' peer waits
    unsigned long long *prof_span = nullptr;  // jac_profile_sweep capture: per-iteration [start, end]
    int prof_it = 0;
    bool pdl = true;                 // sweeps use programmatic dependent launch (JAC_PDL=0: off)

    // cross-partition exchange
    std::vector<std::vector<int32_t>> part_peers;  // [hosted partition] -> neighbour partitions
    std::vector<jac::PartSync> hsync;              // [hosted partition]
    jac::PartSync *dsync = nullptr;
    uint32_t *status_h = nullptr, *status_d = nullptr;  // watchdog / check words (mapped pinned host)
    std::vector<jac::MemRange> ranges;                  // own allocation + connected peers'
    jac::MemRange *dranges = nullptr;
    uint64_t watchdog_ns = 60ull * 1000 * 1000 * 1000;
    std::vector<void *> ipc_opened;
    bool ipc_done = false;
    bool fused = false;                 // fused cross-partition ordering inside the sweep
    std::vector<NcclFace> nccl_faces;   // JAC_F_NCCL: remote faces, sorted (peer, key)
    void *nccl_comm = nullptr;
    std::vector<jac::FaceCopy> vcopies; // JAC_F_VIRTUAL_GPUS | JAC_F_NCCL: the virtual transport
    jac::FaceCopy *dvcopies = nullptr;
    int64_t vcopy_max = 0;
    int32_t *ditem_map = nullptr;       // launch order -> item (~item: remote-touching)
    int32_t nremote = 0;
    std::vector<int32_t> nremote_part;  // remote-touching items per hosted partition
    bool tuned = false;                 // the create-time default variant was re-timed on data

    cudaStream_t stream = nullptr;
    // staged host transfers (jac_set_init_box / jac_get_field_box): two device slabs, a
    // copy stream, events filled[2] / drained[2] and the per-slab block lists; set up at
    // the first transfer
    double *stage[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    bool stage_pitched = false;  // JAC_STAGE_PITCHED=1 (tests): pitched copies even for contiguous slabs
    bool stage_direct = false;   // JAC_DIRECT=1 (experiment): kernels read / write a mapped pinned host box
    cudaStream_t cstream = nullptr;
    cudaEvent_t sev[4] = {nullptr, nullptr, nullptr, nullptr};
    int32_t *dlist = nullptr;
    size_t dlist_cap = 0;
    std::vector<int32_t> by_origin[3];  // table indices sorted by block origin along x / y / z
    // JAC_F_PER_BLOCK (paper-style): one stream per block, events per block and parity
    std::vector<cudaStream_t> bstreams;
    std::vector<cudaEvent_t> bevents;  // [slot * 2 + parity]
    int launch_threads = 1;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaGraphExec_t g1[2] = {nullptr, nullptr}, gU[2] = {nullptr, nullptr};
    int unroll = 10;
    uint64_t exp_mask = 0;  // experiment knobs this context read (JAC_STAT_EXPERIMENT)
    int32_t exp_bits = 0;   // kernel-side timing experiments (SweepArgs::exp_bits)

    bool inited = false;
    int64_t iters = 0;
    double last_ms = 0.0;
    int64_t kernel_launches = 0, graph_launches = 0;
    int64_t local_faces = 0, remote_faces = 0, remote_bytes = 0;

    bool has_remote() const
    {
        for (const auto &p : part_peers)
            if (!p.empty()) return true;
        return false;
    }
    bool virtual_copy() const { return virtual_parts && (flags & JAC_F_NCCL); }
    int kernels_per_iter() const
    {
        if (flags & JAC_F_PER_BLOCK) return (int)(nslots + 2 * local_faces + 2 * remote_faces);
        if (fused) return 1;
        if (flags & JAC_F_NCCL) return virtual_copy() ? 3 : 2;  // sweep + [copy] + unpack (NCCL's own kernels not counted)
        int k = 1;
        if (flags & JAC_F_UNFUSED_PACK) k += 1 + (has_remote() ? 2 : 0);
        else if (has_remote()) k += 1;
        return k;
    }
    double *slot_ptr(int buf, int slot) const
    {
        return arena + (int64_t)(buf * nslots + slot) * geom.bstride;
    }
    jac::Watchdog wd() const { return {status_d, watchdog_ns}; }
    jac::CheckArgs chk() const { return {dranges, (int32_t)ranges.size(), 0, status_d}; }
};

namespace {

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

uint64_t fingerprint(const jac_ctx *c)
{
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
    for (int d = 0; d < 3; ++d) { mix(c->plan.n[d]); mix(c->plan.b[d]); mix(c->plan.g[d]); }
    mix(c->plan.n_gpus); mix(c->flags & (JAC_F_UNFUSED_PACK)); mix(c->geom.bstride); mix(c->geom.ostride);
    mix(c->geom.xgstride);
    return h;
}

// Experiment knobs: environment variables that select a tile variant,
// layout or launch detail for same-box A/B measurements.  They are read only when
// JAC_EXPERIMENT=1, and every knob a context saw is recorded in its
// JAC_STAT_EXPERIMENT mask, so no stray variable silently changes a production run.
const char *const kKnobs[] = {"JAC_L2PROMO", "JAC_ZC",     "JAC_ZCHUNK", "JAC_GCOLS",   "JAC_VARIANT",
                              "JAC_AUTOTUNE", "JAC_A",      "JAC_PALIGN", "JAC_NO_DENSE", "JAC_UNROLL",
                              "JAC_PDL",     "JAC_NO_FUSED_SYNC", "JAC_ORDER_EXP", "JAC_DROP_REMOTE",
                              "JAC_HOLD_SIGNAL", "JAC_REMOTE_SPREAD", "JAC_CHECK_SELFTEST", "JAC_YCHUNK",
                              "JAC_NO_CTA_SYSFENCE", "JAC_REMOTE_COLMAJOR", "JAC_XBAND", "JAC_STAGE_BYTES",
                              "JAC_STAGE_PITCHED", "JAC_DIRECT"};

const char *knob(jac_ctx *c, const char *name)
{
    const char *on = getenv("JAC_EXPERIMENT");
    if (!on || strcmp(on, "1") != 0) return nullptr;
    const char *v = getenv(name);
    if (v)
        for (size_t i = 0; i < sizeof kKnobs / sizeof kKnobs[0]; ++i)
            if (!strcmp(kKnobs[i], name)) c->exp_mask |= 1ull << i;
    return v;
}

int64_t experiment_mask(const jac_ctx *c) { return (int64_t)c->exp_mask; }

jac::SweepArgs sweep_args(const jac_ctx *c, int src, int mode)
{
    jac::SweepArgs a{};
    a.g = c->geom;
    a.blocks = c->dblocks;
    a.arena = c->arena;
    a.xg = c->xg;
    a.outbox = c->outbox;
    a.src = src;
    a.mode = mode;
    a.ntx = c->ntx; a.nty = c->nty; a.ntz = c->ntz; a.zc = c->zc;
    a.nzc = c->nzc; a.ncols = c->ncols; a.nitems = c->nitems; a.gcols = c->gcols;
    if (c->ditem_map && !c->fused) a.item_map = c->ditem_map;  // JAC_ORDER_EXP
    if (c->prof_span) a.span = c->prof_span + 4 * (int64_t)c->prof_it;
    a.wd = c->wd();
    a.chk = c->chk();
    a.exp_bits = c->exp_bits;
    if (c->fused && mode == jac::MODE_FUSED) {
        a.fused_sync = 1;
        a.nremote = c->nremote;
        a.item_map = c->ditem_map;
        a.sync = c->dsync;
    }
    return a;
}

int sweep_mode(const jac_ctx *c)
{
    if (c->flags & JAC_F_SKIP_EXCHANGE) return jac::MODE_NOEXCHANGE;
    if (c->flags & JAC_F_UNFUSED_PACK) return jac::MODE_PACK;
    return jac::MODE_FUSED;
}

int enqueue_sweep(jac_ctx *c, int src)
{
    const jac::SweepArgs a = sweep_args(c, src, sweep_mode(c));
    if (c->variant == kPlain) CK(jac::launch_sweep_plain(a, c->stream));
    else if (c->flags & JAC_F_2D) CK(jac::launch_sweep2d_tma(c->tmap, a, c->variant, c->stream, c->pdl));
    else CK(jac::launch_sweep_tma(c->tmap, a, c->variant, c->stream, c->pdl));
    return JAC_OK;
}

int enqueue_barrier(jac_ctx *c)
{
    // NCCL contexts share no memory with their peers: NCCL (or, for virtual
    // partitions, the copy kernel in stream order) orders the exchange
    if (!c->has_remote() || (c->flags & JAC_F_NCCL)) return JAC_OK;
    jac::BarrierArgs ba{};
    ba.sync = c->dsync;
    ba.nparts = (int32_t)c->parts.size();
    ba.wd = c->wd();
    CK(jac::launch_barrier(ba, c->stream));
    return JAC_OK;
}

// The watchdog word the cross-partition waits set when a neighbour never signalled.
int check_status(jac_ctx *c)
{
    if (!c->status_h) return JAC_OK;
    volatile uint32_t *w = c->status_h;
    const uint32_t f = w[0];
    if (!f) return JAC_OK;
    const uint32_t line = w[1];
    const unsigned long long addr = (unsigned long long)w[2] | ((unsigned long long)w[3] << 32);
    w[0] = w[1] = w[2] = w[3] = 0;
    if (f & (jac::kStatusMisaligned | jac::kStatusOutOfRange | jac::kStatusAssert))
        return fail(JAC_ECUDA, "checked build: %s%s%s at kernels.cu:%u (address %#llx); the store was skipped",
                    (f & jac::kStatusOutOfRange) ? "out-of-range store " : "",
                    (f & jac::kStatusMisaligned) ? "misaligned store " : "",
                    (f & jac::kStatusAssert) ? "failed assertion " : "", line, addr);
    return fail(JAC_ECUDA, "peer watchdog: a neighbour partition did not signal within %.1f s (rank skew, "
                           "dead peer or unequal call sequences); this call's results are invalid",
                (double)c->watchdog_ns * 1e-9);
}

// Device copy of the store ranges (checked build): own allocation + connected peers'.
int upload_ranges(jac_ctx *c)
{
    if (!c->dranges) CK(cudaMalloc(&c->dranges, sizeof(jac::MemRange) * 8));
    if (c->ranges.size() > 8) return fail(JAC_EINVAL, "too many store ranges");
    CK(cudaMemcpy(c->dranges, c->ranges.data(), sizeof(jac::MemRange) * c->ranges.size(), cudaMemcpyHostToDevice));
    return JAC_OK;
}

// One Jacobi iteration reading buffer `src` (all kernels on c->stream).
int enqueue_iteration(jac_ctx *c, int src, cudaEvent_t evs = nullptr, cudaEvent_t eve = nullptr)
{
    int rc;
    // external event-record nodes when captured (jac_profile_sweep), so they time
    if (evs) CK(cudaEventRecordWithFlags(evs, c->stream, cudaEventRecordExternal));
    if ((rc = enqueue_sweep(c, src))) return rc;
    if (eve) CK(cudaEventRecordWithFlags(eve, c->stream, cudaEventRecordExternal));
    if (c->virtual_copy()) {  // virtual partitions: packed faces moved by a copy kernel
        CK(jac::launch_face_copy(c->dvcopies, (int)c->vcopies.size(), c->vcopy_max, c->stream));
        CK(jac::launch_ghost_fill(sweep_args(c, src, jac::MODE_FUSED), 1 - src, c->stream));
        return JAC_OK;
    }
    if (c->flags & JAC_F_NCCL) {  // ablation: library point-to-point instead of peer stores
        const NcclApi *N = nccl_api();
        ncclComm_t comm = (ncclComm_t)c->nccl_comm;
        if (!N || !comm) return fail(JAC_ENCCL, "NCCL not initialised (jac_nccl_init)");
        ncclResult_t r = N->groupStart();
        for (const NcclFace &f : c->nccl_faces) {
            if (r == ncclSuccess) r = N->send(f.send, (size_t)f.count, ncclDouble, f.peer, comm, c->stream);
            if (r == ncclSuccess) r = N->recv(f.recv, (size_t)f.count, ncclDouble, f.peer, comm, c->stream);
        }
        const ncclResult_t r2 = N->groupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess)
            return fail(JAC_ENCCL, "ncclSend/ncclRecv: %s", N->errorString(r != ncclSuccess ? r : r2));
        CK(jac::launch_ghost_fill(sweep_args(c, src, jac::MODE_FUSED), 1 - src, c->stream));
        return JAC_OK;
    }
    if (!c->fused && (rc = enqueue_barrier(c))) return rc;  // fused: ordering is inside the sweep
    if ((c->flags & JAC_F_UNFUSED_PACK) && !(c->flags & JAC_F_SKIP_EXCHANGE)) {
        CK(jac::launch_ghost_fill(sweep_args(c, src, jac::MODE_PACK), 1 - src, c->stream));
        if ((rc = enqueue_barrier(c))) return rc;
    }
    return JAC_OK;
}

int build_graph(jac_ctx *c, int src, int n, cudaGraphExec_t *out)
{
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int rc = JAC_OK;
    for (int u = 0; u < n && rc == JAC_OK; ++u) rc = enqueue_iteration(c, src ^ (u & 1));
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (rc) { if (g) cudaGraphDestroy(g); return rc; }
    if (e != cudaSuccess) return fail(JAC_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(out, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(JAC_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    return JAC_OK;
}

int encode_tmap(jac_ctx *c)
{
    static PFN_encodeTiled encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess)
            return fail(JAC_ECUDA, "cuTensorMapEncodeTiled unavailable");
        encode = (PFN_encodeTiled)fn;
    }
    const jac::Geom &g = c->geom;
    const jac::TileShape ts = jac::tma_tile_shape(c->variant);
    const cuuint64_t dims[4] = {(cuuint64_t)g.P, (cuuint64_t)(g.ey + 2), (cuuint64_t)(g.ez + 2 * g.zg),
                                (cuuint64_t)(2 * c->nslots)};
    const cuuint64_t strides[3] = {(cuuint64_t)g.P * 8, (cuuint64_t)g.Q * 8, (cuuint64_t)g.bstride * 8};
    const cuuint32_t box[4] = {(cuuint32_t)ts.w, (cuuint32_t)(ts.by + 2), 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUtensorMapL2promotion promo = g.ex <= 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (const char *s = knob(c, "JAC_L2PROMO")) {  // experiment knob: 0, 64, 128, 256
        const int v = atoi(s);
        promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
              : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }
    CUresult r = encode(&c->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, c->arena, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(JAC_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return JAC_OK;
}

// Where the boundary layer of face f goes, for a neighbour block (global coords nb)
// hosted by this context, in buffer `buf`: its array base (y/z faces) or its x-ghost
// array on the side facing us (x faces).
double *block_ptr_local(const jac_ctx *c, const int32_t nb[3], int buf, int f)
{
    const jac::Plan &p = c->plan;
    const int32_t part = p.owner(nb[0], nb[1], nb[2]);
    const int32_t ls = p.local_slot(nb[0], nb[1], nb[2]);
    for (size_t h = 0; h < c->parts.size(); ++h)
        if (c->parts[h] == part) {
            const int slot = (int)h * p.blocks_per_part() + ls;
            if ((f >> 1) == 0) return jac::xg_array(c->xg, c->geom, buf, slot, jac::opposite(f) & 1);
            return c->slot_ptr(buf, slot);
        }
    return nullptr;
}

// Tile / work-list geometry for the current c->variant (ntx, nty, z-chunks, item
// count, column groups).  Called at create and for every autotune candidate.
// 2-D x band width in x tiles (64 points each); 0 = the whole block width.  Bands of
// 256 / 512 / 1024 tiles on 65536-131072-wide blocks were equal or slower (0 to +3.5%;
// profiles/r02_j2d_xband.txt): the wide-row penalty is not L2 reuse between y chunks.
constexpr int kXBandTiles = 0;

void configure_tiles(jac_ctx *c)
{
    const jac::Geom &g = c->geom;
    const uint32_t flags = c->flags;
    const int tbx = (c->variant == kPlain) ? 64 : jac::tma_tile_shape(c->variant).bx;
    const int tby = (c->variant == kPlain) ? 8 : jac::tma_tile_shape(c->variant).by;
    c->ntx = (g.ex + tbx - 1) / tbx;
    c->nty = (g.ey + tby - 1) / tby;
    // (plain kernel) z-chunk: enough CTAs for several waves on 148 SMs, chunks of >= 16 planes
    int zc = g.ez;
    const int64_t target = 148 * 4 * 4;
    while ((int64_t)c->nslots * c->ntx * c->nty * ((g.ez + zc - 1) / zc) < target && zc > 16) zc = (zc + 1) / 2;
    if (const char *s = knob(c, "JAC_ZC")) zc = std::max(1, std::min(g.ez, atoi(s)));
    c->zc = zc;
    c->ntz = (g.ez + zc - 1) / zc;
    // TMA kernel work list: columns cut into z-chunks of ~16 planes.  Short
    // chunks keep concurrently running CTAs at nearby z, so the x/y halo rows one
    // CTA stages are L2 hits for its neighbours (long marches drift apart and turn
    // the halos into DRAM re-reads: measured +19.6% reads at 256-plane chunks);
    // the price is 2 extra planes per chunk.
    c->ncols = c->nslots * c->ntx * c->nty;
    {
        const int resident = c->variant == kPlain ? 148 * 4 : jac::sweep_resident_ctas(c->variant);
        // 16 planes: measured best or within 2.5% of best on 512^3 (ODF 1-16), 768^3
        // and 1024^3 (64x16 tiles, 64x32 tiles were slower everywhere)
        int zchunk = 16;
        // small blocks: one item marches the whole block depth (32^3 blocks: 445 us
        // vs 469 at 16 planes; 64^3 blocks keep 16: 404 vs 414 us whole-depth)
        if (g.ez <= 32) zchunk = g.ez;
        // small grids (C1: 64^3): shorter chunks until the launch fills ~3/4 of a wave
        // (measured 24.5 -> 5.2 us per C1 iteration)
        while (zchunk > 2 && 4 * (int64_t)c->ncols * ((g.ez + zchunk - 1) / zchunk) < 3 * (int64_t)resident) zchunk /= 2;
        if (const char *s = knob(c, "JAC_ZCHUNK")) zchunk = std::max(1, atoi(s));
        c->nzc = std::max(1, (g.ez + zchunk - 1) / zchunk);
        c->nitems = c->ncols * c->nzc;
        // Column groups of 2 x SM-count columns: inside a group the chunk k+1 item of a
        // column launches soon after its chunk k item, so the two planes they share are
        // still in L2.  Measured (512^3, lean kernel): groups of 296 beat one resident
        // wave (444 / 592) by 1.3-2.5% at ODF 8-64 -- DRAM reads 1.14 vs 1.21 GB per
        // sweep at ODF 8 -- and 148 / 222 are equal or worse.
        int sms = 148;
        {
            int dev = 0;
            if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        }
        int gcols = 2 * sms;
        if (const char *s = knob(c, "JAC_GCOLS")) gcols = atoi(s);
        c->gcols = std::max(1, std::min(c->ncols, gcols > 0 ? gcols : c->ncols));
        if (flags & JAC_F_2D) {  // 2-D: items = (block, x tile, chunk of 8 y tiles), nzc = y chunks
            // 8 y tiles (128 rows) per item.  4 is 1.6-2.3% faster in the cold regime on
            // every width measured but 1-2% slower at the power-cap equilibrium (it holds
            // a 50-150 MHz lower clock), as 8-plane z-chunks are in 3-D
            // (profiles/r02_j2d_ychunk.txt, r02_zchunk.txt); JAC_YCHUNK overrides.
            int ytiles = 8;
            if (const char *s = knob(c, "JAC_YCHUNK")) ytiles = std::max(1, atoi(s));
            c->nzc = std::max(1, (c->nty + ytiles - 1) / ytiles);
            c->nitems = c->nslots * c->ntx * c->nzc;
            // x bands of <= XBAND_TILES x tiles (decode_item2d).
            int band = kXBandTiles;
            if (const char *s = knob(c, "JAC_XBAND")) band = atoi(s);
            if (band <= 0 || band >= c->ntx) band = c->ntx;
            const int nb = (c->ntx + band - 1) / band;
            c->gcols = (c->ntx + nb - 1) / nb;  // equal bands
        }
    }
}

int build_item_map(jac_ctx *c);

// Host <-> device transfers of the local box through two device staging slabs.  A slab
// is a run of whole planes (3-D) or rows (2-D) of the region, moved over PCIe by one
// pitched copy whose rows span the region's full width, then scattered into (gathered
// from) the blocks by a kernel; the copy of one slab overlaps the kernel of the other
// (copy stream + events).  One pitched copy per block instead ran the link at a quarter
// of its rate for 32^3 blocks (256-byte rows), and the dense rows' x ghosts needed a
// strided gather on the host.
constexpr int64_t kStageSlabBytes = 64ll << 20;

int ensure_staging(jac_ctx *c)
{
    if (c->stage[0]) return JAC_OK;
    int64_t lo[3], ex[3];
    jac_local_box(c, lo, ex);
    const int64_t unit = (ex[2] > 1 ? round_up(ex[0], 32) * ex[1] : round_up(ex[0], 32)) * 8;  // one plane / row
    const int64_t total = ex[0] * ex[1] * ex[2] * 8;
    int64_t slab = kStageSlabBytes;
    if (const char *v = knob(c, "JAC_STAGE_BYTES")) slab = std::max<int64_t>(1, atoll(v));  // tests: many slabs
    c->stage_pitched = knob(c, "JAC_STAGE_PITCHED") != nullptr;
    c->stage_direct = knob(c, "JAC_DIRECT") != nullptr;
    const size_t bytes = (size_t)round_up(std::max(unit, std::min(slab, total)), 256);
    void *p = nullptr;
    if (cudaMalloc(&p, 2 * bytes) != cudaSuccess)
        return fail(JAC_ENOMEM, "cudaMalloc(%zu bytes) for the host-transfer staging slabs", 2 * bytes);
    c->stage[0] = static_cast<double *>(p);
    c->stage[1] = c->stage[0] + bytes / 8;
    c->stage_bytes = bytes;
    CK(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
    for (cudaEvent_t &e : c->sev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    // block lists: a block meets at most ceil(extent / slab) + 1 slabs of the init region
    const jac::Geom &g = c->geom;
    const int64_t bext = ex[2] > 1 ? g.ez + 2 * g.zg : g.ey + 2;
    const int64_t per = std::max<int64_t>(1, (int64_t)bytes / unit);
    c->dlist_cap = (size_t)c->nslots * (size_t)((bext + per - 1) / per + 1);
    CK(cudaMalloc(&c->dlist, c->dlist_cap * sizeof(int32_t)));
    c->ranges.push_back({(unsigned long long)(uintptr_t)p, (unsigned long long)(uintptr_t)p + 2 * bytes});
    return upload_ranges(c);
}

// to_device: the ghost-inclusive local box of `hbox` -> both buffers of every local
// block (jac_set_init_box); else the interiors of the current buffer -> `hbox`
// (jac_get_field_box).  hbox covers the region (check_box).  Returns with the transfer
// queued on c->stream (to_device) or complete (else).
int staged_transfer(jac_ctx *c, bool to_device, double *hbox, const int64_t *origin, const int64_t *extent)
{
    const jac::Geom &g = c->geom;
    int rc;
    if ((rc = ensure_staging(c))) return rc;
    int64_t lo[3], ex[3];
    jac_local_box(c, lo, ex);
    if (!to_device)
        for (int k = 0; k < 3; ++k) {
            const int gh = k == 2 ? g.zg : 1;
            lo[k] += gh;
            ex[k] -= 2 * gh;
        }
    const int od = ex[2] > 1 ? 2 : 1;  // slab dimension: z (3-D), y (2-D or one interior plane)
    // Copy shape per slab, from the host box's layout: a region whose rows and planes
    // are the box's is one contiguous run (one linear copy); full rows of partial planes
    // are one run per plane (a 2-D copy of plane-sized rows); partial rows take a
    // pitched copy per row into 256-byte aligned staging rows.  Host-to-device pitched
    // copies of ~4 KB rows ran at 57% of the link rate (34.4 vs 19.8 ms per 512^3
    // init); linear runs at the rate of a plain copy.
    const bool full_rows = ex[0] == extent[0] && !c->stage_pitched;
    const bool contiguous = full_rows && (od == 1 || ex[1] == extent[1]);
    const int64_t pitch = full_rows ? ex[0] : round_up(ex[0], 32);
    const int64_t unit = (od == 2 ? pitch * ex[1] : pitch) * 8;
#ifndef JAC_CHECKED
    // Partial host rows into the device: a pinned (mapped) host box is read by the
    // scatter kernel itself over PCIe, one launch, no staging -- 44 GB/s, where pitched
    // copies of the rows reach 32 GB/s (linear slab copies: 55 GB/s, so full rows stay
    // staged; read-back stays staged too: 37 GB/s direct vs 52 GB/s pitched).
    // JAC_DIRECT=1 (experiment) takes this path for every pinned box.
    cudaPointerAttributes pa{};
    if ((c->stage_direct || (to_device && !full_rows)) && cudaPointerGetAttributes(&pa, hbox) == cudaSuccess &&
        pa.type == cudaMemoryTypeHost && pa.devicePointer) {
        std::vector<int32_t> all(c->nslots);
        for (int32_t t = 0; t < c->nslots; ++t) all[t] = t;
        CK(cudaMemcpy(c->dlist, all.data(), all.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        jac::StageBox sb;
        for (int k = 0; k < 3; ++k) { sb.o[k] = origin[k]; sb.n[k] = extent[k]; }
        sb.pitch = extent[0];
        const int64_t rows = (int64_t)(g.ey + 2) * (g.ez + 2 * g.zg);
        double *dev_view = static_cast<double *>(pa.devicePointer);
        const jac::SweepArgs a = sweep_args(c, 0, 0);
        if (to_device) CK(jac::launch_stage_scatter(a, c->dlist, c->nslots, rows, dev_view, sb, c->stream));
        else {
            CK(jac::launch_stage_gather(a, c->dlist, c->nslots, rows, dev_view, sb, (int)(c->iters & 1), c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
        return JAC_OK;
    }
#endif
    const int64_t per = std::max<int64_t>(1, (int64_t)c->stage_bytes / unit);
    const int64_t nslab = (ex[od] + per - 1) / per;
    // the blocks whose ghost-inclusive range meets each slab (indices into the table),
    // from the table sorted by origin along the slab dimension
    const int64_t bext[3] = {g.ex + 2, g.ey + 2, g.ez + 2 * g.zg};
    std::vector<int32_t> &order = c->by_origin[od];
    if (order.size() != (size_t)c->nslots) {
        order.resize(c->nslots);
        for (int32_t t = 0; t < c->nslots; ++t) order[t] = t;
        std::stable_sort(order.begin(), order.end(),
                         [&](int32_t x, int32_t y) { return c->hblocks[x].org[od] < c->hblocks[y].org[od]; });
    }
    std::vector<int32_t> list;
    std::vector<int64_t> first((size_t)nslab + 1, 0);
    for (int64_t i = 0; i < nslab; ++i) {
        first[i] = (int64_t)list.size();
        const int64_t s0 = lo[od] + i * per, s1 = std::min(s0 + per, lo[od] + ex[od]);
        // origins in (s0 - bext, s1)
        auto it = std::lower_bound(order.begin(), order.end(), s0 - bext[od] + 1,
                                   [&](int32_t t, int64_t v) { return c->hblocks[t].org[od] < v; });
        for (; it != order.end() && c->hblocks[*it].org[od] < s1; ++it) list.push_back(*it);
    }
    first[nslab] = (int64_t)list.size();
    if (list.size() > c->dlist_cap) {
        if (c->dlist) CK(cudaFree(c->dlist));
        c->dlist = nullptr;
        CK(cudaMalloc(&c->dlist, list.size() * sizeof(int32_t)));
        c->dlist_cap = list.size();
    }
    if (!list.empty()) CK(cudaMemcpy(c->dlist, list.data(), list.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    const jac::SweepArgs a = sweep_args(c, 0, 0);
    cudaEvent_t *filled = c->sev, *drained = c->sev + 2;
    // both slabs start free, after everything already queued on the main stream
    CK(cudaEventRecord(drained[0], c->stream));
    CK(cudaEventRecord(drained[1], c->stream));
    const int cur = (int)(c->iters & 1);
    const cudaPitchedPtr hp = make_cudaPitchedPtr(hbox, (size_t)extent[0] * 8, (size_t)extent[0], (size_t)extent[1]);
    for (int64_t i = 0; i < nslab; ++i) {
        const int b = (int)(i & 1);
        jac::StageBox sb;
        for (int k = 0; k < 3; ++k) { sb.o[k] = lo[k]; sb.n[k] = ex[k]; }
        sb.pitch = pitch;
        sb.o[od] = lo[od] + i * per;
        sb.n[od] = std::min(per, lo[od] + ex[od] - sb.o[od]);
        const int64_t rows = std::min(bext[1], sb.n[1]) * std::min(bext[2], sb.n[2]);  // per block, at most
        const int32_t *L = c->dlist + first[i];
        const int32_t nl = (int32_t)(first[i + 1] - first[i]);
        cudaMemcpy3DParms m{};
        const cudaPitchedPtr dp = make_cudaPitchedPtr(c->stage[b], (size_t)pitch * 8, (size_t)sb.n[0], (size_t)sb.n[1]);
        const cudaPos hpos = make_cudaPos((size_t)(sb.o[0] - origin[0]) * 8, (size_t)(sb.o[1] - origin[1]),
                                          (size_t)(sb.o[2] - origin[2]));
        m.extent = make_cudaExtent((size_t)sb.n[0] * 8, (size_t)sb.n[1], (size_t)sb.n[2]);
        double *hrun = hbox + ((sb.o[2] - origin[2]) * extent[1] + (sb.o[1] - origin[1])) * extent[0] + (sb.o[0] - origin[0]);
        const size_t run = (size_t)(sb.n[0] * sb.n[1] * sb.n[2]) * 8;  // contiguous: the slab's bytes
        const size_t plane_run = (size_t)(sb.n[0] * sb.n[1]) * 8;        // full rows: one plane's rows
        if (to_device) {
            CK(cudaStreamWaitEvent(c->cstream, drained[b], 0));
            m.srcPtr = hp;
            m.srcPos = hpos;
            m.dstPtr = dp;
            m.kind = cudaMemcpyHostToDevice;
            if (contiguous) CK(cudaMemcpyAsync(c->stage[b], hrun, run, cudaMemcpyHostToDevice, c->cstream));
            else if (full_rows)  // one run of sb.n[1] rows per plane
                CK(cudaMemcpy2DAsync(c->stage[b], plane_run, hrun, (size_t)(extent[1] * extent[0]) * 8, plane_run,
                                     (size_t)sb.n[2], cudaMemcpyHostToDevice, c->cstream));
            else CK(cudaMemcpy3DAsync(&m, c->cstream));
            CK(cudaEventRecord(filled[b], c->cstream));
            CK(cudaStreamWaitEvent(c->stream, filled[b], 0));
            CK(jac::launch_stage_scatter(a, L, nl, rows, c->stage[b], sb, c->stream));
            CK(cudaEventRecord(drained[b], c->stream));
        } else {
            CK(cudaStreamWaitEvent(c->stream, drained[b], 0));
            CK(jac::launch_stage_gather(a, L, nl, rows, c->stage[b], sb, cur, c->stream));
            CK(cudaEventRecord(filled[b], c->stream));
            CK(cudaStreamWaitEvent(c->cstream, filled[b], 0));
            m.srcPtr = dp;
            m.dstPtr = hp;
            m.dstPos = hpos;
            m.kind = cudaMemcpyDeviceToHost;
            if (contiguous) CK(cudaMemcpyAsync(hrun, c->stage[b], run, cudaMemcpyDeviceToHost, c->cstream));
            else if (full_rows)
                CK(cudaMemcpy2DAsync(hrun, (size_t)(extent[1] * extent[0]) * 8, c->stage[b], plane_run, plane_run,
                                     (size_t)sb.n[2], cudaMemcpyDeviceToHost, c->cstream));
            else CK(cudaMemcpy3DAsync(&m, c->cstream));
            CK(cudaEventRecord(drained[b], c->cstream));
        }
    }
    if (!to_device) CK(cudaStreamSynchronize(c->cstream));
    return JAC_OK;
}

// Autotune of the wide tile's TMA ring depth (6 stages at 3 CTAs / SM vs 4 stages at
// 4 CTAs / SM) on the context's own decomposition, GPU and data: 1 + 8 sweeps each,
// exchange off, the faster wins (ties within 0.5%: 6 stages).  Measured with the lean
// z-march: 3-D 512^3 ODF 1 and 8 within 0.6% either way (a few boxes: 4 stages 2%
// faster), ODF 16 / 64 6 stages 1.5% / 3% faster.  2-D takes 4 stages without timing:
// 5% faster on every box and in both power regimes (2614 vs 2742 us per 32768^2 sweep).
// Results are bit-identical either way.  JAC_AUTOTUNE=0 (6 stages) or JAC_VARIANT skip it.
// At create: the fixed choices (2-D: 4 stages); whether the 3-D wide tile is timed.
int autotune_at_create(jac_ctx *c)
{
    c->tuned = true;
    if (c->variant != jac::TMA_WIDE || knob(c, "JAC_VARIANT")) return JAC_OK;
    if (c->flags & JAC_F_2D) {  // 2-D: 4 stages measured 5% faster on every box, both regimes
        c->variant = jac::TMA_WIDE4;
        configure_tiles(c);
        return JAC_OK;
    }
    if (const char *s = knob(c, "JAC_AUTOTUNE"); s && atoi(s) == 0) return JAC_OK;
    c->tuned = false;  // timed at the first jac_step / jac_profile_sweep, on the initial field
    return JAC_OK;
}

// The timing itself, run once before the first graph is built: both ring depths sweep
// the context's own initialised field (MODE_NOEXCHANGE reads the current buffer and
// writes only the other buffer's interiors, which the next real sweep overwrites
// whole; no ghost, shell or neighbour memory is touched), so the choice is made on real
// data and in the state the run will be in, not on the zeroed arena of jac_create.
int autotune(jac_ctx *c)
{
    if (c->tuned) return JAC_OK;
    c->tuned = true;
    const int src = (int)(c->iters & 1);
    const int before = c->variant;
    const int cands[2] = {jac::TMA_WIDE, jac::TMA_WIDE4};
    float ms_of[2] = {0.f, 0.f};
    for (int n = 0; n < 2; ++n) {
        const int v = cands[n];
        c->variant = v;
        configure_tiles(c);
        if (jac::prepare_sweep_tma(v) != cudaSuccess || jac::prepare_sweep2d_tma(v) != cudaSuccess)
            return fail(JAC_ECUDA, "autotune: kernel attribute");
        const jac::SweepArgs a = sweep_args(c, src, jac::MODE_NOEXCHANGE);
        auto launch = [&]() {
            return (c->flags & JAC_F_2D) ? jac::launch_sweep2d_tma(c->tmap, a, v, c->stream)
                                         : jac::launch_sweep_tma(c->tmap, a, v, c->stream);
        };
        CK(launch());
        CK(cudaEventRecord(c->ev0, c->stream));
        for (int r = 0; r < 8; ++r) CK(launch());
        CK(cudaEventRecord(c->ev1, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaEventElapsedTime(&ms_of[n], c->ev0, c->ev1));
        c->tuned_ms[n] = ms_of[n] / 8;
    }
    // ties (< 0.5%) go to the usual winner, 6 stages
    c->variant = (ms_of[1] < 0.995f * ms_of[0]) ? jac::TMA_WIDE4 : jac::TMA_WIDE;
    configure_tiles(c);
    if (c->variant != before) {  // the launch order depends on the tile list
        int rc;
        if ((rc = build_item_map(c))) return rc;
        for (size_t h = 0; h < c->hsync.size(); ++h) c->hsync[h].nremote = c->nremote_part[h];
        CK(cudaMemcpy(c->dsync, c->hsync.data(), sizeof(jac::PartSync) * c->hsync.size(), cudaMemcpyHostToDevice));
    }
    return JAC_OK;
}

// Launch order for the fused cross-rank sync: the items touching a face in mask[b]
// first (their completion releases the neighbour ranks), then -- partners -- the 3-D
// items sharing a staged halo (x/y neighbour column, z neighbour chunk) with one of
// them, then the rest, each class in the natural order.  *n_first = first class size.
std::vector<int32_t> remote_first_order(jac_ctx *c, const std::vector<uint32_t> &mask, bool partners,
                                        int32_t *n_first, std::vector<int32_t> *first_per_part = nullptr)
{
    const jac::SweepArgs a0 = sweep_args(c, 0, jac::MODE_NOEXCHANGE);
    const jac::TileShape ts = jac::tma_tile_shape(c->variant);
    const bool two_d = (c->flags & JAC_F_2D) != 0;
    std::vector<jac::TileItem> items(c->nitems);
    std::vector<char> cls(c->nitems, 2);
    for (int32_t it = 0; it < c->nitems; ++it) {
        items[it] = two_d ? jac::decode_item2d(a0, it, ts.bx, ts.by) : jac::decode_item3d(a0, it, ts.bx, ts.by);
        if (jac::item_touches(a0, items[it], mask[items[it].b], ts.bx, ts.by, two_d)) cls[it] = 0;
    }
    if (partners && !two_d) {
        auto key = [](int64_t b, int64_t x0, int64_t y0, int64_t z) {
            return (uint64_t)((b << 48) | (x0 << 32) | (y0 << 16) | z);
        };
        std::unordered_map<uint64_t, int32_t> by_start, by_end;
        for (int32_t it = 0; it < c->nitems; ++it) {
            const jac::TileItem &t = items[it];
            by_start[key(t.b, t.x0, t.y0, t.zs)] = it;
            by_end[key(t.b, t.x0, t.y0, t.ze)] = it;
        }
        auto mark = [&](std::unordered_map<uint64_t, int32_t> &m, uint64_t k) {
            auto f = m.find(k);
            if (f != m.end() && cls[f->second] == 2) cls[f->second] = 1;
        };
        for (int32_t it = 0; it < c->nitems; ++it) {
            if (cls[it] != 0) continue;
            const jac::TileItem &t = items[it];
            mark(by_start, key(t.b, t.x0, t.y0, t.ze));  // z+ neighbour chunk
            mark(by_end, key(t.b, t.x0, t.y0, t.zs));    // z- neighbour chunk
            if (t.x0 >= ts.bx) mark(by_start, key(t.b, t.x0 - ts.bx, t.y0, t.zs));
            mark(by_start, key(t.b, t.x0 + ts.bx, t.y0, t.zs));
            if (t.y0 >= ts.by) mark(by_start, key(t.b, t.x0, t.y0 - ts.by, t.zs));
            mark(by_start, key(t.b, t.x0, t.y0 + ts.by, t.zs));
        }
    }
    std::vector<int32_t> order;
    order.reserve(c->nitems);
    for (char k = 0; k < 3; ++k)
        for (int32_t it = 0; it < c->nitems; ++it)
            if (cls[it] == k) order.push_back(it);
    *n_first = (int32_t)std::count(cls.begin(), cls.end(), (char)0);
    if (first_per_part) {  // class-0 items per hosted partition (PartSync::nremote)
        first_per_part->assign(c->parts.size(), 0);
        for (int32_t it = 0; it < c->nitems; ++it)
            if (cls[it] == 0) (*first_per_part)[c->hblocks[items[it].b].part]++;
    }
    return order;
}

// Launch order of the sweep's work items (depends on the tile variant): with fused
// cross-partition ordering, the remote-touching items (marked ~item) spread over the
// first quarter; sets c->fused, c->nremote and the per-partition remote item counts.
int build_item_map(jac_ctx *c)
{
    c->fused = (c->rank_mode || c->virtual_parts) && c->has_remote() && sweep_mode(c) == jac::MODE_FUSED &&
               c->variant != kPlain && !(c->flags & (JAC_F_NCCL | JAC_F_PER_BLOCK)) && !knob(c, "JAC_NO_FUSED_SYNC");
    // experiment knob (single-GPU contexts): the remote-first launch order of a rank
    // whose z- and y- faces were remote, without any sync -- isolates the cost of the
    // order itself.  1 = remote-first, 2 = remote-first + halo partners.
    const int order_exp = (!c->rank_mode && !c->virtual_parts && knob(c, "JAC_ORDER_EXP")) ? atoi(knob(c, "JAC_ORDER_EXP")) : 0;
    std::vector<int32_t> &nremote_part = c->nremote_part;
    nremote_part.assign(c->parts.size(), 0);
    c->nremote = 0;
    if (c->ditem_map) { cudaFree(c->ditem_map); c->ditem_map = nullptr; }
    if (c->fused || (order_exp && c->variant != kPlain)) {
        std::vector<uint32_t> mask(c->nslots);
        for (int32_t sl = 0; sl < c->nslots; ++sl)
            mask[sl] = c->fused ? c->hblocks[sl].remote_mask
                                : (((c->hblocks[sl].org[2] == 0) ? 1u << jac::ZM : 0u) |
                                   ((c->hblocks[sl].org[1] == 0) ? 1u << jac::YM : 0u));
        // remote-touching items first: their signal leaves early in the sweep, so the
        // next sweep's remote items (which wait for it) find it already set
        int32_t nfirst = 0;
        std::vector<int32_t> order = remote_first_order(c, mask, order_exp == 2, &nfirst, &nremote_part);
        if (c->fused) {
            c->nremote = nfirst;
            // remote-touching items are marked in the map (~item): they wait before their
            // first staging copy and signal after their last store
            // experiment: remote items column-major (all z-chunks of a column back to back,
            // so consecutive chunks share their overlap planes in L2) instead of the natural
            // chunk-major order
            if (knob(c, "JAC_REMOTE_COLMAJOR") && !(c->flags & JAC_F_2D)) {
                const jac::SweepArgs a0 = sweep_args(c, 0, jac::MODE_NOEXCHANGE);
                const jac::TileShape ts = jac::tma_tile_shape(c->variant);
                auto colkey = [&](int32_t it) {
                    const jac::TileItem t = jac::decode_item3d(a0, it, ts.bx, ts.by);
                    return std::make_tuple(t.b, t.y0, t.x0, t.zs);
                };
                std::stable_sort(order.begin(), order.begin() + nfirst,
                                 [&](int32_t x, int32_t y) { return colkey(x) < colkey(y); });
            }
            for (int32_t i = 0; i < nfirst; ++i) order[i] = ~order[i];
            // The remote items are spread evenly over the first quarter of the launch order
            // rather than all launched first: their signal still leaves early (the next
            // sweep's waits stay short), but the first waves no longer consist only of
            // scattered face items that lose their halo partners' L2 reuse and all store
            // over NVLink at once.  Same-box A/B at N = 4 (profiles/r02_remote_spread.txt):
            // C2 ODF 8 0.3461 -> 0.3374-0.3382 ms/iter, ODF 64 -2.0%, C3 -1.3%, C4 ODF 16
            // -0.8%, C5 -0.8%; N = 2 neutral.  JAC_REMOTE_SPREAD=<percent> (0 = all first).
            double f = 0.25;
            if (const char *sp = knob(c, "JAC_REMOTE_SPREAD")) f = std::min(1.0, std::max(0.0, atof(sp) / 100.0));
            if (f > 0 && nfirst > 0 && nfirst < c->nitems) {
                const int64_t span = std::max<int64_t>(nfirst, (int64_t)(f * c->nitems));
                std::vector<int32_t> spread;
                spread.reserve(order.size());
                int32_t r = 0, o = nfirst;
                for (int64_t pos = 0; pos < (int64_t)order.size(); ++pos) {
                    const bool take_remote = r < nfirst && (pos >= span - (nfirst - r) ||
                                                            pos * nfirst >= (int64_t)r * span);
                    spread.push_back(take_remote ? order[r++] : order[o++]);
                }
                order.swap(spread);
            }
        }
        if (cudaMalloc(&c->ditem_map, sizeof(int32_t) * order.size()) != cudaSuccess ||
            cudaMemcpy(c->ditem_map, order.data(), sizeof(int32_t) * order.size(), cudaMemcpyHostToDevice) != cudaSuccess)
            return fail(JAC_ENOMEM, "item map");
        if (c->fused && c->nremote == 0) c->fused = false;
    }
    return JAC_OK;
}

int create_common(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz,
                  int32_t n_gpus, const int32_t *gpu_grid, bool rank_mode, int32_t rank,
                  int32_t device, uint32_t flags, jac_ctx **out)
{
    if (!out) return fail(JAC_EINVAL, "out is NULL");
    *out = nullptr;
    jac::Plan plan;
    std::string err;
    int rc = jac::make_plan(nx, ny, nz, bx, by, bz, n_gpus, gpu_grid, &plan, &err);
    if (rc) return fail(rc, "%s", err.c_str());
    if ((flags & JAC_F_NCCL) && (!(rank_mode || (flags & JAC_F_VIRTUAL_GPUS)) ||
                                 (flags & (JAC_F_UNFUSED_PACK | JAC_F_PER_BLOCK | JAC_F_SKIP_EXCHANGE | JAC_F_NO_TMA))))
        return fail(JAC_EINVAL, "flags: JAC_F_NCCL needs a rank context (jac_create_rank) or JAC_F_VIRTUAL_GPUS, "
                                "and the fused TMA sweep");
    if ((flags & JAC_F_2D) && (nz != 1 || bz != 1))
        return fail(JAC_EINVAL, "flags: JAC_F_2D needs nz == 1 and bz == 1 (the 2-D grid is nx x ny)");
    if ((flags & JAC_F_2D) && (flags & (JAC_F_UNFUSED_PACK | JAC_F_NO_TMA)))
        return fail(JAC_EINVAL, "flags: JAC_F_2D runs the TMA path (no UNFUSED_PACK / NO_TMA)");
    if ((flags & JAC_F_PER_BLOCK) && (rank_mode || (flags & (JAC_F_UNFUSED_PACK | JAC_F_SKIP_EXCHANGE))))
        return fail(JAC_EINVAL, "flags: JAC_F_PER_BLOCK runs on one GPU (not a rank context) and excludes "
                                "JAC_F_UNFUSED_PACK / JAC_F_SKIP_EXCHANGE");
    const bool virt = (flags & JAC_F_VIRTUAL_GPUS) != 0;
    if (rank_mode) {
        if (rank < 0 || rank >= n_gpus) return fail(JAC_EINVAL, "rank %d out of [0,%d)", rank, n_gpus);
        if (virt) return fail(JAC_EINVAL, "flags: JAC_F_VIRTUAL_GPUS is not valid for rank contexts");
    } else if (n_gpus > 1 && !virt) {
        return fail(JAC_EINVAL, "internal: multi-device contexts are groups of rank contexts");
    }
    if ((flags & JAC_F_PER_BLOCK) && n_gpus > 1)
        return fail(JAC_EINVAL, "flags: JAC_F_PER_BLOCK runs one partition on one GPU (n_gpus == 1)");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev < 1) return fail(JAC_EDEVICE, "no CUDA device (%s)", cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(JAC_EDEVICE, "device %d not present (%d devices)", device, ndev);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(JAC_EDEVICE, "device %d is sm_%d%d, this library is built for sm_100a", device, prop.major, prop.minor);
    CK(cudaSetDevice(device));

    jac_ctx *c = new jac_ctx();
    c->plan = plan;
    c->flags = flags;
    c->rank_mode = rank_mode;
    c->virtual_parts = virt && n_gpus > 1;
    c->rank = rank;
    c->device = device;
    if (rank_mode) c->parts = {rank};
    else for (int32_t g = 0; g < n_gpus; ++g) c->parts.push_back(g);
    const int32_t bpp = plan.blocks_per_part();
    c->nslots = (int32_t)c->parts.size() * bpp;

    // geometry (device.hpp layout)
    jac::Geom &g = c->geom;
    g.ex = (int32_t)plan.e[0]; g.ey = (int32_t)plan.e[1]; g.ez = (int32_t)plan.e[2];
    // Narrow blocks (ex <= 64): interior on a 64-byte boundary and 64-byte row pitch,
    // read through a 64-byte-promoted tensor map, so DRAM fetches (64-byte granules)
    // carry no row padding / inline-ghost sectors: 32^3 blocks read 1.21x instead of
    // 1.49x the interior, 475 -> 459 us per 512^3 sweep.  Wide blocks keep A = 4
    // (the padding is a few percent of a row; measured equal or better).
    const bool narrow = g.ex <= 64;
    g.A = narrow ? 2 * jac::kA : jac::kA;
    if (const char *s = knob(c, "JAC_A")) g.A = std::max(2, atoi(s) & ~1);  // layout experiment knob
    int palign = narrow ? 8 : 4;
    if (const char *s = knob(c, "JAC_PALIGN")) palign = std::max(4, atoi(s) & ~3);  // layout experiment knob
    g.P = round_up(g.A + g.ex + 4, palign);  // room for the 32-byte +x ghost sector (A % 4 == 0)
    // Dense rows (3-D, ex % 8 == 0): no padding and no inline ghost columns at all --
    // A = 0, P = ex -- so a block's rows are back to back, 64-byte aligned, and the
    // staged boxes are contiguous DRAM runs.  The x ghosts live in the x-ghost arrays
    // anyway; init fills them directly (jac_set_init_box, hash_init_kernel).  Same-box
    // A/B per sweep: 512^3 in 32^3 blocks 441.6 -> 411.4 us; ODF 1 336 -> 330 us;
    // ODF 8 -2%; ODF 64 365 -> 350 us; 1536^3 ODF 16 -2.6..4.7%.  JAC_NO_DENSE=1 keeps
    // the padded rows.
    if (!(flags & JAC_F_2D) && g.ex % 8 == 0 && !knob(c, "JAC_NO_DENSE")) {
        g.A = 0;
        g.P = g.ex;
    }
    g.Q = g.P * (g.ey + 2);
    g.zg = (flags & JAC_F_2D) ? 0 : 1;
    g.bstride = round_up(g.Q * (g.ez + 2 * g.zg), 32);
    g.nslots = c->nslots;
    g.eyp = (int32_t)round_up(g.ey, 4);
    g.xgstride = round_up((int64_t)g.eyp * g.ez + jac::kXgPad, 32);
    // face buffer sizes (x faces in the x-ghost layout, pitch eyp: JAC_F_NCCL packs them so)
    const int64_t fx = (int64_t)g.eyp * g.ez, fy = (int64_t)g.ex * g.ez, fz = (int64_t)g.ex * g.ey;
    int64_t o = 0;
    const int64_t fsz[6] = {fx, fx, fy, fy, fz, fz};
    for (int f = 0; f < 6; ++f) { g.ooff[f] = o; o += round_up(fsz[f], 4); }
    g.ostride = (flags & (JAC_F_UNFUSED_PACK | JAC_F_PER_BLOCK | JAC_F_NCCL)) ? round_up(o, 32) : 0;

    // tile shape / variant
    if (flags & JAC_F_NO_TMA) c->variant = kPlain;
    // (32-wide blocks: 32 x 16 tiles; the 32 x 32 tile won only while y-face rows
    // took the general epilogue -- lean y faces: 445 vs 462 us for 512^3 in 32^3 blocks)
    // (64-wide blocks: 6-stage ring, 377-379 vs 399-409 us for 512^3 in 64^3 blocks;
    // 32-wide blocks: 6 stages within noise of 4, which stay)
    // 32-wide blocks of a large grid take a whole 32 x 32 face per item (half the items
    // of 32 x 16 tiles, so half the per-item prologues and ring fills): 1024^3 in 32^3
    // blocks 3.28-3.33 -> 3.09 ms, 512^3 in 32^3 blocks 396-398 -> 392 us.  Small grids
    // (launch / latency bound: C1 3.9 vs 4.1 us) and rows not a multiple of 32 (ragged
    // 22-row blocks 4.3 vs 5.1 us) keep the 32 x 16 tile (profiles/r02_tile_variants.txt).
    else if (g.ex <= 32) {
        const bool tall = g.ey % 32 == 0 && (int64_t)c->nslots * g.ex * g.ey * g.ez >= (int64_t)1 << 24;
        c->variant = tall ? jac::TMA_EXACT32_TALL : jac::TMA_EXACT32;
    } else c->variant = (g.ex <= 64) ? jac::TMA_EXACT64_6 : jac::TMA_WIDE;
    if (const char *s = knob(c, "JAC_VARIANT"); s && c->variant != kPlain) {
        const int v = atoi(s);  // tuning knob; EXACT* only where one tile spans the block row
        if (v == jac::TMA_WIDE || v == jac::TMA_WIDE4 || v == jac::TMA_NARROW || v == jac::TMA_WIDE_TALL ||
            ((v == jac::TMA_EXACT32 || v == jac::TMA_EXACT32_TALL || v == jac::TMA_EXACT32_6) && g.ex <= 32) ||
            ((v == jac::TMA_EXACT64 || v == jac::TMA_EXACT64_6) && g.ex <= 64))
            c->variant = v;
    }
    configure_tiles(c);
    if (knob(c, "JAC_NO_CTA_SYSFENCE")) c->exp_bits |= jac::kExpNoCtaSysFence;  // UNSAFE timing experiment
    if (const char *s = knob(c, "JAC_UNROLL")) c->unroll = std::max(2, atoi(s) & ~1);
    if (const char *s = knob(c, "JAC_PDL")) c->pdl = atoi(s) != 0;
    if ((int64_t)c->nslots * c->ntx * c->nty * c->ntz > 0x7fffffffLL) {
        delete c;
        return fail(JAC_EINVAL, "too many tiles for one launch");
    }

    // allocation: [ctrl: one PartSync word block per hosted partition][arena][x-ghost
    // arrays][outbox]
    c->ctrl_off = 0;
    c->ctrl_stride = round_up((int64_t)n_gpus + 2, 16);
    c->arena_off = (size_t)round_up(std::max<int64_t>(65536, (int64_t)c->parts.size() * c->ctrl_stride * 8), 65536);
    const size_t arena_bytes = (size_t)2 * c->nslots * g.bstride * sizeof(double);
    c->xg_off = c->arena_off + arena_bytes;
    const size_t xg_bytes = (size_t)2 * c->nslots * 2 * g.xgstride * sizeof(double);
    c->outbox_off = c->xg_off + xg_bytes;
    // outbox: one set of faces per block; JAC_F_PER_BLOCK double-buffers it by parity
    // (JAC_F_NCCL: send buffers then receive buffers)
    const size_t outbox_bytes = (size_t)((flags & (JAC_F_PER_BLOCK | JAC_F_NCCL)) ? 2 : 1) * c->nslots * g.ostride * sizeof(double);
    c->part_peers.assign(c->parts.size(), {});
    c->alloc_bytes = c->outbox_off + outbox_bytes;
    e = cudaMalloc(&c->alloc, c->alloc_bytes);
    if (e != cudaSuccess) {
        delete c;
        return fail(JAC_ENOMEM, "cudaMalloc(%zu bytes) for the block arena: %s", c->alloc_bytes, cudaGetErrorString(e));
    }
    c->ctrl = reinterpret_cast<uint64_t *>(c->alloc + c->ctrl_off);
    c->arena = reinterpret_cast<double *>(c->alloc + c->arena_off);
    c->xg = reinterpret_cast<double *>(c->alloc + c->xg_off);
    c->outbox = outbox_bytes ? reinterpret_cast<double *>(c->alloc + c->outbox_off) : nullptr;
    auto bail = [&](int code) { jac_destroy(c); return code; };
    if (cudaMemset(c->alloc, 0, c->alloc_bytes) != cudaSuccess) return bail(fail(JAC_ECUDA, "cudaMemset arena"));

    // descriptor table
    c->hblocks.resize(c->nslots);
    auto hosted = [&](int32_t part) {  // index of a partition among the hosted ones, or -1
        const auto it = std::find(c->parts.begin(), c->parts.end(), part);
        return it == c->parts.end() ? -1 : (int32_t)(it - c->parts.begin());
    };
    for (int32_t s = 0; s < c->nslots; ++s) {
        const int32_t h = s / bpp, part = c->parts[h], ls = s % bpp;
        int32_t blk[3];
        plan.block_of(part, ls, blk);
        jac::DevBlock &d = c->hblocks[s];
        memset(&d, 0, sizeof d);
        d.slot = s;
        d.part = h;
        for (int k = 0; k < 3; ++k) d.org[k] = (int32_t)(blk[k] * plan.e[k]);
        for (int f = 0; f < 6; ++f) {
            int32_t nb[3];
            if (!plan.neighbor(blk, f, nb)) continue;
            const int32_t owner = plan.owner(nb[0], nb[1], nb[2]);
            const int32_t oh = hosted(owner);
            const bool same_part = owner == part;
            if (same_part) c->local_faces++;
            else c->remote_faces++;
            const int64_t count = (f >> 1) == 0 ? fx : (f >> 1) == 1 ? fy : fz;
            if (!same_part) {
                c->remote_bytes += 8 * count;
                d.remote_mask |= 1u << f;
                auto &pp = c->part_peers[h];
                if (std::find(pp.begin(), pp.end(), owner) == pp.end()) pp.push_back(owner);
            }
            if (!same_part && (flags & JAC_F_NCCL)) {
                // pack into this block's send buffer; the batched ghost kernel unpacks the
                // receive buffer after the transport (grouped ncclSend / ncclRecv, or the
                // copy kernel between virtual partitions)
                d.pack_mask |= 1u << f;
                double *sendb = c->outbox + (int64_t)s * g.ostride + g.ooff[f];
                double *recvb = c->outbox + (int64_t)(c->nslots + s) * g.ostride + g.ooff[f];
                d.nb[f][0] = d.nb[f][1] = sendb;
                d.nb_out[f] = recvb;
                if (oh >= 0) {  // virtual: into the neighbour block's receive buffer
                    const int32_t ns = oh * bpp + plan.local_slot(nb[0], nb[1], nb[2]);
                    c->vcopies.push_back({sendb, c->outbox + (int64_t)(c->nslots + ns) * g.ostride +
                                                     g.ooff[jac::opposite(f)], count});
                    c->vcopy_max = std::max(c->vcopy_max, count);
                } else {
                    const int64_t gb = ((int64_t)blk[2] * plan.b[1] + blk[1]) * plan.b[0] + blk[0];
                    const int64_t gn = ((int64_t)nb[2] * plan.b[1] + nb[1]) * plan.b[0] + nb[0];
                    c->nccl_faces.push_back({owner, std::min(gb, gn) * 3 + (f >> 1), count, sendb, recvb});
                }
            } else if (oh >= 0) {
                // the neighbour's memory is in this allocation (same partition, or another
                // virtual partition): direct-to-ghost stores
                d.nb[f][0] = block_ptr_local(c, nb, 0, f);
                d.nb[f][1] = block_ptr_local(c, nb, 1, f);
                if (c->outbox && (flags & JAC_F_UNFUSED_PACK)) {
                    const int32_t ns = oh * bpp + plan.local_slot(nb[0], nb[1], nb[2]);
                    d.nb_out[f] = c->outbox + (int64_t)ns * g.ostride + g.ooff[jac::opposite(f)];
                }
            }
            // else: another rank's memory; pointers filled when the peers are connected
        }
    }
    for (const auto &pp : c->part_peers)
        if (pp.size() > 6) return bail(fail(JAC_EINVAL, "more than 6 neighbour partitions"));
#ifdef JAC_CHECKED
    // checker self-test (tests): the first local face of the table stores 1 MiB past the
    // end of the allocation; the checked kernels must report and skip those stores
    if (knob(c, "JAC_CHECK_SELFTEST")) {
        bool done = false;
        for (jac::DevBlock &d : c->hblocks)
            for (int f = 0; f < 6 && !done; ++f)
                if (d.nb[f][0] && !((d.remote_mask >> f) & 1u)) {
                    d.nb[f][0] = d.nb[f][1] = reinterpret_cast<double *>(c->alloc + c->alloc_bytes + (1 << 20));
                    done = true;
                }
    }
#endif
    // negative-control experiment (tests): faces between virtual partitions get no store
    // target, so a neighbour partition's ghosts go stale -- the result must differ
    if (c->virtual_parts && knob(c, "JAC_DROP_REMOTE"))
        for (jac::DevBlock &d : c->hblocks)
            for (int f = 0; f < 6; ++f)
                if ((d.remote_mask >> f) & 1u) d.nb[f][0] = d.nb[f][1] = nullptr;
    if ((int64_t)c->parts.size() * c->ctrl_stride > (int64_t)(c->arena_off / 8))
        return bail(fail(JAC_EINVAL, "n_gpus too large for the control block"));
    std::sort(c->nccl_faces.begin(), c->nccl_faces.end(), [](const NcclFace &x, const NcclFace &y) {
        return x.peer != y.peer ? x.peer < y.peer : x.key < y.key;  // same order on both sides
    });
    if (!c->vcopies.empty()) {
        if (c->vcopies.size() > 65535) return bail(fail(JAC_EINVAL, "too many virtual remote faces"));
        if (cudaMalloc(&c->dvcopies, sizeof(jac::FaceCopy) * c->vcopies.size()) != cudaSuccess ||
            cudaMemcpy(c->dvcopies, c->vcopies.data(), sizeof(jac::FaceCopy) * c->vcopies.size(),
                       cudaMemcpyHostToDevice) != cudaSuccess)
            return bail(fail(JAC_ENOMEM, "virtual transport list"));
    }
    if (cudaMalloc(&c->dblocks, sizeof(jac::DevBlock) * c->nslots) != cudaSuccess)
        return bail(fail(JAC_ENOMEM, "cudaMalloc descriptor table"));
    if (cudaMemcpy(c->dblocks, c->hblocks.data(), sizeof(jac::DevBlock) * c->nslots, cudaMemcpyHostToDevice) != cudaSuccess)
        return bail(fail(JAC_ECUDA, "descriptor table upload"));
    if (c->variant != kPlain) {
        if ((rc = encode_tmap(c))) return bail(rc);
        if (jac::prepare_sweep_tma(c->variant) != cudaSuccess) return bail(fail(JAC_ECUDA, "sweep kernel attribute"));
        if ((flags & JAC_F_2D) && jac::prepare_sweep2d_tma(c->variant) != cudaSuccess)
            return bail(fail(JAC_ECUDA, "2-D sweep kernel attribute"));
    }
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess)
        return bail(fail(JAC_ECUDA, "stream/event creation"));
    if (flags & JAC_F_PER_BLOCK) {
        c->bstreams.assign(c->nslots, nullptr);
        c->bevents.assign((size_t)2 * c->nslots, nullptr);
        for (auto &st : c->bstreams)
            if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
                return bail(fail(JAC_ECUDA, "per-block stream creation"));
        for (auto &ev : c->bevents)
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
                return bail(fail(JAC_ECUDA, "per-block event creation"));
    }
    if ((rc = autotune_at_create(c))) return bail(rc);
    if ((rc = build_item_map(c))) return bail(rc);
    // watchdog word of the cross-partition waits: mapped pinned host memory, read after
    // every synchronising call
    if (cudaHostAlloc(&c->status_h, 4 * sizeof(uint32_t), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&c->status_d, c->status_h, 0) != cudaSuccess)
        return bail(fail(JAC_ENOMEM, "watchdog status word"));
    for (int k = 0; k < 4; ++k) c->status_h[k] = 0;
    c->ranges.push_back({(unsigned long long)(uintptr_t)c->alloc, (unsigned long long)(uintptr_t)c->alloc + c->alloc_bytes});
    if ((rc = upload_ranges(c))) return bail(rc);
    if ((rc = ensure_staging(c))) return bail(rc);  // host-transfer slabs (adds its store range)
    // per-partition sync table: own control words; neighbours' flag slots are local
    // for virtual partitions, filled when the peers are connected for a rank context
    c->hsync.assign(c->parts.size(), jac::PartSync{});
    for (size_t h = 0; h < c->parts.size(); ++h) {
        jac::PartSync &ps = c->hsync[h];
        ps.ctrl = c->ctrl + (int64_t)h * c->ctrl_stride;
        ps.count = reinterpret_cast<unsigned long long *>(ps.ctrl + 1 + n_gpus);
        ps.npeers = (int32_t)c->part_peers[h].size();
        ps.nremote = c->nremote_part[h];
        // watchdog experiment (tests): partition 0 (the global id) never signals its sweeps
        if (c->parts[h] == 0 && knob(c, "JAC_HOLD_SIGNAL")) ps.nremote = 0x7fffffff;
        for (int n = 0; n < ps.npeers; ++n) {
            const int32_t q = c->part_peers[h][n];
            ps.peer_id[n] = q;
            const int32_t qh = hosted(q);
            if (qh >= 0) ps.peer_slot[n] = c->ctrl + (int64_t)qh * c->ctrl_stride + 1 + c->parts[h];
        }
    }
    if (cudaMalloc(&c->dsync, sizeof(jac::PartSync) * c->hsync.size()) != cudaSuccess ||
        cudaMemcpy(c->dsync, c->hsync.data(), sizeof(jac::PartSync) * c->hsync.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return bail(fail(JAC_ENOMEM, "partition sync table"));
    c->ipc_done = !rank_mode;
    *out = c;
    return JAC_OK;
}

// ---------------------------------------------------------------- paper-style mode
// One iteration t for the blocks b = first, first + stride, ...: on the block's own
// stream wait for every neighbour's pack of t-1, unpack each face, stencil, pack
// each face, record the block's event for parity t.
int enqueue_per_block(jac_ctx *c, int64_t t, int first, int stride)
{
    const int src = (int)(t & 1), dst = 1 - src, par = (int)(t & 1), ppar = 1 - par;
    jac::SweepArgs base = sweep_args(c, src, jac::MODE_NOEXCHANGE);
    for (int b = first; b < c->nslots; b += stride) {
        cudaStream_t s = c->bstreams[b];
        const jac::DevBlock &d = c->hblocks[b];
        int nbs[6];
        for (int f = 0; f < 6; ++f) {
            nbs[f] = -1;
            if (!d.nb[f][0]) continue;
            int32_t blk[3], nb[3];
            for (int k = 0; k < 3; ++k) blk[k] = (int32_t)(d.org[k] / c->plan.e[k]);
            c->plan.neighbor(blk, f, nb);
            const int32_t part = c->plan.owner(nb[0], nb[1], nb[2]);
            const int32_t h = (int32_t)(std::find(c->parts.begin(), c->parts.end(), part) - c->parts.begin());
            nbs[f] = h * c->plan.blocks_per_part() + c->plan.local_slot(nb[0], nb[1], nb[2]);
        }
        if (t > 0) {  // at t = 0 the ghosts come from jac_set_init*
            for (int f = 0; f < 6; ++f)
                if (nbs[f] >= 0) CK(cudaStreamWaitEvent(s, c->bevents[(size_t)nbs[f] * 2 + ppar], 0));
            for (int f = 0; f < 6; ++f)
                if (nbs[f] >= 0) CK(jac::launch_unpack_face(base, b, nbs[f], f, src, ppar, s));
        }
        jac::SweepArgs a = base;  // the stencil of this block alone
        a.blocks = c->dblocks + b;
        a.slot_base = b;
        a.ncols = c->ntx * c->nty;
        a.nitems = a.ncols * c->nzc;
        a.gcols = a.ncols;
        a.ntz = c->ntz;
        if (c->variant == kPlain) {
            CK(jac::launch_sweep_plain_one(a, s));
        } else if (c->flags & JAC_F_2D) {
            a.nitems = c->ntx * c->nzc;  // (x tile, y chunk) items of this block
            a.gcols = c->gcols;          // x band
            CK(jac::launch_sweep2d_tma(c->tmap, a, c->variant, s));
        } else {
            CK(jac::launch_sweep_tma(c->tmap, a, c->variant, s));
        }
        for (int f = 0; f < 6; ++f)
            if (nbs[f] >= 0) CK(jac::launch_pack_face(base, b, f, dst, par, s));
        CK(cudaEventRecord(c->bevents[(size_t)b * 2 + par], s));
    }
    return JAC_OK;
}

struct HostBarrier {
    std::mutex m;
    std::condition_variable cv;
    int n, waiting = 0;
    long gen = 0;
    explicit HostBarrier(int n_) : n(n_) {}
    void wait()
    {
        std::unique_lock<std::mutex> lk(m);
        const long g = gen;
        if (++waiting == n) { waiting = 0; ++gen; cv.notify_all(); }
        else cv.wait(lk, [&] { return gen != g; });
    }
};

int per_block_step(jac_ctx *c, int32_t n)
{
    for (cudaStream_t s : c->bstreams) CK(cudaStreamWaitEvent(s, c->ev0, 0));
    const int T = std::max(1, std::min(c->launch_threads, c->nslots));
    int rc = JAC_OK;
    if (T == 1) {
        for (int it = 0; it < n && rc == JAC_OK; ++it) rc = enqueue_per_block(c, c->iters + it, 0, 1);
    } else {
        HostBarrier bar(T);
        std::vector<int> rcs(T, JAC_OK);
        std::vector<std::string> errs(T);
        std::vector<std::thread> pes;
        for (int p = 0; p < T; ++p)
            pes.emplace_back([&, p] {
                cudaSetDevice(c->device);
                for (int it = 0; it < n; ++it) {
                    if (rcs[p] == JAC_OK) {
                        rcs[p] = enqueue_per_block(c, c->iters + it, p, T);
                        if (rcs[p]) errs[p] = g_err;
                    }
                    bar.wait();  // every block's event for parity t is recorded before t+1 waits on it
                }
            });
        for (auto &th : pes) th.join();
        for (int p = 0; p < T; ++p)
            if (rcs[p]) { g_err = errs[p]; return rcs[p]; }
    }
    if (rc) return rc;
    if (n > 0) {
        const int last = (int)((c->iters + n - 1) & 1);
        for (int b = 0; b < c->nslots; ++b) CK(cudaStreamWaitEvent(c->stream, c->bevents[(size_t)b * 2 + last], 0));
    }
    return JAC_OK;
}

int require_ready(const jac_ctx *c)
{
    if (!c) return fail(JAC_EINVAL, "ctx is NULL");
    if (c->rank_mode && !c->ipc_done) return fail(JAC_ESTATE, "rank context: call jac_import_ipc before init/step");
    return JAC_OK;
}

int local_slot_of(const jac_ctx *c, int32_t ix, int32_t iy, int32_t iz, int32_t *slot)
{
    const jac::Plan &p = c->plan;
    if (ix < 0 || iy < 0 || iz < 0 || ix >= p.b[0] || iy >= p.b[1] || iz >= p.b[2])
        return fail(JAC_EINVAL, "block index (%d,%d,%d) outside (%d,%d,%d)", ix, iy, iz, p.b[0], p.b[1], p.b[2]);
    const int32_t part = p.owner(ix, iy, iz);
    for (size_t h = 0; h < c->parts.size(); ++h)
        if (c->parts[h] == part) {
            *slot = (int32_t)h * p.blocks_per_part() + p.local_slot(ix, iy, iz);
            return JAC_OK;
        }
    return fail(JAC_EINVAL, "block (%d,%d,%d) is owned by partition %d, not by this context", ix, iy, iz, part);
}

int finish_init(jac_ctx *c)
{
    int rc;
    if ((rc = enqueue_barrier(c))) return rc;  // neighbours may write our ghosts only after this
    CK(cudaStreamSynchronize(c->stream));
    if ((rc = check_status(c))) return rc;
    c->inited = true;
    c->iters = 0;
    return JAC_OK;
}

// ---------------------------------------------------------------- jac_step phases
// jac_step = check, begin (graphs, start event), launches in chunks, end (stop event,
// synchronise, watchdog).  A group context runs the phases of its sub-contexts
// interleaved, chunk by chunk, so every device has its share queued before any host
// wait (the devices' sweeps wait on one another's flags).
int step_check(jac_ctx *c, int32_t n)
{
    int rc;
    if ((rc = require_ready(c))) return rc;
    if (n < 0) return fail(JAC_EINVAL, "n_iters = %d < 0", n);
    if (!c->inited) return fail(JAC_ESTATE, "jac_step before jac_set_init / jac_set_init_hash");
    return JAC_OK;
}

bool use_graphs(const jac_ctx *c) { return !(c->flags & (JAC_F_NO_GRAPH | JAC_F_PER_BLOCK)); }

// The slow, once-only part of a step's start: the deferred autotune and the graphs.
int step_prepare(jac_ctx *c)
{
    int rc;
    if ((rc = autotune(c))) return rc;
    if (use_graphs(c) && !c->g1[0]) {
        for (int s = 0; s < 2; ++s) {
            if ((rc = build_graph(c, s, 1, &c->g1[s]))) return rc;
            if ((rc = build_graph(c, s, c->unroll, &c->gU[s]))) return rc;
        }
    }
    return JAC_OK;
}

int step_begin(jac_ctx *c)
{
    int rc;
    if ((rc = step_prepare(c))) return rc;
    // Multi-GPU: the devices start a step at different times -- one process per GPU
    // enters jac_step tens to hundreds of microseconds apart after a host barrier, and a
    // single-process group launches its devices one after the other.  A device-side
    // neighbour barrier first aligns the GPUs, so the step's device time (CUDA events,
    // max over devices / ranks) measures the iterations, not the launch skew, which the
    // early devices' first sweeps would otherwise absorb waiting for the late ones'
    // signals (torchrun, C2 at N = 4: rank times 0.339-0.350 ms/iter before, 0.3384-0.3392
    // after; profiles/r02_scaling_same_lease.json).
    // The barrier is a neighbour barrier, so one round aligns only neighbours; after as
    // many rounds as the partition grid's diameter every partition has (transitively)
    // waited for every other (a 1x2x2 grid: 2 rounds; 2x2x2: 3).
    if (c->rank_mode && c->has_remote() && !(c->flags & JAC_F_NCCL)) {
        const int rounds = (c->plan.g[0] - 1) + (c->plan.g[1] - 1) + (c->plan.g[2] - 1);
        for (int r = 0; r < rounds; ++r)
            if ((rc = enqueue_barrier(c))) return rc;
    }
    CK(cudaEventRecord(c->ev0, c->stream));
    return JAC_OK;
}

// iterations the next launch covers: one unrolled graph, else one iteration
int32_t step_chunk(const jac_ctx *c, int32_t left) { return (use_graphs(c) && left >= c->unroll) ? c->unroll : 1; }

// Enqueues k iterations (k == unroll: the unrolled graph; k == 1) and advances the
// context's iteration count (the parity of the next launch).
int step_launch(jac_ctx *c, int32_t k)
{
    const int src = (int)(c->iters & 1);
    if (use_graphs(c)) {
        CK(cudaGraphLaunch(k == c->unroll ? c->gU[src] : c->g1[src], c->stream));
        c->graph_launches++;
    } else {
        int rc;
        if ((rc = enqueue_iteration(c, src))) return rc;
    }
    c->iters += k;
    c->kernel_launches += (int64_t)k * c->kernels_per_iter();
    return JAC_OK;
}

int step_end(jac_ctx *c, int32_t n)
{
    CK(cudaEventRecord(c->ev1, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    c->last_ms = ms;
    if (c->flags & JAC_F_PER_BLOCK) {  // per_block_step enqueued all n iterations
        c->iters += n;
        c->kernel_launches += (int64_t)n * c->kernels_per_iter();
    }
    return check_status(c);
}

// Rank context c: fills the REMOTE face pointers of the descriptor table and the
// neighbours' flag slots from the neighbour ranks' allocation bases (IPC-mapped
// memory of other processes, or plain peer pointers of a group's sub-contexts) and
// the layout offsets of their records.
int connect_peers(jac_ctx *c, const std::vector<char *> &base, const IpcRecord *recs)
{
    const jac::Plan &p = c->plan;
    const int32_t bpp = p.blocks_per_part();
    const jac::Geom &g = c->geom;
    for (int32_t s = 0; s < c->nslots; ++s) {
        int32_t blk[3];
        p.block_of(c->rank, s, blk);
        for (int f = 0; f < 6; ++f) {
            int32_t nb[3];
            if (!p.neighbor(blk, f, nb)) continue;
            const int32_t q = p.owner(nb[0], nb[1], nb[2]);
            if (q == c->rank) continue;
            const int32_t ns = p.local_slot(nb[0], nb[1], nb[2]);
            double *arena = reinterpret_cast<double *>(base[q] + recs[q].arena_off);
            double *xg = reinterpret_cast<double *>(base[q] + recs[q].xg_off);
            for (int buf = 0; buf < 2; ++buf)
                c->hblocks[s].nb[f][buf] = (f >> 1) == 0 ? jac::xg_array(xg, g, buf, ns, jac::opposite(f) & 1)
                                                         : arena + (int64_t)(buf * bpp + ns) * g.bstride;
            if (c->outbox) {
                const double *ob = reinterpret_cast<const double *>(base[q] + recs[q].outbox_off);
                c->hblocks[s].nb_out[f] = ob + (int64_t)ns * g.ostride + g.ooff[jac::opposite(f)];
            }
        }
    }
    jac::PartSync &ps = c->hsync[0];
    for (int n = 0; n < ps.npeers; ++n) {
        const int32_t q = ps.peer_id[n];
        uint64_t *pc = reinterpret_cast<uint64_t *>(base[q] + recs[q].ctrl_off);  // rank q hosts one partition
        ps.peer_slot[n] = pc + 1 + c->rank;
    }
    for (int n = 0; n < ps.npeers; ++n) {
        const int32_t q = ps.peer_id[n];
        c->ranges.push_back({(unsigned long long)(uintptr_t)base[q],
                             (unsigned long long)(uintptr_t)base[q] + recs[q].alloc_bytes});
    }
    int rc;
    if ((rc = upload_ranges(c))) return rc;
    CK(cudaMemcpy(c->dblocks, c->hblocks.data(), sizeof(jac::DevBlock) * c->nslots, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->dsync, c->hsync.data(), sizeof(jac::PartSync) * c->hsync.size(), cudaMemcpyHostToDevice));
    c->ipc_done = true;
    return JAC_OK;
}


// ---------------------------------------------------------------- group contexts
// jac_create(n_gpus > 1): one process drives every GPU.  The
// group holds one rank-mode sub-context per device -- partition g on device g -- and
// connects them with plain peer pointers (cudaDeviceEnablePeerAccess) instead of IPC
// records, so every sub-context runs exactly the rank path: in-sweep peer stores over
// NVLink and the device-flag handshake.  Calls fan out to the sub-contexts.

struct DeviceGuard {  // restores the caller's current device
    int dev = -1;
    DeviceGuard() { if (cudaGetDevice(&dev) != cudaSuccess) dev = -1; }
    ~DeviceGuard() { if (dev >= 0) cudaSetDevice(dev); }
};

// Runs fn(sub) on every sub-context concurrently, one host thread per device: the
// collective cold-path calls (init, profiling) contain cross-device barriers, so no
// device's call may wait for another's to return.  Returns the first error.
template <class F>
int for_each_sub(jac_ctx *G, F fn)
{
    const size_t n = G->subs.size();
    std::vector<int> rcs(n, JAC_OK);
    std::vector<std::string> errs(n);
    std::vector<std::thread> th;
    for (size_t i = 0; i < n; ++i)
        th.emplace_back([&, i] {
            cudaSetDevice(G->subs[i]->device);
            rcs[i] = fn(G->subs[i]);
            if (rcs[i]) errs[i] = g_err;
        });
    for (auto &t : th) t.join();
    for (size_t i = 0; i < n; ++i)
        if (rcs[i]) { g_err = errs[i]; return rcs[i]; }
    return JAC_OK;
}

jac_ctx *owner_sub(const jac_ctx *G, int32_t ix, int32_t iy, int32_t iz)
{
    const jac::Plan &p = G->plan;
    if (ix < 0 || iy < 0 || iz < 0 || ix >= p.b[0] || iy >= p.b[1] || iz >= p.b[2]) return nullptr;
    return G->subs[p.owner(ix, iy, iz)];
}

int create_group(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz, int32_t n_gpus,
                 const int32_t *gpu_grid, uint32_t flags, jac_ctx **out)
{
    if (!out) return fail(JAC_EINVAL, "out is NULL");
    *out = nullptr;
    jac::Plan plan;
    std::string err;
    int rc = jac::make_plan(nx, ny, nz, bx, by, bz, n_gpus, gpu_grid, &plan, &err);
    if (rc) return fail(rc, "%s", err.c_str());
    if (flags & (JAC_F_NCCL | JAC_F_PER_BLOCK))
        return fail(JAC_EINVAL, "flags: JAC_F_NCCL / JAC_F_PER_BLOCK are not available in a multi-GPU "
                                "single-process context (use jac_create_rank, one process per GPU)");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev < n_gpus)
        return fail(JAC_EDEVICE, "n_gpus = %d but %d CUDA devices are visible", n_gpus, e == cudaSuccess ? ndev : 0);
    DeviceGuard guard;
    jac_ctx *G = new jac_ctx();
    G->group = true;
    G->plan = plan;
    G->flags = flags;
    auto bail = [&](int code) { std::string m = g_err; jac_destroy(G); g_err = m; return code; };
    for (int32_t g = 0; g < n_gpus; ++g) {
        jac_ctx *sub = nullptr;
        if ((rc = create_common(nx, ny, nz, bx, by, bz, n_gpus, gpu_grid, true, g, g, flags, &sub))) return bail(rc);
        sub->in_group = true;
        G->subs.push_back(sub);
        G->parts.push_back(g);
    }
    // peer access between neighbour devices, then the rank path's connection step with
    // plain pointers
    for (jac_ctx *c : G->subs)
        for (int32_t q : c->part_peers[0]) {
            int ok = 0;
            CK(cudaDeviceCanAccessPeer(&ok, c->device, G->subs[q]->device));
            if (!ok) return bail(fail(JAC_EDEVICE, "device %d cannot access device %d (P2P unavailable)", c->device, q));
            CK(cudaSetDevice(c->device));
            const cudaError_t pe = cudaDeviceEnablePeerAccess(G->subs[q]->device, 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
                return bail(fail(JAC_EDEVICE, "cudaDeviceEnablePeerAccess(%d -> %d): %s", c->device, q,
                                 cudaGetErrorString(pe)));
            cudaGetLastError();  // clear cudaErrorPeerAccessAlreadyEnabled
        }
    std::vector<char *> base(n_gpus);
    std::vector<IpcRecord> recs(n_gpus);
    for (int32_t q = 0; q < n_gpus; ++q) {
        const jac_ctx *c = G->subs[q];
        base[q] = c->alloc;
        memset(&recs[q], 0, sizeof(IpcRecord));
        recs[q].magic = kIpcMagic;
        recs[q].rank = q;
        recs[q].arena_off = c->arena_off;
        recs[q].outbox_off = c->outbox_off;
        recs[q].ctrl_off = c->ctrl_off;
        recs[q].xg_off = c->xg_off;
        recs[q].alloc_bytes = c->alloc_bytes;
    }
    for (jac_ctx *c : G->subs) {
        CK(cudaSetDevice(c->device));
        if ((rc = connect_peers(c, base, recs.data()))) return bail(rc);
    }
    G->ipc_done = true;
    G->nslots = 0;
    for (jac_ctx *c : G->subs) G->nslots += c->nslots;
    *out = G;
    return JAC_OK;
}

int group_step(jac_ctx *G, int32_t n)
{
    int rc;
    if (n < 0) return fail(JAC_EINVAL, "n_iters = %d < 0", n);
    DeviceGuard guard;
    for (jac_ctx *c : G->subs)
        if ((rc = step_check(c, n))) return rc;
    for (jac_ctx *c : G->subs) {  // autotune / graphs first, so the starts below are quick
        CK(cudaSetDevice(c->device));
        if ((rc = step_prepare(c))) return rc;
    }
    // Per device: the aligning barrier, the start event and the first chunk back to back,
    // so each device's first iterations are already queued when its barrier completes
    // (the barrier releases every device once the last one has started its own).
    int32_t left = n;
    const int32_t k0 = n > 0 ? step_chunk(G->subs[0], n) : 0;
    for (jac_ctx *c : G->subs) {
        CK(cudaSetDevice(c->device));
        if ((rc = step_begin(c))) return rc;
        if (k0 && (rc = step_launch(c, k0))) return rc;
    }
    left -= k0;
    while (left > 0) {  // interleaved: every device's chunk queued in turn
        const int32_t k = step_chunk(G->subs[0], left);
        for (jac_ctx *c : G->subs) {
            CK(cudaSetDevice(c->device));
            if ((rc = step_launch(c, k))) return rc;
        }
        left -= k;
    }
    int first = JAC_OK;
    std::string msg;
    double ms = 0.0;
    for (jac_ctx *c : G->subs) {  // every device is synchronised even if one failed
        cudaSetDevice(c->device);
        rc = step_end(c, n);
        if (rc && !first) { first = rc; msg = g_err; }
        ms = std::max(ms, c->last_ms);
    }
    G->last_ms = ms;
    G->iters = G->subs[0]->iters;
    if (first) g_err = msg;
    return first;
}

}  // namespace

extern "C" {

int jac_version(void) { return 100; }

const char *jac_last_error(void) { return g_err.c_str(); }

int jac_plan(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz, int32_t n_gpus,
             const int32_t *gpu_grid_in, int32_t *gpu_grid_out, int64_t *block_extent_out)
{
    jac::Plan p;
    std::string err;
    int rc = jac::make_plan(nx, ny, nz, bx, by, bz, n_gpus, gpu_grid_in, &p, &err);
    if (rc) return fail(rc, "%s", err.c_str());
    for (int d = 0; d < 3; ++d) {
        if (gpu_grid_out) gpu_grid_out[d] = p.g[d];
        if (block_extent_out) block_extent_out[d] = p.e[d];
    }
    return JAC_OK;
}

int jac_plan_face(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz,
                  int32_t n_gpus, const int32_t *gpu_grid_in, int32_t ix, int32_t iy, int32_t iz,
                  int32_t f, int32_t *kind, int32_t *owner)
{
    jac::Plan p;
    std::string err;
    int rc = jac::make_plan(nx, ny, nz, bx, by, bz, n_gpus, gpu_grid_in, &p, &err);
    if (rc) return fail(rc, "%s", err.c_str());
    if (!kind || !owner) return fail(JAC_EINVAL, "kind/owner is NULL");
    if (f < 0 || f > 5) return fail(JAC_EINVAL, "face %d not in 0..5", f);
    if (ix < 0 || iy < 0 || iz < 0 || ix >= p.b[0] || iy >= p.b[1] || iz >= p.b[2])
        return fail(JAC_EINVAL, "block index out of range");
    const int32_t blk[3] = {ix, iy, iz};
    int32_t nb[3];
    if (!p.neighbor(blk, f, nb)) { *kind = JAC_FACE_BOUNDARY; *owner = -1; return JAC_OK; }
    *owner = p.owner(nb[0], nb[1], nb[2]);
    *kind = (*owner == p.owner(ix, iy, iz)) ? JAC_FACE_LOCAL : JAC_FACE_REMOTE;
    return JAC_OK;
}

int jac_create(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz, int32_t n_gpus,
               const int32_t *gpu_grid, uint32_t flags, jac_ctx **out)
{
    NvtxRange range("jac_create");
    try {
        if (n_gpus > 1 && !(flags & JAC_F_VIRTUAL_GPUS))
            return create_group(nx, ny, nz, bx, by, bz, n_gpus, gpu_grid, flags, out);
        return create_common(nx, ny, nz, bx, by, bz, n_gpus, gpu_grid, false, 0, 0, flags, out);
    } catch (...) { return fail(JAC_ENOMEM, "host allocation failed"); }
}

int jac_create_rank(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz,
                    int32_t n_gpus, const int32_t *gpu_grid, int32_t rank, int32_t device,
                    uint32_t flags, jac_ctx **out)
{
    try {
        return create_common(nx, ny, nz, bx, by, bz, n_gpus, gpu_grid, true, rank, device, flags, out);
    } catch (...) { return fail(JAC_ENOMEM, "host allocation failed"); }
}

size_t jac_ipc_handle_bytes(void) { return sizeof(IpcRecord); }

int jac_export_ipc(jac_ctx *c, void *out)
{
    if (!c || !out) return fail(JAC_EINVAL, "ctx/out is NULL");
    if (!c->rank_mode) return fail(JAC_ESTATE, "jac_export_ipc needs a rank context");
    CK(cudaSetDevice(c->device));
    IpcRecord r;
    memset(&r, 0, sizeof r);
    r.magic = kIpcMagic;
    r.rank = c->rank;
    r.fingerprint = fingerprint(c);
    r.arena_off = c->arena_off;
    r.outbox_off = c->outbox_off;
    r.ctrl_off = c->ctrl_off;
    r.xg_off = c->xg_off;
    r.alloc_bytes = c->alloc_bytes;
    CK(cudaIpcGetMemHandle(&r.handle, c->alloc));
    memcpy(out, &r, sizeof r);
    return JAC_OK;
}

int jac_nccl_init(jac_ctx *c, const void *id)
{
    if (!c || !id) return fail(JAC_EINVAL, "ctx/id is NULL");
    if (!(c->flags & JAC_F_NCCL)) return fail(JAC_ESTATE, "jac_nccl_init needs a JAC_F_NCCL rank context");
    if (c->nccl_comm) return fail(JAC_ESTATE, "jac_nccl_init called twice");
    const NcclApi *N = nccl_api();
    if (!N) return fail(JAC_ENCCL, "libnccl.so.2 could not be loaded");
    CK(cudaSetDevice(c->device));
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    ncclComm_t comm = nullptr;
    const ncclResult_t r = N->commInitRank(&comm, c->plan.n_gpus, uid, c->rank);
    if (r != ncclSuccess) return fail(JAC_ENCCL, "ncclCommInitRank: %s", N->errorString(r));
    c->nccl_comm = comm;
    c->ipc_done = true;
    return JAC_OK;
}

size_t jac_nccl_id_bytes(void) { return sizeof(ncclUniqueId); }

int jac_nccl_get_unique_id(void *out)
{
    if (!out) return fail(JAC_EINVAL, "out is NULL");
    const NcclApi *N = nccl_api();
    if (!N) return fail(JAC_ENCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId uid;
    const ncclResult_t r = N->getUniqueId(&uid);
    if (r != ncclSuccess) return fail(JAC_ENCCL, "ncclGetUniqueId: %s", N->errorString(r));
    memcpy(out, &uid, sizeof uid);
    return JAC_OK;
}

int jac_import_ipc(jac_ctx *c, const void *all)
{
    if (!c || !all) return fail(JAC_EINVAL, "ctx/all is NULL");
    if (!c->rank_mode) return fail(JAC_ESTATE, "jac_import_ipc needs a rank context");
    if (c->flags & JAC_F_NCCL) return fail(JAC_ESTATE, "JAC_F_NCCL contexts use jac_nccl_init, not IPC");
    if (c->ipc_done) return fail(JAC_ESTATE, "jac_import_ipc called twice");
    CK(cudaSetDevice(c->device));
    const IpcRecord *recs = static_cast<const IpcRecord *>(all);
    const jac::Plan &p = c->plan;
    const uint64_t fp = fingerprint(c);
    std::vector<char *> base(p.n_gpus, nullptr);
    for (int32_t q : c->part_peers[0]) {
        const IpcRecord &r = recs[q];
        if (r.magic != kIpcMagic || r.rank != q) return fail(JAC_EINVAL, "all: record %d is not a jacobi3d IPC record of rank %d", q, q);
        if (r.fingerprint != fp) return fail(JAC_EINVAL, "all: rank %d was created with a different decomposition/flags", q);
        void *ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, r.handle, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(ptr);
        base[q] = static_cast<char *>(ptr);
    }
    return connect_peers(c, base, recs);
}

int jac_local_box(const jac_ctx *c, int64_t *origin, int64_t *extent)
{
    if (!c || !origin || !extent) return fail(JAC_EINVAL, "ctx/origin/extent is NULL");
    const jac::Plan &p = c->plan;
    int64_t lo[3] = {INT64_MAX, INT64_MAX, INT64_MAX}, hi[3] = {0, 0, 0};
    if (c->group) {  // the union of the devices' boxes
        for (const jac_ctx *sc : c->subs) {
            int64_t o[3], e[3];
            jac_local_box(sc, o, e);
            for (int k = 0; k < 3; ++k) { lo[k] = std::min(lo[k], o[k]); hi[k] = std::max(hi[k], o[k] + e[k]); }
        }
        for (int k = 0; k < 3; ++k) { origin[k] = lo[k]; extent[k] = hi[k] - lo[k]; }
        return JAC_OK;
    }
    for (const jac::DevBlock &d : c->hblocks)
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min<int64_t>(lo[k], d.org[k]);
            hi[k] = std::max<int64_t>(hi[k], d.org[k] + p.e[k] + (k == 2 ? 2 * c->geom.zg : 2));
        }
    for (int k = 0; k < 3; ++k) { origin[k] = lo[k]; extent[k] = hi[k] - lo[k]; }
    return JAC_OK;
}

namespace {
// The host box must cover the context's ghost-inclusive local box (init), or only its
// local interiors (interior = true: read-back).
int check_box(const jac_ctx *c, const void *box, const int64_t *origin, const int64_t *extent, bool interior = false)
{
    if (!box || !origin || !extent) return fail(JAC_EINVAL, "box/origin/extent is NULL");
    int64_t lo[3], ex[3];
    jac_local_box(c, lo, ex);
    const int zg = c->group ? c->subs[0]->geom.zg : c->geom.zg;
    if (interior)
        for (int k = 0; k < 3; ++k) {
            const int gh = k == 2 ? zg : 1;
            lo[k] += gh;
            ex[k] -= 2 * gh;
        }
    for (int k = 0; k < 3; ++k)
        if (origin[k] < 0 || extent[k] < 1 || origin[k] > lo[k] || origin[k] + extent[k] < lo[k] + ex[k] ||
            origin[k] + extent[k] > c->plan.n[k] + (k == 2 ? 2 * zg : 2))
            return fail(JAC_EINVAL, "box origin/extent (dim %d: %lld+%lld) does not cover the local blocks (%lld+%lld)",
                        k, (long long)origin[k], (long long)extent[k], (long long)lo[k], (long long)ex[k]);
    return JAC_OK;
}
// Copies the part of interior sub-box [lo, lo+ext) held by context c into out
// (x fastest, ext[2] x ext[1] x ext[0]); *covered += the cells copied.
int region_copy(jac_ctx *c, const int64_t *lo, const int64_t *ext, double *out, int64_t *covered)
{
    const jac::Plan &p = c->plan;
    CK(cudaSetDevice(c->device));
    const jac::Geom &g = c->geom;
    for (int32_t s = 0; s < c->nslots; ++s) {
        const jac::DevBlock &d = c->hblocks[s];
        int64_t a[3], b[3];
        bool empty = false;
        for (int k = 0; k < 3; ++k) {
            a[k] = std::max<int64_t>(lo[k], d.org[k]);
            b[k] = std::min<int64_t>(lo[k] + ext[k], d.org[k] + p.e[k]);
            empty |= a[k] >= b[k];
        }
        if (empty) continue;
        *covered += (b[0] - a[0]) * (b[1] - a[1]) * (b[2] - a[2]);
        cudaMemcpy3DParms m{};
        m.srcPtr = make_cudaPitchedPtr(c->slot_ptr((int)(c->iters & 1), s), (size_t)g.P * 8, (size_t)g.P, (size_t)(g.ey + 2));
        m.srcPos = make_cudaPos((size_t)(g.A + a[0] - d.org[0]) * 8, (size_t)(1 + a[1] - d.org[1]), (size_t)(g.zg + a[2] - d.org[2]));
        m.dstPtr = make_cudaPitchedPtr(out, (size_t)ext[0] * 8, (size_t)ext[0], (size_t)ext[1]);
        m.dstPos = make_cudaPos((size_t)(a[0] - lo[0]) * 8, (size_t)(a[1] - lo[1]), (size_t)(a[2] - lo[2]));
        m.extent = make_cudaExtent((size_t)(b[0] - a[0]) * 8, (size_t)(b[1] - a[1]), (size_t)(b[2] - a[2]));
        m.kind = cudaMemcpyDeviceToHost;
        CK(cudaMemcpy3DAsync(&m, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return JAC_OK;
}
}  // namespace

int jac_set_init_box(jac_ctx *c, const double *box, const int64_t *origin, const int64_t *extent)
{
    NvtxRange range("jac_set_init_box");
    int rc;
    if ((rc = require_ready(c))) return rc;
    if ((rc = check_box(c, box, origin, extent))) return rc;
    if (c->group) {
        DeviceGuard guard;
        rc = for_each_sub(c, [&](jac_ctx *sc) { return jac_set_init_box(sc, box, origin, extent); });
        c->inited = rc == JAC_OK;
        c->iters = 0;
        return rc;
    }
    CK(cudaSetDevice(c->device));
    if ((rc = enqueue_barrier(c))) return rc;  // neighbours finished writing our ghosts
    if ((rc = staged_transfer(c, true, const_cast<double *>(box), origin, extent))) return rc;
    if (c->geom.A != 0)  // inline ghost columns -> x-ghost arrays (dense rows: written by the scatter)
        CK(jac::launch_xghost_extract(sweep_args(c, 0, 0), c->stream));
    return finish_init(c);
}

int jac_set_init(jac_ctx *c, const double *padded)
{
    if (!c) return fail(JAC_EINVAL, "ctx is NULL");
    if (!padded) return fail(JAC_EINVAL, "padded is NULL");
    const int64_t o[3] = {0, 0, 0};
    const int zg = c->group ? c->subs[0]->geom.zg : c->geom.zg;
    const int64_t e[3] = {c->plan.n[0] + 2, c->plan.n[1] + 2, c->plan.n[2] + 2 * zg};
    return jac_set_init_box(c, padded, o, e);
}

int jac_set_init_hash(jac_ctx *c, uint64_t seed)
{
    NvtxRange range("jac_set_init_hash");
    int rc;
    if ((rc = require_ready(c))) return rc;
    if (c->group) {
        DeviceGuard guard;
        rc = for_each_sub(c, [&](jac_ctx *sc) { return jac_set_init_hash(sc, seed); });
        c->inited = rc == JAC_OK;
        c->iters = 0;
        return rc;
    }
    CK(cudaSetDevice(c->device));
    if ((rc = enqueue_barrier(c))) return rc;
    CK(jac::launch_hash_init(sweep_args(c, 0, 0), c->plan.n[0], c->plan.n[1], seed, c->stream));
    if (c->geom.A != 0)  // dense rows: hash_init_kernel writes the x-ghost arrays itself
        CK(jac::launch_xghost_extract(sweep_args(c, 0, 0), c->stream));
    return finish_init(c);
}

int jac_step(jac_ctx *c, int32_t n)
{
    NvtxRange range("jac_step");
    int rc;
    if (c && c->group) return group_step(c, n);
    if ((rc = step_check(c, n))) return rc;
    CK(cudaSetDevice(c->device));
    if ((rc = step_begin(c))) return rc;
    if (c->flags & JAC_F_PER_BLOCK) {
        if ((rc = per_block_step(c, n))) return rc;
    } else {
        for (int32_t left = n; left > 0;) {
            const int32_t k = step_chunk(c, left);
            if ((rc = step_launch(c, k))) return rc;
            left -= k;
        }
    }
    return step_end(c, n);
}

int jac_profile_sweep(jac_ctx *c, int32_t n, double *avg_ms)
{
    NvtxRange range("jac_profile_sweep");
    int rc;
    if ((rc = require_ready(c))) return rc;
    if (n < 1 || !avg_ms) return fail(JAC_EINVAL, "n_iters must be >= 1 and avg_sweep_ms non-NULL");
    if (!c->inited) return fail(JAC_ESTATE, "jac_profile_sweep before init");
    if (c->group) {  // every device profiles concurrently; the slowest device's figures
        DeviceGuard guard;
        std::vector<double> ms(c->subs.size(), 0.0);
        rc = for_each_sub(c, [&](jac_ctx *sc) { return jac_profile_sweep(sc, n, &ms[sc->rank]); });
        if (rc) return rc;
        *avg_ms = *std::max_element(ms.begin(), ms.end());
        c->last_gap_ms = -1.0;
        c->last_wait_sum_ns = c->last_wait_max_ns = 0;
        for (const jac_ctx *sc : c->subs) {
            c->last_gap_ms = std::max(c->last_gap_ms, sc->last_gap_ms);
            c->last_wait_sum_ns = std::max(c->last_wait_sum_ns, sc->last_wait_sum_ns);
            c->last_wait_max_ns = std::max(c->last_wait_max_ns, sc->last_wait_max_ns);
        }
        c->iters = c->subs[0]->iters;
        return JAC_OK;
    }
    if (c->flags & JAC_F_PER_BLOCK) return fail(JAC_EINVAL, "jac_profile_sweep: not available with JAC_F_PER_BLOCK");
    CK(cudaSetDevice(c->device));
    if ((rc = autotune(c))) return rc;
    struct Events {  // destroyed on every return path
        std::vector<cudaEvent_t> v;
        ~Events() { for (cudaEvent_t e : v) if (e) cudaEventDestroy(e); }
    } evs;
    // TMA sweeps time themselves (first CTA start after the dependency wait, last CTA
    // end, %globaltimer) so the profile graph keeps the programmatic-dependent-launch
    // overlap of jac_step; the plain-load kernel is bracketed by event-record nodes.
    const bool use_span = c->variant != kPlain;
    struct Span {  // freed on every return path
        unsigned long long *d = nullptr;
        jac_ctx *c;
        ~Span() { if (d) cudaFree(d); c->prof_span = nullptr; }
    } span{nullptr, c};
    std::vector<unsigned long long> hspan(4 * (size_t)n, 0ull);  // [start, end, wait sum, wait max]
    for (int it = 0; it < n; ++it) hspan[4 * it] = ~0ull;
    if (use_span) {
        CK(cudaMalloc(&span.d, sizeof(unsigned long long) * hspan.size()));
        CK(cudaMemcpy(span.d, hspan.data(), sizeof(unsigned long long) * hspan.size(), cudaMemcpyHostToDevice));
    } else {
        evs.v.assign(2 * (size_t)n, nullptr);
        for (auto &e : evs.v) CK(cudaEventCreate(&e));
    }
    std::vector<cudaEvent_t> &ev = evs.v;
    int src = (int)(c->iters & 1);
    // The n iterations are captured into one graph, so the sweep is timed exactly as
    // jac_step runs it.
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    rc = JAC_OK;
    c->prof_span = span.d;
    for (int it = 0; it < n && rc == JAC_OK; ++it, src ^= 1) {
        c->prof_it = it;
        rc = use_span ? enqueue_iteration(c, src) : enqueue_iteration(c, src, ev[2 * it], ev[2 * it + 1]);
    }
    c->prof_span = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
    if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (e != cudaSuccess) return fail(JAC_ECUDA, "profile graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(JAC_ECUDA, "profile graph instantiate: %s", cudaGetErrorString(e));
    e = cudaGraphLaunch(exec, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaGraphExecDestroy(exec);
    if (e != cudaSuccess) return fail(JAC_ECUDA, "profile graph: %s", cudaGetErrorString(e));
    std::vector<float> dur(n), gap(n > 1 ? n - 1 : 0);
    if (use_span) {
        CK(cudaMemcpy(hspan.data(), span.d, sizeof(unsigned long long) * hspan.size(), cudaMemcpyDeviceToHost));
        for (int it = 0; it < n; ++it) dur[it] = (float)((double)(hspan[4 * it + 1] - hspan[4 * it]) * 1e-6);
        for (int it = 0; it + 1 < n; ++it)
            gap[it] = (float)(((double)hspan[4 * it + 4] - (double)hspan[4 * it + 1]) * 1e-6);
        // peer waits of the remote CTAs: median over sweeps of the summed wait, max of any
        std::vector<unsigned long long> ws(n);
        c->last_wait_max_ns = 0;
        for (int it = 0; it < n; ++it) {
            ws[it] = hspan[4 * it + 2];
            c->last_wait_max_ns = std::max<int64_t>(c->last_wait_max_ns, (int64_t)hspan[4 * it + 3]);
        }
        std::sort(ws.begin(), ws.end());
        c->last_wait_sum_ns = (int64_t)ws[n / 2];
    } else {
        for (int it = 0; it < n; ++it) CK(cudaEventElapsedTime(&dur[it], ev[2 * it], ev[2 * it + 1]));
        for (int it = 0; it + 1 < n; ++it) CK(cudaEventElapsedTime(&gap[it], ev[2 * it + 1], ev[2 * it + 2]));
    }
    // end of sweep i -> start of sweep i+1: the graph's launch / dependency gap
    // (plus whatever the iteration enqueues after the sweep: nothing in the fused
    // mode; the ghost-fill kernel / NCCL calls in the ablation modes)
    if (!gap.empty()) {
        std::sort(gap.begin(), gap.end());
        const size_t m = gap.size();
        c->last_gap_ms = (m & 1) ? gap[m / 2] : 0.5 * ((double)gap[m / 2 - 1] + gap[m / 2]);
    } else {
        c->last_gap_ms = -1.0;
    }
    c->iters += n;
    c->kernel_launches += (int64_t)n * c->kernels_per_iter();
    if ((rc = check_status(c))) return rc;
    // median: robust to the first launches of a multi-rank run, whose remote items may
    // wait for a neighbour rank that started its profiling graph a little later
    std::sort(dur.begin(), dur.end());
    *avg_ms = (n & 1) ? dur[n / 2] : 0.5 * ((double)dur[n / 2 - 1] + dur[n / 2]);
    return JAC_OK;
}

int jac_last_profile_gap_ms(const jac_ctx *c, double *ms)
{
    if (!c || !ms) return fail(JAC_EINVAL, "ctx/ms is NULL");
    if (c->last_gap_ms < 0) return fail(JAC_ESTATE, "no jac_profile_sweep with n_iters >= 2 yet");
    *ms = c->last_gap_ms;
    return JAC_OK;
}

int jac_get_block_padded(jac_ctx *c, int32_t ix, int32_t iy, int32_t iz, double *out)
{
    if (!c || !out) return fail(JAC_EINVAL, "ctx/out is NULL");
    if (c->group) {
        jac_ctx *sc = owner_sub(c, ix, iy, iz);
        if (!sc) return fail(JAC_EINVAL, "block index (%d,%d,%d) out of range", ix, iy, iz);
        DeviceGuard guard;
        return jac_get_block_padded(sc, ix, iy, iz, out);
    }
    int32_t s;
    int rc;
    if ((rc = local_slot_of(c, ix, iy, iz, &s))) return rc;
    CK(cudaSetDevice(c->device));
    const jac::Geom &g = c->geom;
    cudaMemcpy3DParms m{};
    const bool dense = (g.A == 0);  // dense rows store no x-edge corner cells: they read as NaN
    if (dense)
        std::fill(out, out + (size_t)(g.ex + 2) * (g.ey + 2) * (g.ez + 2 * g.zg), std::nan(""));
    m.srcPtr = make_cudaPitchedPtr(c->slot_ptr((int)(c->iters & 1), s), (size_t)g.P * 8, (size_t)g.P, (size_t)(g.ey + 2));
    m.srcPos = make_cudaPos(dense ? 0 : (size_t)(g.A - 1) * 8, 0, 0);
    m.dstPtr = make_cudaPitchedPtr(out, (size_t)(g.ex + 2) * 8, (size_t)(g.ex + 2), (size_t)(g.ey + 2));
    m.dstPos = make_cudaPos(dense ? 8 : 0, 0, 0);
    m.extent = make_cudaExtent((size_t)(g.ex + (dense ? 0 : 2)) * 8, (size_t)(g.ey + 2), (size_t)(g.ez + 2 * g.zg));
    m.kind = cudaMemcpyDeviceToHost;
    CK(cudaMemcpy3DAsync(&m, c->stream));
    // the x ghosts live in the x-ghost arrays: patch columns 0 and ex+1 (interior j, k)
    std::vector<double> xgh((size_t)2 * g.ez * g.eyp);
    const int cur = (int)(c->iters & 1);
    for (int side = 0; side < 2; ++side)
        CK(cudaMemcpyAsync(xgh.data() + (size_t)side * g.ez * g.eyp, jac::xg_array(c->xg, g, cur, s, side),
                           (size_t)g.ez * g.eyp * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const int64_t sx = g.ex + 2, sxy = sx * (g.ey + 2);
    for (int64_t k = 0; k < g.ez; ++k)
        for (int64_t j = 0; j < g.ey; ++j) {
            out[(k + g.zg) * sxy + (j + 1) * sx] = xgh[k * g.eyp + j];
            out[(k + g.zg) * sxy + (j + 1) * sx + g.ex + 1] = xgh[(size_t)g.ez * g.eyp + k * g.eyp + j];
        }
    return JAC_OK;
}

int jac_get_block(jac_ctx *c, int32_t ix, int32_t iy, int32_t iz, double *out)
{
    if (!c || !out) return fail(JAC_EINVAL, "ctx/out is NULL");
    if (c->group) {
        jac_ctx *sc = owner_sub(c, ix, iy, iz);
        if (!sc) return fail(JAC_EINVAL, "block index (%d,%d,%d) out of range", ix, iy, iz);
        DeviceGuard guard;
        return jac_get_block(sc, ix, iy, iz, out);
    }
    int32_t s;
    int rc;
    if ((rc = local_slot_of(c, ix, iy, iz, &s))) return rc;
    CK(cudaSetDevice(c->device));
    const jac::Geom &g = c->geom;
    cudaMemcpy3DParms m{};
    m.srcPtr = make_cudaPitchedPtr(c->slot_ptr((int)(c->iters & 1), s), (size_t)g.P * 8, (size_t)g.P, (size_t)(g.ey + 2));
    m.srcPos = make_cudaPos((size_t)g.A * 8, 1, (size_t)g.zg);
    m.dstPtr = make_cudaPitchedPtr(out, (size_t)g.ex * 8, (size_t)g.ex, (size_t)g.ey);
    m.extent = make_cudaExtent((size_t)g.ex * 8, (size_t)g.ey, (size_t)g.ez);
    m.kind = cudaMemcpyDeviceToHost;
    CK(cudaMemcpy3DAsync(&m, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return JAC_OK;
}

int jac_get_field_box(jac_ctx *c, double *box, const int64_t *origin, const int64_t *extent)
{
    NvtxRange range("jac_get_field_box");
    if (!c) return fail(JAC_EINVAL, "ctx is NULL");
    int rc;
    if ((rc = check_box(c, box, origin, extent, true))) return rc;
    if (c->group) {  // the devices' regions are disjoint: read them back concurrently
        DeviceGuard guard;
        return for_each_sub(c, [&](jac_ctx *sc) { return jac_get_field_box(sc, box, origin, extent); });
    }
    CK(cudaSetDevice(c->device));
    return staged_transfer(c, false, box, origin, extent);
}

int jac_get_field(jac_ctx *c, double *padded)
{
    if (!c) return fail(JAC_EINVAL, "ctx is NULL");
    if (!padded) return fail(JAC_EINVAL, "padded is NULL");
    const int64_t o[3] = {0, 0, 0};
    const int zg = c->group ? c->subs[0]->geom.zg : c->geom.zg;
    const int64_t e[3] = {c->plan.n[0] + 2, c->plan.n[1] + 2, c->plan.n[2] + 2 * zg};
    return jac_get_field_box(c, padded, o, e);
}

int jac_get_region(jac_ctx *c, const int64_t *lo, const int64_t *ext, double *out)
{
    if (!c || !lo || !ext || !out) return fail(JAC_EINVAL, "ctx/lo/ext/out is NULL");
    const jac::Plan &p = c->plan;
    for (int k = 0; k < 3; ++k)
        if (lo[k] < 0 || ext[k] < 1 || lo[k] + ext[k] > p.n[k])
            return fail(JAC_EINVAL, "region dim %d [%lld, +%lld) outside the interior", k, (long long)lo[k], (long long)ext[k]);
    DeviceGuard guard;
    int64_t covered = 0;
    int rc;
    if (c->group) {
        for (jac_ctx *sc : c->subs)
            if ((rc = region_copy(sc, lo, ext, out, &covered))) return rc;
    } else if ((rc = region_copy(c, lo, ext, out, &covered))) {
        return rc;
    }
    if (covered != ext[0] * ext[1] * ext[2]) return fail(JAC_EINVAL, "region is not entirely local to this context");
    return JAC_OK;
}

int jac_get_layout(const jac_ctx *c, int32_t *gpu_grid, int64_t *block_extent, int64_t *iterations_done)
{
    if (!c) return fail(JAC_EINVAL, "ctx is NULL");
    for (int d = 0; d < 3; ++d) {
        if (gpu_grid) gpu_grid[d] = c->plan.g[d];
        if (block_extent) block_extent[d] = c->plan.e[d];
    }
    if (iterations_done) *iterations_done = c->iters;
    return JAC_OK;
}

int jac_get_grid(const jac_ctx *c, int64_t *n, int32_t *blocks, uint32_t *flags)
{
    if (!c) return fail(JAC_EINVAL, "ctx is NULL");
    for (int d = 0; d < 3; ++d) {
        if (n) n[d] = c->plan.n[d];
        if (blocks) blocks[d] = c->plan.b[d];
    }
    if (flags) *flags = c->flags;
    return JAC_OK;
}

int jac_block_owner(const jac_ctx *c, int32_t ix, int32_t iy, int32_t iz, int32_t *gpu)
{
    if (!c || !gpu) return fail(JAC_EINVAL, "ctx/gpu is NULL");
    const jac::Plan &p = c->plan;
    if (ix < 0 || iy < 0 || iz < 0 || ix >= p.b[0] || iy >= p.b[1] || iz >= p.b[2])
        return fail(JAC_EINVAL, "block index out of range");
    *gpu = p.owner(ix, iy, iz);
    return JAC_OK;
}

int jac_last_step_ms(const jac_ctx *c, double *ms)
{
    if (!c || !ms) return fail(JAC_EINVAL, "ctx/ms is NULL");
    *ms = c->last_ms;
    return JAC_OK;
}

int jac_get_stats(const jac_ctx *c, int64_t *st)
{
    if (!c || !st) return fail(JAC_EINVAL, "ctx/stats is NULL");
    if (c->group) {  // totals over the devices; kernels per iteration and variant of device 0
        int64_t sub[JAC_STAT_N];
        for (int k = 0; k < JAC_STAT_N; ++k) st[k] = 0;
        for (const jac_ctx *sc : c->subs) {
            jac_get_stats(sc, sub);
            for (int k = 0; k < JAC_STAT_N; ++k) st[k] += sub[k];
        }
        st[JAC_STAT_EPOCH_MIN] = INT64_MAX;
        st[JAC_STAT_EPOCH_MAX] = 0;
        for (const jac_ctx *sc : c->subs) {
            jac_get_stats(sc, sub);
            st[JAC_STAT_EPOCH_MIN] = std::min(st[JAC_STAT_EPOCH_MIN], sub[JAC_STAT_EPOCH_MIN]);
            st[JAC_STAT_EPOCH_MAX] = std::max(st[JAC_STAT_EPOCH_MAX], sub[JAC_STAT_EPOCH_MAX]);
        }
        jac_get_stats(c->subs[0], sub);
        st[JAC_STAT_KERNELS_PER_ITER] = sub[JAC_STAT_KERNELS_PER_ITER];
        st[JAC_STAT_SWEEP_VARIANT] = sub[JAC_STAT_SWEEP_VARIANT];
        st[JAC_STAT_FUSED_SYNC] = sub[JAC_STAT_FUSED_SYNC];
        st[JAC_STAT_PEER_WAIT_NS] = c->last_wait_sum_ns;
        st[JAC_STAT_PEER_WAIT_MAX_NS] = c->last_wait_max_ns;
        return JAC_OK;
    }
    st[JAC_STAT_KERNEL_LAUNCHES] = c->kernel_launches;
    st[JAC_STAT_GRAPH_LAUNCHES] = c->graph_launches;
    st[JAC_STAT_KERNELS_PER_ITER] = c->kernels_per_iter();
    st[JAC_STAT_LOCAL_BLOCKS] = c->nslots;
    st[JAC_STAT_LOCAL_FACES] = c->local_faces;
    st[JAC_STAT_REMOTE_FACES] = c->remote_faces;
    st[JAC_STAT_REMOTE_BYTES] = c->remote_bytes;
    st[JAC_STAT_ARENA_BYTES] = (int64_t)(2 * (size_t)c->nslots * c->geom.bstride * 8);
    st[JAC_STAT_SWEEP_VARIANT] = c->variant;
    st[JAC_STAT_PARTITIONS] = (int64_t)c->parts.size();
    st[JAC_STAT_REMOTE_ITEMS] = c->nremote;
    st[JAC_STAT_FUSED_SYNC] = c->fused ? 1 : 0;
    // epochs of the hosted partitions' control words (device read; 0 without peers)
    st[JAC_STAT_EPOCH_MIN] = 0;
    st[JAC_STAT_EPOCH_MAX] = 0;
    if (c->ctrl && !c->hsync.empty()) {
        int64_t lo = INT64_MAX, hi = 0;
        cudaSetDevice(c->device);
        for (const jac::PartSync &ps : c->hsync) {
            uint64_t e = 0;
            if (cudaMemcpy(&e, ps.ctrl, sizeof e, cudaMemcpyDeviceToHost) != cudaSuccess)
                return fail(JAC_ECUDA, "jac_get_stats: control word read");
            lo = std::min<int64_t>(lo, (int64_t)e);
            hi = std::max<int64_t>(hi, (int64_t)e);
        }
        st[JAC_STAT_EPOCH_MIN] = lo;
        st[JAC_STAT_EPOCH_MAX] = hi;
    }
    st[JAC_STAT_EXPERIMENT] = experiment_mask(c);
    st[JAC_STAT_PEER_WAIT_NS] = c->last_wait_sum_ns;
    st[JAC_STAT_PEER_WAIT_MAX_NS] = c->last_wait_max_ns;
    return JAC_OK;
}

int jac_set_option(jac_ctx *c, int32_t option, int64_t value)
{
    if (!c) return fail(JAC_EINVAL, "ctx is NULL");
    if (c->group) {
        for (jac_ctx *sc : c->subs) {
            const int rc = jac_set_option(sc, option, value);
            if (rc) return rc;
        }
        return JAC_OK;
    }
    switch (option) {
    case JAC_OPT_LAUNCH_THREADS:
        if (value < 1 || value > 64) return fail(JAC_EINVAL, "JAC_OPT_LAUNCH_THREADS value %lld not in 1..64", (long long)value);
        c->launch_threads = (int)value;
        return JAC_OK;
    case JAC_OPT_WATCHDOG_MS:
        if (value < 0) return fail(JAC_EINVAL, "JAC_OPT_WATCHDOG_MS value %lld < 0", (long long)value);
        c->watchdog_ns = (uint64_t)value * 1000000ull;  // captured graphs read it at launch: rebuild them
        for (int s = 0; s < 2; ++s) {
            if (c->g1[s]) { cudaGraphExecDestroy(c->g1[s]); c->g1[s] = nullptr; }
            if (c->gU[s]) { cudaGraphExecDestroy(c->gU[s]); c->gU[s] = nullptr; }
        }
        return JAC_OK;
    default:
        return fail(JAC_EINVAL, "unknown option %d", option);
    }
}

int jac_destroy(jac_ctx *c)
{
    if (!c) return JAC_OK;
    if (c->group) {  // no device may still store into a neighbour that is being freed
        DeviceGuard guard;
        for (jac_ctx *sc : c->subs) { cudaSetDevice(sc->device); cudaStreamSynchronize(sc->stream); }
        for (jac_ctx *sc : c->subs) jac_destroy(sc);
        delete c;
        return JAC_OK;
    }
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (cudaStream_t s : c->bstreams) if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    for (cudaEvent_t e : c->bevents) if (e) cudaEventDestroy(e);
    for (int s = 0; s < 2; ++s) {
        if (c->g1[s]) cudaGraphExecDestroy(c->g1[s]);
        if (c->gU[s]) cudaGraphExecDestroy(c->gU[s]);
    }
    for (void *p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    if (c->nccl_comm) {
        if (const NcclApi *N = nccl_api()) N->commDestroy((ncclComm_t)c->nccl_comm);
    }
    if (c->cstream) { cudaStreamSynchronize(c->cstream); cudaStreamDestroy(c->cstream); }
    for (cudaEvent_t e : c->sev) if (e) cudaEventDestroy(e);
    if (c->stage[0]) cudaFree(c->stage[0]);
    if (c->dlist) cudaFree(c->dlist);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->dblocks) cudaFree(c->dblocks);
    if (c->ditem_map) cudaFree(c->ditem_map);
    if (c->dsync) cudaFree(c->dsync);
    if (c->dranges) cudaFree(c->dranges);
    if (c->dvcopies) cudaFree(c->dvcopies);
    if (c->status_h) cudaFreeHost(c->status_h);
    if (c->alloc) cudaFree(c->alloc);
    delete c;
    return JAC_OK;
}

}  // extern "C"
