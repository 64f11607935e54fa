// device.hpp -- data shared by the host engine and the sm_100a kernels:
// the device-resident block-descriptor table (north-star subsystem 1) and the
// launch arguments.  No method arithmetic lives here.
//
// HBM layout.  Every block ("chare") owns two ghosted arrays (ping,
// pong) of (ez+2) planes x (ey+2) rows x P doubles.  Element (i,j,k) of a block,
// i in [-1,ex], j in [-1,ey], k in [-1,ez] (-1 and e* are ghosts), lives at
//     base + (k+zg)*Q + (j+1)*P + A + i,     Q = P*(ey+2)
// (zg = 1; the 2-D mode, JAC_F_2D, has a single plane k = 0 and zg = 0)
// with A = 4 so the interior row starts on a 32-byte sector (and 16-byte aligned
// double2 accesses); narrow blocks (ex <= 64) use A = 8 and a 64-byte row pitch so
// rows start on 64-byte DRAM granules (engine.cu, geometry).  All slots of one GPU sit in one arena: slot s of buffer b
// starts at arena + (b*nslots + s)*bstride, which lets ONE 4-D TMA tensor map
// {P, ey+2, ez+2, 2*nslots} cover every block of the GPU.
//
// x-face ghosts do NOT live in the rows (one strided double per row would cost a
// whole 32-byte sector per row on both the write and the read side).  Each block
// owns, per buffer, two contiguous x-ghost arrays XG[side] of ez x eyp doubles,
// element (j, k) at xg + k*eyp + j: side 0 = the ghost column i = -1, side 1 =
// i = ex.  Senders store them as 128-byte runs (16 rows of a tile), receivers stage
// them with one bulk copy per plane.  XG(buf, slot, side) =
//     xg + ((buf*nslots + slot)*2 + side)*xgstride.
// The y- and z-face ghosts stay in place (whole rows / planes, coalesced).
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define JAC_HD __host__ __device__
#else
#define JAC_HD
#endif

namespace jac {

enum Face { XM = 0, XP = 1, YM = 2, YP = 3, ZM = 4, ZP = 5 };
JAC_HD inline constexpr int opposite(int f) { return f ^ 1; }

constexpr int kA = 4;        // x offset of interior column 0 inside a row
constexpr int kXgPad = 32;   // doubles of slack after each x-ghost array (bulk-copy overrun)

struct DevBlock {
    int32_t slot;            // own slot in this GPU's arena
    int32_t org[3];          // global interior origin of the block (x, y, z)
    uint32_t remote_mask;    // bit f: face f's neighbour lives in another partition (another
                             // GPU, or another virtual partition under JAC_F_VIRTUAL_GPUS)
    uint32_t pack_mask;      // bit f: nb[f][*] is a packed send buffer (JAC_F_NCCL), layout
                             // x: [k][eyp] (x-ghost layout), y: [k][ex], z: [j][ex]
    int32_t part;            // index of the owning partition in the context's PartSync table
    int32_t pad_;
    double *nb[6][2];        // per face and buffer, where this block's boundary layer
                             // goes: y/z faces -> the neighbour block's array base;
                             // x faces -> the neighbour's x-ghost array (side
                             // opposite to f).  Local or peer-mapped (IPC); nullptr =
                             // global boundary face.
    const double *nb_out[6]; // neighbour's outbox region for the face opposite to f
                             // (JAC_F_UNFUSED_PACK only)
};

struct Geom {
    int32_t ex, ey, ez;      // block interior extents
    int32_t A;               // kA, or 2*kA for narrow blocks
    int64_t P, Q;            // row / plane pitch in doubles
    int64_t bstride;         // doubles between consecutive slots (256-byte multiple)
    int32_t nslots;          // slots per buffer in the arena
    int32_t eyp;             // x-ghost array row pitch (ey rounded up to 4)
    int32_t zg;              // z ghost planes per side: 1 (3-D), 0 (2-D: one plane, k = 0)
    int32_t pad_;
    int64_t xgstride;        // doubles per x-ghost array (incl. kXgPad, 256-byte multiple)
    int64_t ostride;         // outbox doubles per slot
    int64_t ooff[6];         // outbox face offsets inside a slot
};

enum SweepMode { MODE_FUSED = 0, MODE_PACK = 1, MODE_NOEXCHANGE = 2 };
// JAC_NO_CTA_SYSFENCE experiment: remote CTAs skip their system fence before the count
// (UNSAFE: peer data may trail the flag) -- measures that fence's cost, nothing else
constexpr int32_t kExpNoCtaSysFence = 1;

// Cross-partition ordering state of one partition hosted by a context (one per rank
// context; one per virtual partition under JAC_F_VIRTUAL_GPUS).  Its control words
// live in the hosting context's ctrl area: [0] = epoch (phases completed here),
// [1 + q] = the flag word partition q stores its epoch into (st.release.sys, over
// NVLink for a peer GPU), [1 + n_gpus] = count of this sweep's finished remote CTAs.
// Checked build (-DJAC_CHECKED, libjacobi3d_checked.so): every global store of the
// kernels is tested against these ranges (the context's allocation and its peers') and
// its alignment, every TMA coordinate against the tensor extent; a violation is
// recorded in the mapped status words and the store is skipped -- the substitute for
// compute-sanitizer, which is closed on this pool.  Unused in the production build.
struct MemRange {
    unsigned long long lo, hi;  // [lo, hi) byte addresses
};
constexpr uint32_t kStatusMisaligned = 2u;  // status[0] bits (with kStatusPeerTimeout)
constexpr uint32_t kStatusOutOfRange = 4u;
constexpr uint32_t kStatusAssert = 8u;
struct CheckArgs {
    const MemRange *ranges;  // device table
    int32_t nranges;
    int32_t pad_;
    uint32_t *status;        // mapped host words: [0] flags, [1] first failing source line,
                             // [2..3] its address (low, high)
};

struct PartSync {
    uint64_t *ctrl;
    unsigned long long *count;
    uint64_t *peer_slot[6];  // per neighbour partition: &its_ctrl[1 + this partition]
    int32_t peer_id[6];      // neighbour partition ids
    int32_t npeers;
    int32_t nremote;         // items of one sweep touching a remote face of this partition
};

// Watchdog of the cross-partition waits (wait_peers, barrier_kernel): a wait longer
// than spin_limit_ns (0 = forever) gives up, ORs kStatusPeerTimeout into *status (a
// mapped host word the engine checks after every call) and continues -- the results of
// that sweep are then wrong and the call returns JAC_ECUDA; the CUDA context survives.
constexpr uint32_t kStatusPeerTimeout = 1u;
struct Watchdog {
    uint32_t *status;        // mapped pinned host word, or nullptr
    uint64_t spin_limit_ns;
};

struct SweepArgs {
    Geom g;
    const DevBlock *blocks;  // [nslots]
    double *arena;
    double *xg;              // x-ghost arrays
    double *outbox;
    int32_t src;             // buffer read (0/1); the sweep writes 1-src
    int32_t mode;            // SweepMode
    int32_t ntx, nty, ntz;   // tiles per block in x, y, z (ntz: plain kernel only)
    int32_t zc;              // planes per z-chunk (plain kernel only)
    // TMA kernel work list.  column = (b*nty + ty)*ntx + tx; columns are cut into
    // groups of gcols (about the number of resident CTAs), and items run group by
    // group, z-chunk-major inside a group: item = g*gcols*nzc + zi*gsize + (col - g*gcols).
    // z-chunk zi of a column covers planes [zi*ez/nzc, (zi+1)*ez/nzc).  2-D: gcols =
    // x tiles per band (decode_item2d).
    int32_t nzc, ncols, nitems, gcols;
    // Fused cross-partition ordering (contexts with remote faces, fused mode).  Only
    // the items that touch a remote face share memory with a neighbour partition: they
    // launch first (item_map), wait for the neighbours' signal of the previous sweep,
    // and the last of them per partition (PartSync::nremote) signals this sweep's.
    // Other items never wait.
    const int32_t *item_map; // launch order -> item (~item for a remote-touching item), or nullptr
    const PartSync *sync;    // [partitions hosted], indexed by DevBlock::part
    Watchdog wd;
    int32_t fused_sync;
    int32_t nremote;         // remote-touching items of all hosted partitions (the first
                             // nremote entries of item_map)
    int32_t slot_base;       // slot of blocks[0] (JAC_F_PER_BLOCK launches one block's table
                             // entry; 0 otherwise: the work list enumerates slots in order)
    int32_t exp_bits;        // timing experiments only (kExpNoCtaSysFence); 0 in production
    CheckArgs chk;           // checked build only
    // jac_profile_sweep: when set, every CTA atomicMin's %globaltimer into span[0] after
    // the dependency wait and atomicMax's it into span[1] when done (ns); remote CTAs add
    // their peer-wait time to span[2] and max it into span[3]
    unsigned long long *span;
};

// One contiguous face copy of the virtual transport (JAC_F_VIRTUAL_GPUS | JAC_F_NCCL):
// a packed send buffer of one partition into the matching receive buffer of another,
// standing in for one ncclSend / ncclRecv pair.
struct FaceCopy {
    const double *src;
    double *dst;
    int64_t count;           // doubles
};

struct TileItem {
    int b, x0, y0, zs, ze;   // 2-D: zs, ze = the item's y-tile range [zs, ze)
};

// item -> (block, tile, z-chunk) for the 3-D sweep (see SweepArgs work list)
JAC_HD inline TileItem decode_item3d(const SweepArgs &a, int item, int BX, int BY)
{
    TileItem t;
    const int grp = item / (a.gcols * a.nzc);
    const int r = item - grp * a.gcols * a.nzc;
    const int rest = a.ncols - grp * a.gcols;
    const int gsize = a.gcols < rest ? a.gcols : rest;
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

// item -> (block, x tile, chunk of y tiles) for the 2-D sweep; nzc = y chunks per block.
// The x tiles of a block are cut into bands of gcols tiles; items run band by band,
// x tile fastest inside a band (y-chunk-major).  Production uses one band (the whole
// width): bands of 256-1024 tiles and narrow column groups of 296 tiles, chunk-major, were
// measured equal or slower (profiles/r02_j2d_xband.txt, r02_j2d_column_groups.txt).
JAC_HD inline TileItem decode_item2d(const SweepArgs &a, int item, int BX, int BY)
{
    TileItem t;
    const int per_b = a.ntx * a.nzc;
    t.b = item / per_b;
    const int w = item - t.b * per_b;
    const int band = w / (a.gcols * a.nzc);
    const int r = w - band * a.gcols * a.nzc;
    const int rest = a.ntx - band * a.gcols;
    const int bw = a.gcols < rest ? a.gcols : rest;
    const int yc = r / bw;
    const int tx = band * a.gcols + (r - yc * bw);
    const int tpc = (a.nty + a.nzc - 1) / a.nzc;
    t.x0 = tx * BX;
    t.zs = yc * tpc;
    t.ze = (t.zs + tpc < a.nty) ? t.zs + tpc : a.nty;
    t.y0 = t.zs * BY;
    return t;
}

// Does the item read or write the ghost layer of a face in `mask`?
JAC_HD inline bool item_touches(const SweepArgs &a, const TileItem &t, uint32_t mask, int BX, int BY, bool two_d)
{
    if (!mask) return false;
    const Geom &g = a.g;
    bool hit = false;
    if (mask & (1u << XM)) hit |= t.x0 == 0;
    if (mask & (1u << XP)) hit |= t.x0 + BX >= g.ex;
    if (two_d) {
        if (mask & (1u << YM)) hit |= t.zs == 0;
        if (mask & (1u << YP)) hit |= t.ze * BY >= g.ey;
    } else {
        if (mask & (1u << YM)) hit |= t.y0 == 0;
        if (mask & (1u << YP)) hit |= t.y0 + BY >= g.ey;
        if (mask & (1u << ZM)) hit |= t.zs == 0;
        if (mask & (1u << ZP)) hit |= t.ze >= g.ez;
    }
    return hit;
}

JAC_HD inline double *xg_array(double *xg, const Geom &g, int buf, int slot, int side)
{
    return xg + ((int64_t)(buf * g.nslots + slot) * 2 + side) * g.xgstride;
}

// Neighbour barrier between partitions: every hosted partition bumps its epoch and
// stores it into each neighbour's flag word, then waits until every neighbour's flag
// in its own control block has reached it (monotonically increasing epochs).
struct BarrierArgs {
    const PartSync *sync;    // device table [nparts]
    int32_t nparts;
    int32_t pad_;
    Watchdog wd;
};

}  // namespace jac
