/*
 * jacobi3d.h -- C ABI of the B200-native overdecomposed Jacobi3D library
 * (libjacobi3d.so, built from paper_2605_12734_b200/csrc/).
 *
 * The operation (§5 "jacobi2d": "applies the Jacobi iterative method
 * on a 2D grid. The grid is divided among charm++ chares/MPI ranks, which
 * communicate by halo exchanges. The application is run for 100 iterations without
 * convergence checks"), lifted to 3D: a global fp64 grid of
 * nx*ny*nz updated points plus a fixed 1-cell Dirichlet shell (R6, R7) is swept
 *     u'(p) = ((((((u(p) + u(x-)) + u(x+)) + u(y-)) + u(y+)) + u(z-)) + u(z+)) * fl(1/7)
 * (R2-R4).  The grid is overdecomposed into bx*by*bz blocks ("chares"), ODF =
 * blocks / GPUs (§3.1 "putting 8-16 chares per GPU device"),
 * each block with its own ghosted storage; every iteration exchanges faces between
 * blocks on the same GPU and on other GPUs (§4) and sweeps
 * every block.  Results are bit-identical to the undecomposed iteration for every
 * ODF and GPU count.
 *
 * Conventions for every function:
 *   - returns JAC_OK (0) or a negative jac_status; on error jac_last_error()
 *     returns a thread-local message naming the offending argument.
 *   - host pointers are borrowed for the duration of the call only; the context
 *     owns every device allocation, stream, event and CUDA graph it creates.
 *   - one context is driven by one host thread at a time (no internal locking).
 *   - padded host arrays are (nz+2)*(ny+2)*(nx+2) doubles, x fastest:
 *     p(i,j,k) = (k*(ny+2) + j)*(nx+2) + i, 0 <= i <= nx+1 etc.; interior is
 *     1..nx, 1..ny, 1..nz.
 *   - block (ix,iy,iz) covers interior points [ix*ex,(ix+1)*ex) x [iy*ey,..) x
 *     [iz*ez,..) (0-based), ex = nx/bx etc.; GPU partitions are contiguous
 *     sub-boxes of the block grid (SPEC.md:259-265 contiguous block_map),
 *     partition id g = (pz*gy + py)*gx + px.
 */
#ifndef JACOBI3D_H
#define JACOBI3D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the library is built with -fvisibility=hidden */
#endif

typedef struct jac_ctx jac_ctx; /* opaque */

enum jac_status {
    JAC_OK = 0,
    JAC_EINVAL = -1,  /* null pointer, extent < 1, n_gpus < 1, n_iters < 0, bad index */
    JAC_EDECOMP = -2, /* nx % bx, bx % gx (likewise y, z), gx*gy*gz != n_gpus, or
                         (bx*by*bz) % n_gpus != 0 (non-integral ODF): SPEC.md:254-258,
                         "tiling mismatch -> configuration error" SPEC.md:475 */
    JAC_EDEVICE = -3, /* no CUDA device, device not sm_100, too few devices */
    JAC_ENOMEM = -4,  /* device or pinned-host allocation failed */
    JAC_ECUDA = -5,   /* any other CUDA runtime / driver error (message has the name) */
    JAC_ENCCL = -6,   /* reserved for the NCCL transport (JAC_F_NCCL) */
    JAC_ESTATE = -7   /* call out of order: jac_step before init, import twice, ... */
};

enum jac_flags {
    JAC_F_DEFAULT = 0,
    JAC_F_FMA = 1u << 0,          /* accepted, no effect: the update has no a*b+c (R5) */
    JAC_F_NO_GRAPH = 1u << 1,     /* launch every kernel from the host each iteration
                                     (ablation of the CUDA-Graph iteration) */
    JAC_F_NCCL = 1u << 2,         /* rank contexts, ablation of the peer-store exchange: the
                                     sweep packs REMOTE faces into send buffers, grouped
                                     ncclSend / ncclRecv move them (one per face), the
                                     batched ghost kernel unpacks (north-star subsystem 4,
                                     "NCCL send/recv").  Bootstrap with jac_nccl_* below.
                                     With JAC_F_VIRTUAL_GPUS: the same packed layout, moved
                                     by an on-device copy kernel standing in for NCCL. */
    JAC_F_UNFUSED_PACK = 1u << 4, /* north-star layout: the sweep packs faces into an
                                     outbox and a separate batched ghost-copy kernel
                                     fills the ghosts (PAPER.md:90 pack/unpack kernels) */
    JAC_F_NO_TMA = 1u << 5,       /* plain per-point global-load sweep (no TMA staging) */
    JAC_F_VIRTUAL_GPUS = 1u << 6, /* test-only: all n_gpus partitions live on device 0 in one
                                     context and are swept by ONE kernel per iteration, but
                                     faces between partitions take the REMOTE path of a
                                     multi-GPU run: per-partition remote masks, the
                                     remote-first item order, per-partition epoch / flag /
                                     count words with the in-sweep wait and signal, the
                                     barrier kernel, and (with JAC_F_NCCL) packed send /
                                     receive buffers.  Inside one kernel the previous sweep
                                     has completed, so the waits are satisfied on entry (they
                                     check the epoch bookkeeping, not timing): kernels that
                                     wait on one another never share a GPU. */
    JAC_F_SKIP_EXCHANGE = 1u << 7, /* timing-only ablation: no face writes. WRONG results */
    JAC_F_PER_BLOCK = 1u << 8,     /* paper-style execution: one stream per
                                      block ("non-blocking per-chare streams")
                                      and, per iteration and block, one unpack launch per
                                      face, one stencil launch, one pack launch per face
                                      (SPEC.md:474), ordered by per-block events; no graph.
                                      Launching host threads (the paper's PEs per process,
                                      PAPER.md:95) via jac_set_option.  One GPU, one
                                      partition (n_gpus == 1); 3-D or 2-D. */
    JAC_F_2D = 1u << 9             /* Jacobi2D (the paper's evaluated app,
                                      PAPER.md:280-294): nz == 1, bz == 1; 5-point mean
                                      u' = ((((c + x-) + x+) + y-) + y+) * fl(1/5)
                                      ("5-point average"); padded host
                                      arrays are (ny+2)*(nx+2) (no z shell); hash init
                                      key p = j*(nx+2) + i.  TMA paths only (fused or
                                      JAC_F_PER_BLOCK). */
};

/* Options for jac_set_option. */
enum jac_option {
    JAC_OPT_LAUNCH_THREADS = 1, /* JAC_F_PER_BLOCK: host threads enqueueing the blocks'
                                  work (1..64, default 1); blocks are dealt round-robin */
    JAC_OPT_WATCHDOG_MS = 2     /* cross-partition wait limit in ms (default 60000; 0 = wait
                                  forever).  A sweep or barrier whose neighbour partition
                                  has not signalled within the limit stops waiting, the
                                  call returns JAC_ECUDA ("peer watchdog") and that call's
                                  results are invalid; the CUDA context stays usable.  Rank
                                  contexts: every rank starts its next collective call
                                  within this limit of its neighbours. */
};

/* Face kinds of the block-descriptor table (the analog of the paper's pre-filled
 * location table, "requires a runtime option that pre-fills the
 * location table", and its three transports). */
enum jac_face_kind { JAC_FACE_BOUNDARY = 0, JAC_FACE_LOCAL = 1, JAC_FACE_REMOTE = 2 };

/* ---------------------------------------------------------------- planning (host only)
 * Pure host computation, no device needed.  Validates a decomposition and returns
 * the GPU grid (given, or by the minimum-inter-GPU-face-area rule R10 when
 * gpu_grid_in is NULL; ties prefer splitting z, then y, then x) and the uniform
 * block extent.  gpu_grid_out[3] and block_extent_out[3] are caller-owned. */
int jac_plan(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz,
             int32_t n_gpus, const int32_t *gpu_grid_in, int32_t *gpu_grid_out,
             int64_t *block_extent_out);

/* Face kind and neighbour of face f (0..5 = x-,x+,y-,y+,z-,z+) of block (ix,iy,iz)
 * under the plan above.  *owner = partition owning the neighbour (or -1 at the
 * global boundary).  Host only. */
int jac_plan_face(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz,
                  int32_t n_gpus, const int32_t *gpu_grid_in, int32_t ix, int32_t iy,
                  int32_t iz, int32_t f, int32_t *kind, int32_t *owner);

/* ---------------------------------------------------------------- lifecycle
 * jac_create: one process drives all n_gpus partitions.
 * Partition g runs on CUDA device g: the context holds one sub-context per device,
 * neighbour devices get peer access (cudaDeviceEnablePeerAccess) and faces to another
 * GPU are stored into its ghost cells over NVLink by the sweep kernel, ordered by the
 * device-flag handshake -- the same path as jac_create_rank, with plain peer pointers
 * instead of IPC.  jac_step launches every device's iterations and returns after all
 * devices finish; the other calls fan out to the devices.  JAC_EDEVICE if fewer than
 * n_gpus devices are visible or two neighbour devices lack P2P access; JAC_EINVAL for
 * JAC_F_NCCL / JAC_F_PER_BLOCK with n_gpus > 1 (rank contexts only).  Under
 * JAC_F_VIRTUAL_GPUS every partition lives on device 0 (test mode, see the flag).
 * Allocates everything (two ghosted arrays per block, descriptor table, control
 * words, streams, events, two host-transfer staging slabs of up to 64 MiB); nothing
 * is allocated inside jac_step (PAPER.md:190-194
 * "persistent Views ... preallocated buffers"). *out receives the context. */
int jac_create(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz,
               int32_t n_gpus, const int32_t *gpu_grid, uint32_t flags, jac_ctx **out);

/* jac_create_rank: the calling process owns partition `rank` of n_gpus on CUDA
 * device `device` (one process per GPU).  Before jac_set_init the ranks exchange
 * their IPC handles (jac_export_ipc on every rank, all-gather, jac_import_ipc on
 * every rank); faces to other ranks are then stored directly into the peer's
 * ghost cells over NVLink by the sweep kernel (the single-copy replacement of the
 * paper's two-copy IPC staging).  All ranks must call jac_set_init*,
 * jac_step and jac_destroy collectively with the same arguments. */
int jac_create_rank(int64_t nx, int64_t ny, int64_t nz, int32_t bx, int32_t by, int32_t bz,
                    int32_t n_gpus, const int32_t *gpu_grid, int32_t rank, int32_t device,
                    uint32_t flags, jac_ctx **out);

/* Bytes of one rank's exported handle record (a cudaIpcMemHandle plus layout
 * fingerprint). */
size_t jac_ipc_handle_bytes(void);
/* Writes this rank's record into out[jac_ipc_handle_bytes()]. */
int jac_export_ipc(jac_ctx *c, void *out);
/* all = n_gpus records in rank order (all-gathered by the caller).  Opens the
 * neighbours' memory, fills REMOTE face pointers of the device table. */
int jac_import_ipc(jac_ctx *c, const void *all);

/* JAC_F_NCCL bootstrap (instead of the IPC exchange): rank 0 calls
 * jac_nccl_get_unique_id(out[jac_nccl_id_bytes()]), the caller broadcasts the bytes,
 * every rank calls jac_nccl_init (collective; creates the communicator on the
 * context's device).  libnccl.so.2 is loaded at run time; JAC_ENCCL if missing. */
size_t jac_nccl_id_bytes(void);
int jac_nccl_get_unique_id(void *out);
int jac_nccl_init(jac_ctx *c, const void *id);

/* Copies the padded initial field (host, see conventions) into BOTH ghosted
 * buffers of every local block, ghosts included, so the shell is Dirichlet data in
 * both ("outer halo = initial boundary values") and the first sweep's
 * ghosts are the neighbours' initial values.  Resets iterations_done to 0.  The
 * data moves through device staging slabs (whole planes / rows per slab, a kernel
 * scatters each into the blocks); a pinned host array is read by DMA at the link
 * rate, a pageable one is staged again by the driver. */
int jac_set_init(jac_ctx *c, const double *padded);
/* Same as jac_set_init for a sub-box of the padded global array: `box` holds
 * extent[2] x extent[1] x extent[0] doubles (x fastest) whose element (0,0,0) is
 * padded global cell (origin[0], origin[1], origin[2]).  It must cover the ghosted
 * region of every local block (jac_local_box returns the smallest such box), else
 * JAC_EINVAL.  This is how one rank of a multi-GPU run initialises its partition
 * without holding the whole grid. */
int jac_set_init_box(jac_ctx *c, const double *box, const int64_t *origin, const int64_t *extent);
/* Padded-coordinate bounding box (origin[3], extent[3]) of this context's local
 * blocks, ghost layers included. */
int jac_local_box(const jac_ctx *c, int64_t *origin, int64_t *extent);
/* Device-side synthetic init: every padded cell p gets R11's splitmix64 hash value
 * of key (seed << 40) + p, scaled to [0,1). */
int jac_set_init_hash(jac_ctx *c, uint64_t seed);

/* Runs exactly n_iters >= 0 Jacobi sweeps (R12; 0 = identity; accumulates across
 * calls).  Blocking: returns after this context's GPUs finish.  The first call after
 * jac_create (or the first jac_profile_sweep) also times the two ring depths of the
 * wide tile on the initialised field (18 extra sweeps that write only the other
 * buffer's interiors; results unaffected) unless JAC_AUTOTUNE=0 / JAC_VARIANT are set
 * as experiment knobs.  JAC_ECUDA with "peer watchdog" if a neighbour partition did
 * not signal within JAC_OPT_WATCHDOG_MS (the results of this call are then invalid). */
int jac_step(jac_ctx *c, int32_t n_iters);

/* Interior of block (ix,iy,iz) after the sweeps so far, ex*ey*ez doubles, x fastest,
 * into caller-owned host `out`.  The block must be local to this context. */
int jac_get_block(jac_ctx *c, int32_t ix, int32_t iy, int32_t iz, double *out);
/* Debug (pin P11): the whole ghosted block of the current buffer.  Rank contexts: a
 * neighbour rank may still be storing into this block's ghosts until every rank has
 * returned from its jac_step -- call it after a collective barrier for valid ghosts
 * (interiors are always valid).  Single-process contexts synchronise all devices in
 * jac_step, so no barrier is needed.
 * (ex+2)*(ey+2)*(ez+2) doubles, x fastest.  In the dense row layout (3-D blocks with
 * ex % 8 == 0) the x-edge cells of the ghost rows and planes (x ghost
 * column with a y or z ghost index) are not stored -- the stencil never reads them --
 * and are returned as NaN. */
int jac_get_block_padded(jac_ctx *c, int32_t ix, int32_t iy, int32_t iz, double *out);
/* Interiors of all local blocks written into the padded host array (shell and
 * non-local blocks untouched). */
int jac_get_field(jac_ctx *c, double *padded);
/* Interiors of all local blocks written into a padded sub-box laid out as for
 * jac_set_init_box (cells outside local interiors untouched).  The box must cover the
 * local interiors (not necessarily their ghost layer): a box of exactly the interiors
 * is read back with one linear copy per staging slab. */
int jac_get_field_box(jac_ctx *c, double *box, const int64_t *origin, const int64_t *extent);

/* Interior sub-box [lo, lo+ext) (0-based interior coordinates, x fastest) into
 * caller-owned host `out` (ext[2]*ext[1]*ext[0] doubles).  Every cell must belong to
 * a block local to this context.  For probes and sampled parity checks of grids too
 * large to read back whole. */
int jac_get_region(jac_ctx *c, const int64_t *lo, const int64_t *ext, double *out);

int jac_get_layout(const jac_ctx *c, int32_t *gpu_grid, int64_t *block_extent,
                   int64_t *iterations_done);
/* The creation arguments: interior dims n[3] (x, y, z), global blocks[3] and flags
 * (any pointer may be NULL).  Lets a caller size host arrays for a context it holds. */
int jac_get_grid(const jac_ctx *c, int64_t *n, int32_t *blocks, uint32_t *flags);
/* Partition (GPU) owning block (ix,iy,iz). */
int jac_block_owner(const jac_ctx *c, int32_t ix, int32_t iy, int32_t iz, int32_t *gpu);

/* Device time of the last jac_step (CUDA events recorded on the launching
 * stream(s) around its launches; max over this context's devices), in ms. */
int jac_last_step_ms(const jac_ctx *c, double *ms);
/* Runs n_iters iterations as one captured graph (same stream, same kernels and launch
 * attributes as jac_step); returns the median sweep-kernel duration in ms (the
 * roofline's per-launch figure): each TMA sweep records its span on the device clock
 * (first CTA start after the dependency wait, last CTA end); the plain-load ablation
 * kernel is bracketed by CUDA event-record nodes.  Advances the state like jac_step. */
int jac_profile_sweep(jac_ctx *c, int32_t n_iters, double *avg_sweep_ms);
/* Median device-time gap, in ms, between the end of one sweep launch and the start
 * of the next inside the last jac_profile_sweep graph (n_iters >= 2): the per-
 * iteration launch / dependency cost of the graph-replayed iteration (in the fused
 * mode nothing else runs between sweeps).
 * JAC_ESTATE before such a profile.  The launch/sync-gap evidence SURVEY.md §8(d.1)
 * asks of an nsys timeline, on the device clock. */
int jac_last_profile_gap_ms(const jac_ctx *c, double *gap_ms);

enum jac_stat {
    JAC_STAT_KERNEL_LAUNCHES = 0, /* our kernels launched so far (graph nodes counted) */
    JAC_STAT_GRAPH_LAUNCHES = 1,
    JAC_STAT_KERNELS_PER_ITER = 2,
    JAC_STAT_LOCAL_BLOCKS = 3,
    JAC_STAT_LOCAL_FACES = 4,     /* exchanged faces inside a partition per iteration */
    JAC_STAT_REMOTE_FACES = 5,    /* exchanged faces between partitions per iteration */
    JAC_STAT_REMOTE_BYTES = 6,    /* bytes stored to other partitions per iteration */
    JAC_STAT_ARENA_BYTES = 7,     /* device bytes of the ghosted block arena */
    JAC_STAT_SWEEP_VARIANT = 8,   /* sweep tile variant (kernels.hpp TmaVariant; 2 = plain loads) */
    JAC_STAT_PARTITIONS = 9,      /* partitions hosted (1 per device; n_gpus when virtual) */
    JAC_STAT_REMOTE_ITEMS = 10,   /* sweep work items that wait / signal (fused sync), per iteration */
    JAC_STAT_FUSED_SYNC = 11,     /* 1: cross-partition ordering runs inside the sweep */
    JAC_STAT_EPOCH_MIN = 12,      /* min / max over hosted partitions of the epoch word: the */
    JAC_STAT_EPOCH_MAX = 13,      /* synchronised phases (sweeps + barriers) completed */
    JAC_STAT_EXPERIMENT = 14,     /* bit mask of active experiment knobs (JAC_EXPERIMENT=1);
                                     0 in production: no environment variable changes the library */
    JAC_STAT_PEER_WAIT_NS = 15,   /* last jac_profile_sweep: median over its sweeps of the time the
                                     remote CTAs spent waiting for neighbour signals, summed (ns) */
    JAC_STAT_PEER_WAIT_MAX_NS = 16, /* ... and the longest single wait (ns); group: max over devices */
    JAC_STAT_N = 17
};
int jac_get_stats(const jac_ctx *c, int64_t *stats /* [JAC_STAT_N] */);

/* Sets a run-time option (enum jac_option).  JAC_EINVAL for an unknown option or
 * an out-of-range value. */
int jac_set_option(jac_ctx *c, int32_t option, int64_t value);

/* NULL-safe.  Rank contexts: every rank must have finished its last jac_step
 * (caller barrier) before any rank destroys. */
int jac_destroy(jac_ctx *c);

const char *jac_last_error(void);
int jac_version(void); /* 10000*major + 100*minor + patch */

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* JACOBI3D_H */
