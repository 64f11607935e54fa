/*
 * jacobi3d_microbench.h -- the paper's runtime microbenchmarks re-measured on B200
 * (SURVEY.md §8(f) NEXT-3 and NEXT-4), exported by libjacobi3d.so.  These are
 * measurements of the GPU runtime the overdecomposed path runs on, not part of the
 * Jacobi hot path.  All functions return JAC_OK (0) or a negative jac_status
 * (jacobi3d.h); jac_last_error() explains failures.  Times are microseconds.
 */
#ifndef JACOBI3D_MICROBENCH_H
#define JACOBI3D_MICROBENCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* E1 (§3.1): "a CPU core ... fires an empty kernel, waits for its
 * completion, and then fires the next kernel, repeatedly".  Mean round trip of
 * launch + cudaStreamSynchronize over `iters` launches on `device`. */
int jac_mb_launch_latency(int32_t device, int32_t iters, double *us_per_kernel);

/* E2 (Fig. fullOverlap): `total_threads` CUDA threads of work are
 * split into `odf` kernels on `odf` streams, all enqueued up front behind a
 * cuStreamWaitValue32 on a host-mapped flag, then released at once.  Each thread
 * runs `work` dependent FMA iterations.  *host_us = host time from releasing the flag
 * to the completion of every stream; *device_us = span between the earliest kernel
 * start and the latest kernel end (%globaltimer). */
int jac_mb_overlap(int32_t device, int64_t total_threads, int32_t odf, int32_t work, double *host_us,
                   double *device_us);

/* E3 (Fig. kernel_launch_rate): `threads` host threads (the paper's
 * PEs) each own `chares` chares with one stream each; a chare fires its next kernel
 * as soon as its previous one completed (polled, like the Charm++ scheduler polling
 * HAPI completions).  Each kernel occupies every SM (one empty CTA per SM x 4) and
 * does no work.  Counts completions over `seconds`. */
int jac_mb_launch_rate(int32_t device, int32_t chares, int32_t threads, double seconds, double *kernels_per_s);

/* E4/E5 (Figs. overdecomposed-comms / -compute): `total_bytes`
 * moved from device `src` to device `dst` over NVLink split into `odf` sender /
 * receiver pairs (one stream pair and one cudaMemcpyPeerAsync each); with
 * `with_compute` != 0 every receive is followed by an O(n) kernel on the received
 * message on the destination.  *us = time until the last transfer (and kernel) done.
 * The source holds a counter-based byte pattern; after timing, one more transfer
 * (without the consumer kernel) lands in a zeroed destination and every delivered
 * byte is compared with the source on the destination device (byte conservation,
 * SPEC.md:398): any difference returns JAC_ECUDA naming the count. */
int jac_mb_pipeline(int32_t src, int32_t dst, int64_t total_bytes, int32_t odf, int32_t with_compute, double *us);

/* E4/E5 with the design's transport: the same `odf` messages (separate buffers,
 * 4 KiB apart) moved by ONE kernel on `src` that stores them into `dst`'s memory over
 * NVLink (message table on the device, as the sweep's face table); with
 * `with_compute` one batched O(n) kernel on `dst` consumes all messages.  Host wall
 * time from launch until both devices are done, best of 5.  Delivery verified as for
 * jac_mb_pipeline. */
int jac_mb_pipeline_batched(int32_t src, int32_t dst, int64_t total_bytes, int32_t odf, int32_t with_compute,
                            double *us);
/* Bytes the calling thread's last jac_mb_pipeline[_batched] call verified (0 before). */
int64_t jac_mb_last_verified_bytes(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif
